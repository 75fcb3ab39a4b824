# complex dense chain: FAST (3M over int8-emulated products at N >= 3072) vs DMMA
cd "$(dirname "$0")/.."
for n in 4096 8192; do
  timeout 300 python tools/bench_complex.py $n
  NNB_ARITHMETIC=dmma timeout 300 python tools/bench_complex.py $n
done
