# int8 GEMM L2 eviction hints (NNB_DEBUG=1 NNB_OZ_HINTS bits: 1 A evict_last, 2 B evict_first)
cd "$(dirname "$0")/.."
for h in 0 1 0 1; do
  echo "hints $h"; NNB_DEBUG=1 NNB_OZ_HINTS=$h timeout 300 python tools/sharded_emul_scan.py 32768 "" 2>&1 | grep single
done
