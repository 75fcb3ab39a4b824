# int8 GEMM raster group size at N=32768 (NNB_DEBUG=1 NNB_OZ_GROUP): the nest's device time
cd "$(dirname "$0")/.."
for g in 16 8 12 24 32 16; do
  echo "group $g"; NNB_DEBUG=1 NNB_OZ_GROUP=$g timeout 300 python tools/sharded_emul_scan.py 32768 "" 2>&1 | grep single
done
