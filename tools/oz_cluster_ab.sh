# A/B of the int8 GEMM with and without B multicast across CTA pairs (NNB_OZ_CLUSTER=2):
# parity tests, then the device nest at N=32768 (tools/sharded_emul_scan.py prints the
# per-class device time) for each setting
cd "$(dirname "$0")/.."
NNB_DEBUG=1 NNB_OZ_CLUSTER=2 timeout 300 python -m pytest tests/test_gpu_ozaki.py -q -x > gpurun_out/ozc_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/ozc_pytest.log
for c in 1 2 1 2; do
  NNB_DEBUG=1 NNB_OZ_CLUSTER=$c timeout 300 python tools/sharded_emul_scan.py 32768 1 >> gpurun_out/ozc_scan_$c.log 2>&1
done
