# A/B: 2-SM (cta_group::2) vs 1-SM int8 GEMM in the Ozaki emulation
timeout 300 python -m pytest tests/test_gpu_ozaki.py -x -q > gpurun_out/${1}_oz_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${1}_oz_tests.log
timeout 300 python tools/bench_ozaki.py 4096 8192 16384 > gpurun_out/${1}_oz_pair.log 2>&1; echo "rc=$?" >> gpurun_out/${1}_oz_pair.log
NNB_DEBUG=1 NNB_OZ_SINGLE_SM=1 timeout 300 python tools/bench_ozaki.py 4096 8192 16384 > gpurun_out/${1}_oz_single.log 2>&1
echo done
