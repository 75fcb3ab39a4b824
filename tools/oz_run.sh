# GPU check of the int8-emulated products: parity tests, timing vs DMMA, ncu launch list
tag=${1:-r02}
timeout 300 python -m pytest tests/test_gpu_ozaki.py -x -q > gpurun_out/${tag}_oz_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_oz_tests.log
timeout 400 python tools/bench_ozaki.py ${SIZES:-8192 16384 32768} > gpurun_out/${tag}_oz_bench.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_oz_bench.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_oz_launches.csv python tools/bench_ozaki.py 8192 > gpurun_out/${tag}_oz_ncu.log 2>&1
echo done
