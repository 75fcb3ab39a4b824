CMD="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e"
timeout 1200 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 2400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/bench_launches.csv $CMD > gpurun_out/ncu_bench.log 2>&1
echo "rc=$?"; tail -c 300 gpurun_out/plain.log
