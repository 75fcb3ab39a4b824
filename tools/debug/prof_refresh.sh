timeout 300 python tools/prof_drive.py mimo > gpurun_out/pd_mimo.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:batched_z16_kernel -c 1 \
    -o gpurun_out/prof_batched_r01e python tools/prof_drive.py mimo > gpurun_out/ncu_b.log 2>&1
timeout 300 python tools/bench_complex.py 4096 > gpurun_out/pd_cplx.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum --clock-control none \
    --csv --log-file gpurun_out/launches_cplx.csv python tools/bench_complex.py 4096 > gpurun_out/ncu_c.log 2>&1
ls -la gpurun_out/*.ncu-rep gpurun_out/launches_cplx.csv
