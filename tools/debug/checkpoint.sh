# Full GPU checkpoint: tests, smoke, bench, launch list, sparse ncu capture.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 1200 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?" >> gpurun_out/bench_full.err
timeout 600 python tools/prof_drive.py sparse > gpurun_out/prof_sparse_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmv_rows_kernel -s 20 -c 1 \
    -o gpurun_out/prof_spmv_r01d python tools/prof_drive.py sparse > gpurun_out/ncu_spmv.log 2>&1
timeout 600 python tools/prof_drive.py all > gpurun_out/prof_all_plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/launches_r01d.csv python tools/prof_drive.py all > gpurun_out/ncu_launches.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log | tail -2; tail -2 gpurun_out/bench_full.err
