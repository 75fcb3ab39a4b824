timeout 300 python tools/bench_sparse.py > /dev/null 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__cycles_active.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed \
  --clock-control none -k regex:spmv_factor_pipeline -s 4 -c 1 python tools/bench_sparse.py 2>&1 | grep -E "spmv_factor|duration|bytes|hit_rate|warps_active|cycles_active|throughput" | head -20
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,lts__t_sector_hit_rate.pct,lts__throughput.avg.pct_of_peak_sustained_elapsed \
  --clock-control none -k regex:spmv_rows_kernel -s 3 -c 1 python tools/bench_sparse.py 2>&1 | grep -E "spmv_rows|duration|bytes|hit_rate|throughput" | head -10
