M="gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,gpc__cycles_elapsed.avg.per_second"
python tools/bench_ozaki.py 16384 > gpurun_out/r02m_plain.log 2>&1
for g in 4 8 16 32; do
NNB_DEBUG=1 NNB_OZ_GROUP=$g ncu --metrics $M --clock-control none -k regex:oz_gemm -c 1 --csv python tools/bench_ozaki.py 16384 > gpurun_out/r02m_g$g.csv 2>&1
NNB_DEBUG=1 NNB_OZ_GROUP=$g python tools/bench_ozaki.py 16384 32768 > gpurun_out/r02m_g$g.log 2>&1
done
echo done
