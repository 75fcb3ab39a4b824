# int8 peak + ncu full capture of one oz_gemm_kernel launch (N=8192)
python tools/microbench/int8_peak.py > gpurun_out/r02_int8_peak.json 2> gpurun_out/r02_int8_peak.err
python tools/bench_ozaki.py 8192 > gpurun_out/r02f_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:oz_gemm -c 1 -o gpurun_out/r02_oz_gemm python tools/bench_ozaki.py 8192 > gpurun_out/r02f_ncu.log 2>&1
echo done
