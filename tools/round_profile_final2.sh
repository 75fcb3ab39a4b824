# Round-2 final evidence after the CRT reconstruction: GPU suite, bench (both arms), smoke, the ncu launch list of the dense bench
# leg (with DRAM bytes), full captures of the int8 GEMM / split / reconstruction at N=32768
# and of the temporal-blocked stencil pass.  Outputs under gpurun_out/final2_*.
cd "$(dirname "$0")/.."
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/final2_gpu_suite.txt 2>&1; echo "rc=$?" >> gpurun_out/final2_gpu_suite.txt
timeout 900 python bench.py > gpurun_out/final2_bench.json 2> gpurun_out/final2_bench.err; echo "rc=$?" >> gpurun_out/final2_bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/final2_ref.json 2> gpurun_out/final2_ref.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final2_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/final2_smoke.log
L="--legs dense --steps 2 --warmup 1 --no-cpu --no-e2e --no-dmma --no-symmetric --no-emulated"
timeout 600 python bench.py $L > gpurun_out/final2_launch_plain.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/final2_bench_launches.csv python bench.py $L > gpurun_out/final2_launch_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"oz_gemm|oz_recon|oz_split" -s 6 -c 4 \
  -o gpurun_out/final2_oz32k python bench.py $L > gpurun_out/final2_oz_ncu.log 2>&1
timeout 300 python tools/prof_sparse_tb.py > gpurun_out/final2_tb_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stencil_tb -s 12 -c 1 \
  -o gpurun_out/final2_stencil_tb python tools/prof_sparse_tb.py > gpurun_out/final2_tb_ncu.log 2>&1
echo done
