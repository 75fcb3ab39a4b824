# round-2 evidence run: GPU suite, bench (both arms), ncu launch list of the bench, full captures
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02_final_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02_final_pytest.log
timeout 900 python bench.py > gpurun_out/r02_final_bench.json 2> gpurun_out/r02_final_bench.err; echo "rc=$?" >> gpurun_out/r02_final_bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02_final_ref.json 2> gpurun_out/r02_final_ref.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_final_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r02_final_smoke.log
python bench.py --legs dense --steps 2 --warmup 1 --no-cpu --no-e2e --no-dmma --no-symmetric > gpurun_out/r02_launch_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_bench_launches.csv python bench.py --legs dense --steps 2 --warmup 1 --no-cpu --no-e2e --no-dmma --no-symmetric > gpurun_out/r02_launch_ncu.log 2>&1
python tools/prof_sparse_tb.py > gpurun_out/r02_tb_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:stencil_tb -s 12 -c 1 -o gpurun_out/r02_stencil_tb python tools/prof_sparse_tb.py > gpurun_out/r02_tb_ncu.log 2>&1
python tools/bench_ozaki.py 8192 > gpurun_out/r02_oz_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"oz_gemm|oz_recon|oz_split" -c 4 -o gpurun_out/r02_oz_all python tools/bench_ozaki.py 8192 > gpurun_out/r02_oz_ncu.log 2>&1
echo done
