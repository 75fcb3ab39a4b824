# Round-end evidence: GPU tests, smoke, bench (both arms), prof_drive launch list, bench launch list.
mkdir -p gpurun_out
bash tools/debug/checkpoint.sh
bash tools/debug/bench_launches.sh
