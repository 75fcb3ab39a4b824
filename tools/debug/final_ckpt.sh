mkdir -p gpurun_out
bash tools/debug/checkpoint.sh
timeout 300 python tools/prof_drive.py mimo > gpurun_out/pd_mimo.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:batched_z16_kernel -c 1 \
    -o gpurun_out/prof_batched_herm_r01 python tools/prof_drive.py mimo > gpurun_out/ncu_b.log 2>&1
timeout 300 python tools/prof_drive.py detect > gpurun_out/pd_det.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:mimo_detect_kernel -c 1 \
    -o gpurun_out/prof_detect_herm_r01 python tools/prof_drive.py detect > gpurun_out/ncu_d.log 2>&1
ls -la gpurun_out/*.ncu-rep
