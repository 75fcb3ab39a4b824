# CRT reconstruction change: GPU suite, the dense bench leg, and one full capture of the
# reconstruction kernel at N=32768.  Outputs under gpurun_out/crt_*.
cd "$(dirname "$0")/.."
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/crt_gpu_suite.txt 2>&1; echo "rc=$?" >> gpurun_out/crt_gpu_suite.txt
L="--legs dense --steps 3 --warmup 3 --no-cpu --no-dmma --no-symmetric --no-emulated"
timeout 600 python bench.py $L > gpurun_out/crt_dense.json 2> gpurun_out/crt_dense.err; echo "rc=$?" >> gpurun_out/crt_dense.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"oz_recon" -s 2 -c 1 \
  -o gpurun_out/crt_recon32k python bench.py --legs dense --steps 1 --warmup 1 --no-cpu --no-e2e --no-dmma --no-symmetric --no-emulated \
  > gpurun_out/crt_recon_ncu.log 2>&1
echo done
