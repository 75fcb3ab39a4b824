# A/B of reconstruction-kernel builds (libnnb_v*.so, one per variant): the dense bench leg's
# live per-kernel timing for each, then the Ozaki parity tests on the last variant listed.
# Usage: tools/recon_ab.sh "3 4 3 4"   Outputs gpurun_out/ab_v*.json.
cd "$(dirname "$0")/.."
P=paper_2212_02406_b200
cp $P/libnnb.so /tmp/libnnb_keep.so
for v in $1; do
  cp $P/libnnb_v$v.so $P/libnnb.so
  timeout 400 python bench.py --legs dense --steps 3 --warmup 3 --no-cpu --no-e2e --no-dmma --no-symmetric --no-emulated \
    > gpurun_out/ab_v$v.json 2> gpurun_out/ab_v$v.err
done
timeout 900 python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_c3_golden.py tests/test_gpu_symmetric.py -x -q \
  > gpurun_out/ab_tests.txt 2>&1
cp /tmp/libnnb_keep.so $P/libnnb.so
echo done
