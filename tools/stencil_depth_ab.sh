cd $GRAFT_REPO_ROOT
python -m pytest tests -m gpu -x -q -k "sparse or c5 or stencil" > gpurun_out/s67_tests.log 2>&1; tail -2 gpurun_out/s67_tests.log
for d in 4 8 4 8; do
 NNB_DEBUG=1 NNB_STENCIL_DEPTH=$d python bench.py --legs sparse --no-cpu --no-e2e --steps 5 --warmup 3 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); s=d['legs']['sparse']; print('depth $d', s['ms_per_step'], s['sharded_emulated']['schedule_ms_all_ranks'], s['clocks']['sm_mhz'])"
done
