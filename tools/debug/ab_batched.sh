set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "batched or mimo" 2>&1 | tail -5
for v in 3m_nopf 4m_nopf 3m 4m; do NNB_BATCHED_VARIANT=$v timeout 120 python tools/bench_batched.py; done
