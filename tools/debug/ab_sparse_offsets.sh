timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -q -x -k "sparse" 2>&1 | tail -2
for v in "NNB_SPARSE_OFFSETS=rows" "NNB_SPARSE_OFFSETS=groups" "NNB_SPARSE_OFFSETS=rows" "NNB_SPARSE_OFFSETS=groups"; do echo $v; env $v timeout 300 python tools/bench_sparse.py; done
