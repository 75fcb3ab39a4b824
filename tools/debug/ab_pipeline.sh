timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -q -x -k "sparse" 2>&1 | tail -3
for v in "NNB_SPARSE_PIPELINE=0" "NNB_SPARSE_BLOCK_ROWS=4096" "NNB_SPARSE_BLOCK_ROWS=2048" "NNB_SPARSE_BLOCK_ROWS=8192" "NNB_SPARSE_PIPELINE=0" "NNB_SPARSE_BLOCK_ROWS=4096"; do
  echo $v; env $v timeout 120 python tools/bench_sparse.py 2>&1 | tail -1
done
