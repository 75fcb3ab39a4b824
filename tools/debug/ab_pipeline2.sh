timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "sparse_vs_reference or sparse_full" 2>&1 | tail -2
for v in "NNB_SPARSE_PIPELINE=0" "NNB_SPARSE_BLOCK_ROWS=2048" "NNB_SPARSE_BLOCK_ROWS=1024" "NNB_SPARSE_BLOCK_ROWS=4096"; do
  echo $v; env $v timeout 120 python tools/bench_sparse.py 2>&1 | tail -1
done
