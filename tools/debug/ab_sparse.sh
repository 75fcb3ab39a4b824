set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -q -x -k "sparse" 2>&1 | tail -3
for v in "NNB_SPARSE_COL=32" "NNB_SPARSE_COL=16" "NNB_SPARSE_COL=32" "NNB_SPARSE_COL=16"; do env $v timeout 300 python tools/bench_sparse.py; done
NNB_SPARSE_COL=16 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 100 --csv --log-file gpurun_out/sp_col16.csv python tools/bench_sparse.py > /dev/null 2>&1
