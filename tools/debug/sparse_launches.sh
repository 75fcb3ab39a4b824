for v in "NNB_SELL_UNROLL=1" "NNB_SPARSE_FORMAT=csr"; do
  tag=$(echo $v | tr '=' '_')
  env $v timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 150 --csv --log-file gpurun_out/sp_$tag.csv python tools/bench_sparse.py > gpurun_out/sp_$tag.log 2>&1
done
