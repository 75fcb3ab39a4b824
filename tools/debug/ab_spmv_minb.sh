set -e
for v in 1 8 1 8; do
  nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -DNNB_SPMV_MINB=$v \
    -c paper_2212_02406_b200/csrc/sparse.cu -o build/sparse.o 2>/dev/null
  nvcc -gencode arch=compute_100a,code=sm_100a -shared build/*.o -o paper_2212_02406_b200/libnnb.so -lcudart -ldl
  echo "MINB=$v"; timeout 300 python tools/bench_sparse.py
done
