set -e
for v in 256 128 512 1024 256; do
  nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC --expt-relaxed-constexpr \
    -DNNB_SPMV_THREADS=$v -c paper_2212_02406_b200/csrc/sparse.cu -o build/sparse.o
  nvcc -gencode arch=compute_100a,code=sm_100a -shared build/*.o -o paper_2212_02406_b200/libnnb.so -lcudart -ldl
  echo "THREADS=$v"; timeout 300 python tools/bench_sparse.py
done
