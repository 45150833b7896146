# A/B diagnostics: gls_create with the library's DMMA GEMM vs cuBLAS DGEMM for the same products
# (a separate libgls build with -DGLS_AB_CUBLAS, loaded via LD_PRELOAD-free path swap).
set -e
cd paper_1210_7325_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -DGLS_AB_CUBLAS \
  -I ../../include -o ../libgls_ab.so gls_api.cu dgemm.cu chol_inv.cu fused_trsm_gls.cu ozaki_gls.cu ooc_file.cu gwfgls.cu -lcublas
cd ../..
cp paper_1210_7325_b200/libgls.so /tmp/libgls_orig.so
python tools/bench_create.py 10000 1500 2>&1 | grep create
cp paper_1210_7325_b200/libgls_ab.so paper_1210_7325_b200/libgls.so
python tools/bench_create.py 10000 1500 2>&1 | grep create
GLS_DGEMM_CUBLAS=1 python tools/bench_create.py 10000 1500 2>&1 | grep create
GLS_DGEMM_CUBLAS=1 GLS_TRACE_CHOL=1 python tools/bench_create.py 10000 2>&1 | tail -10
cp /tmp/libgls_orig.so paper_1210_7325_b200/libgls.so
