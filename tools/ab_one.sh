# Build a variant of the library into ab/$1/libgjinv.so: every object from the in-tree build
# except $2 (one .cu), which is recompiled with the extra nvcc flags that follow.
#   bash tools/ab_one.sh k2_off gj_batched64e.cu -DGJ_K2_SMSP_ROLES=0
set -e
name=$1; src=$2; shift 2
out=ab/$name
mkdir -p $out
cp paper_1401_7962_b200/csrc/build/*.o $out/
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr "$@" \
  -I include -c paper_1401_7962_b200/csrc/$src -o $out/${src%.cu}.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $out/libgjinv.so $out/*.o
echo $out/libgjinv.so
