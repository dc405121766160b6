# Build a variant of the library with extra nvcc flags into $1 (e.g. /tmp/ab1/libgjinv.so):
#   bash tools/ab_build.sh /tmp/ab1 -DGJ_K1B_UNROLL=2
set -e
out=$1; shift
mkdir -p $out
cd paper_1401_7962_b200/csrc
for f in $(ls *.cu | sed "s/\.cu$//"); do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr "$@" -I ../../include -c $f.cu -o $out/$f.o &
done
wait
for f in $(ls *.cu | sed "s/\.cu$//"); do test -f $out/$f.o || { echo "ab_build: $f.cu failed to compile" >&2; exit 1; }; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $out/libgjinv.so $out/*.o -lcuda
