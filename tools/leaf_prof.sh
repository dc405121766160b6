# Diagnostic: the library built with -DGJ_LEAF_PROF into /tmp, per-phase cycle sums of the
# leaf step (thread 0 of CTA 0) for one n = 8192 fp64 / fp32 inversion.
set -e
mkdir -p /tmp/leafprof
cd paper_1401_7962_b200/csrc
for f in $(ls *.cu | sed "s/\.cu$//"); do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -DGJ_LEAF_PROF -I ../../include -c $f.cu -o /tmp/leafprof/$f.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o /tmp/leafprof/libgjinv.so /tmp/leafprof/*.o -lcuda
cd ../..
python tools/leaf_prof.py
