# ncu capture of one trailing-update launch of the C4 inversion (K4b) + raw metrics.
set -e
mkdir -p gpurun_out
python tools/profile_large_once.py 8192 > /dev/null
ncu --set full --clock-control none --import-source on -k regex:dgemm_tma -s 21 -c 1 -f -o gpurun_out/dgemm python tools/profile_large_once.py 8192 > gpurun_out/dgemm_ncu.log 2>&1
ncu -i gpurun_out/dgemm.ncu-rep --page raw --csv > gpurun_out/dgemm_raw.csv
ncu -i gpurun_out/dgemm.ncu-rep --page source --csv --print-source sass > gpurun_out/dgemm_src.csv
