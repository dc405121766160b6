set -e
mkdir -p gpurun_out
python tools/profile_k2d_once.py > /dev/null
ncu --set full --clock-control none --import-source on -k regex:gj_batched64 -s 0 -c 1 -f -o gpurun_out/k2g python tools/profile_k2d_once.py > gpurun_out/k2g_ncu.log 2>&1
ncu -i gpurun_out/k2g.ncu-rep --page raw --csv > gpurun_out/k2g_raw.csv
ncu -i gpurun_out/k2g.ncu-rep --page source --csv --print-source sass > gpurun_out/k2g_src.csv
