# ncu capture of the C2 kernel (K1f, gj_blk32_kernel<2,4,2,1>) + per-opcode source page; run under gpurun.
set -e
mkdir -p gpurun_out
python tools/profile_k1b_once.py
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:'gj_blk32_kernelILi2ELi4ELi2ELi1E' -s 1 -c 1 -f -o gpurun_out/k1b python tools/profile_k1b_once.py > gpurun_out/k1b_ncu.log 2>&1
ncu -i gpurun_out/k1b.ncu-rep --page source --csv --print-source sass > gpurun_out/k1b_src.csv
ncu -i gpurun_out/k1b.ncu-rep --page raw --csv > gpurun_out/k1b_raw.csv
python tools/ncu_sass_hist.py gpurun_out/k1b_src.csv 1048576 > gpurun_out/k1b_hist.txt
