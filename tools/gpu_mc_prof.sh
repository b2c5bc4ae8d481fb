# MC tile kernel captures: C4 (beta = 1) and C5 (full Case II, beta free), FP64
set -x
mkdir -p gpurun_out
timeout 400 ncu --set full --clock-control none --import-source on -k regex:mc_tile_kernel -s 2 -c 1 -o gpurun_out/full_t2 python tools/profile_kernels.py t2 > gpurun_out/prof_t2.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:mc_tile_kernel -s 2 -c 1 -o gpurun_out/full_c5 python tools/profile_kernels.py c5 > gpurun_out/prof_c5.log 2>&1
ls -la gpurun_out
