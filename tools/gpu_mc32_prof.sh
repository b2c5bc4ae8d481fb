# FP32 MC tile kernel: pipe metrics for C4 / C5 / single-candidate pricing and one --set full capture (C4)
set -x
mkdir -p gpurun_out
M=gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,launch__registers_per_thread,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,smsp__inst_executed_pipe_xu.sum,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fmaheavy.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_xu_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active
for m in t2 c5 mc; do SABR_PRECISION=fp32 timeout 300 ncu --metrics $M -k regex:mc_tile --clock-control none --csv --log-file gpurun_out/ncu32_$m.csv python tools/profile_kernels.py $m > /dev/null 2>&1; done
if [ "${FULL:-1}" = "1" ]; then SABR_PRECISION=fp32 timeout 400 ncu --set full --clock-control none --import-source on -k regex:mc_tile_kernel -s 2 -c 1 -o gpurun_out/full_t2_f32 python tools/profile_kernels.py t2 > /dev/null 2>&1; fi
ls -la gpurun_out
