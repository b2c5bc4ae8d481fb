# MC kernel iteration: MC/T_II parity tests, ncu kernel metrics for C4/C5, bench with secondary items
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -rf -k "mc or case2 or cliquet" > gpurun_out/pytest_gpu.log 2>&1
M=gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,launch__registers_per_thread,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum
timeout 300 ncu --metrics $M -k regex:mc_tile --clock-control none --csv --log-file gpurun_out/ncu_mc_t2.csv python tools/profile_kernels.py t2 > /dev/null 2>&1
timeout 300 ncu --metrics $M -k regex:mc_tile --clock-control none --csv --log-file gpurun_out/ncu_mc_c5.csv python tools/profile_kernels.py c5 > /dev/null 2>&1
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1
if [ "${FULL:-0}" = "1" ]; then timeout 400 ncu --set full --clock-control none --import-source on -k regex:mc_tile_kernel -s 2 -c 1 -o gpurun_out/full_t2 python tools/profile_kernels.py t2 > /dev/null 2>&1; fi
ls -la gpurun_out
