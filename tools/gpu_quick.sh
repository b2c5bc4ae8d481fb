# quick kernel-time comparison of the T_II MC tile kernel variants
M=gpu__time_duration.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,launch__registers_per_thread
for v in "fp64 8" "fp32 8" "fp32 4" "fp32 16"; do set -- $v
SABR_PRECISION=$1 SABR_MC_CB=$2 timeout 300 ncu --metrics $M -k regex:mc_tile --clock-control none --csv --log-file gpurun_out/q_$1_$2.csv python tools/profile_kernels.py t2 > /dev/null 2>&1
done
timeout 300 python -m pytest tests/test_gpu_mc.py -q -k fp32 > gpurun_out/q_pytest.log 2>&1
