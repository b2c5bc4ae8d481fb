# SA level-kernel iteration: latency probe, parity tests of the SA paths, bench (no secondary), ncu metrics
set -x
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/latency_probe tools/latency_probe.cu && /tmp/latency_probe > gpurun_out/latency.log 2>&1
timeout 600 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -rf -k "annealer or calibration or kernel_variants or costs" > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/bench.log 2>&1
M=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread
for m in sa case1; do timeout 300 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/ncu_metrics_$m.csv python tools/profile_kernels.py $m > gpurun_out/prof_$m.log 2>&1; done
if [ "${FULL:-0}" = "1" ]; then timeout 300 ncu --set full --clock-control none --import-source on -k regex:sa_level -s 1 -c 1 -o gpurun_out/full_sa python tools/profile_kernels.py sa > /dev/null 2>&1; fi
ls -la gpurun_out
