# one full gpurun round: smoke, GPU tests, launch list of the bench command, ncu metrics of every
# hot kernel (-> profiles/fp64_per_eval.json), both bench arms (+ torchrun N=1, full configs), full
# captures of the C2 / C3 / C4 kernels, sanitizers
#   TESTS=0 skips the GPU test suite, FULL=0 the ncu --set full captures
set -x
mkdir -p gpurun_out
timeout 200 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1
if [ "${TESTS:-1}" = "1" ]; then
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rf --durations=30 > gpurun_out/pytest_gpu.log 2>&1
fi
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-secondary --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
M=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__inst_executed_pipe_fp64.sum,smsp__inst_executed_pipe_xu.sum,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum
for m in sa case1 t2 mc c5; do timeout 400 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/ncu_metrics_$m.csv python tools/profile_kernels.py $m > gpurun_out/prof_$m.log 2>&1; done
for m in t2 c5 mc; do SABR_PRECISION=fp32 timeout 300 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/ncu_metrics_${m}_fp32.csv python tools/profile_kernels.py $m > gpurun_out/prof_${m}_fp32.log 2>&1; done
# the per-unit instruction counts of this build first, so the bench's rooflines use them
python tools/update_flops.py round > gpurun_out/update_flops.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --full-configs --no-cpu-baseline > gpurun_out/bench_full.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 2 --warmup 3 --no-secondary > gpurun_out/bench_torchrun.log 2>&1
if [ "${FULL:-1}" = "1" ]; then
timeout 300 ncu --set full --clock-control none --import-source on -k regex:sa_level -s 1 -c 1 -o gpurun_out/full_sa python tools/profile_kernels.py sa > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:sa_level -s 1 -c 1 -o gpurun_out/full_case1 python tools/profile_kernels.py case1 > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:mc_tile_kernel -s 2 -c 1 -o gpurun_out/full_t2 python tools/profile_kernels.py t2 > /dev/null 2>&1
SABR_PRECISION=fp32 timeout 400 ncu --set full --clock-control none --import-source on -k regex:mc_tile_kernel -s 2 -c 1 -o gpurun_out/full_t2_fp32 python tools/profile_kernels.py t2 > /dev/null 2>&1
fi
# memory / race checks of the hot kernels (small shapes)
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python __graft_entry__.py smoke > gpurun_out/sanitizer_memcheck.log 2>&1
timeout 600 compute-sanitizer --tool racecheck --print-limit 20 python __graft_entry__.py smoke > gpurun_out/sanitizer_racecheck.log 2>&1
ls -la gpurun_out
