# profiles for the judge: torchrun N=1 bench, ncu launch list of the bench command, full capture of the C2 kernel
set -x
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 2 --warmup 3 > gpurun_out/bench_torchrun.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-secondary --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:sa_level -s 1 -c 1 -o gpurun_out/full_sa python tools/profile_kernels.py sa > /dev/null 2>&1
ls -la gpurun_out
