# state check on a fresh box: smoke, GPU parity tests, both bench arms, launch list, full capture of the C2 kernel
set -x
mkdir -p gpurun_out
timeout 200 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1
timeout 600 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -rf > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python bench.py --steps 2 --warmup 3 > gpurun_out/bench.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-secondary --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:sa_level -s 1 -c 1 -o gpurun_out/full_sa python tools/profile_kernels.py sa > /dev/null 2>&1
ls -la gpurun_out
