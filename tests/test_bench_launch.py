"""bench.py's launch contract: --gpus N is authoritative.  Without a launcher
and N > 1 it re-executes itself under torch.distributed.run with N ranks; under
a launcher whose WORLD_SIZE differs from N it exits non-zero.  The GPU test runs
the N = 2 path end to end with both ranks on one GPU (SABR_BENCH_SHARED_GPU=1:
gloo for torch's collectives, the engine's host all-gather / peer mailboxes)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_single_gpu_runs_in_process():
    assert bench.launch_plan(1, {}, []) == ("run", None)
    assert bench.launch_plan(1, {"WORLD_SIZE": "1"}, []) == ("run", None)


def test_multi_gpu_without_launcher_reexecs_under_torchrun():
    what, cmd = bench.launch_plan(8, {}, ["--gpus", "8", "--steps", "5"])
    assert what == "exec"
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=8" in cmd and "--master-addr=127.0.0.1" in cmd
    assert cmd[-4:] == ["--gpus", "8", "--steps", "5"]
    assert os.path.basename(cmd[cmd.index("--master-addr=127.0.0.1") + 2]) == "bench.py"


def test_launcher_world_size_must_match_gpus():
    assert bench.launch_plan(4, {"WORLD_SIZE": "4"}, []) == ("run", None)
    what, msg = bench.launch_plan(8, {"WORLD_SIZE": "1"}, [])
    assert what == "error" and "WORLD_SIZE=1" in msg
    assert bench.launch_plan(0, {}, [])[0] == "error"


def test_mismatch_exits_nonzero():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "3"], env=env,
                       capture_output=True, text=True, timeout=300)
    assert p.returncode == 2 and "--gpus 3" in p.stderr


@pytest.mark.gpu
def test_bench_two_ranks_shared_gpu():
    env = dict(os.environ, SABR_BENCH_SHARED_GPU="1", MASTER_PORT="29617")
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        env.pop(k, None)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1", "--warmup", "1",
                        "--no-secondary", "--no-cpu-baseline"], env=env, capture_output=True, text=True,
                       timeout=900, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-3000:]
    line = json.loads([l for l in p.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["config"]["chains"] == 200_000
    assert "rank 0/2" in p.stderr and "rank 1/2" in p.stderr
