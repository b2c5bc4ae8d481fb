"""The engine's multi-rank path on the GPU: 1, 2 and 3 ranks (processes
sharing one GPU; per-level record all-gather over gloo through
sabr_ctx_init_host_exchange instead of NCCL) must return bit-identical
reports for every calibrator: chains are keyed by their global index and the
merge is a lexicographic (value, chain) minimum (annealer.cpp:141-159).  With
fewer T_II chains than ranks (or SABR_T2_SHARD=paths) the ranks split the MC
path tiles instead and all-gather the tile partials every SA step; the tile
reduction order is the single-rank one, so those reports are identical too."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORKER = os.path.join(ROOT, "tests", "mr_engine_worker.py")


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def run(world, peer=False):
    port = free_port()
    extra = ["peer"] if peer else []
    procs = [subprocess.Popen([sys.executable, WORKER, str(r), str(world), str(port)] + extra, cwd=ROOT,
                              stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True) for r in range(world)]
    outs = [p.communicate(timeout=900) for p in procs]
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, e[-3000:]
    return json.loads(outs[0][0].strip().splitlines()[-1])


def test_ranks_give_identical_reports():
    one = run(1)
    for world in (2, 3):
        many = run(world)
        assert many.keys() == one.keys()
        for k in one:
            assert many[k] == one[k], (world, k)


def test_fused_peer_exchange_gives_identical_reports():
    """The T_I level kernels' last CTAs exchange the level records through
    CUDA-IPC mailboxes (peer memory) and merge in-kernel: same reports as one
    rank (the other calibrators keep the host all-gather)."""
    one = run(1)
    for world in (2, 3):
        many = run(world, peer=True)
        for k in one:
            assert many[k] == one[k], (world, k)
