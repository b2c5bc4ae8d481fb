"""World-size-2 (gloo, CPU) test of the multi-GPU decomposition of the
annealer: chains split contiguously over ranks, each rank reduces its chains
of a level to one record (oracle/sabr_oracle.c:orc_level_record), the records
are all-gathered, and every rank applies the engine's own merge rule
(sabr_merge_level_records = the device merge_level of the NCCL path).  The
result must be bit-identical to the single-process reference annealer for any
rank count - the reference's own "groups" two-level reduction
(annealer.cpp:141-159) is the same decomposition."""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2407_20713_b200 as pkg
from paper_2407_20713_b200 import _abi as A
from oracles import Restate, have_restate

pytestmark = pytest.mark.skipif(not have_restate(), reason="oracle restatement not built")

CASES = [
    (A.OBJ_BOWL3, [-5.0] * 3, [5.0] * 3, [0.0, 0.0, 0.0], 0, dict(workers=5, groups=3, seed=1)),
    (A.OBJ_CORNER2, [-2.0, -2.0], [2.0, 2.0], [0.0, 0.0], A.PRED_SUM_LE_1, dict(workers=7, groups=1, seed=3)),
    (A.OBJ_SQUARE1, [-1.0], [1.0], [0.5], 0, dict(workers=8, groups=2, seed=2, max_evals=700)),
]


def schedule(kw):
    return pkg.AnnealingSchedule(**{**dict(t0=5.0, cooling=0.8, chain_length=30, t_min=1e-4), **kw})


def sharded_run(rank, world, case):
    obj, lo, hi, start, pred, kw = case
    orc = Restate()
    lib = A.load_library()
    orc.lib.orc_builtin_value.restype = C.c_double
    sch = schedule(kw)
    dim = len(lo)
    lo_a, hi_a = (C.c_double * dim)(*lo), (C.c_double * dim)(*hi)
    st = A.sabr_sa_state()
    for i in range(dim):
        st.incumbent[i] = st.best[i] = start[i]
    v0 = orc.lib.orc_builtin_value(obj, (C.c_double * dim)(*start))
    st.incumbent_value = st.best_value = v0 if v0 == v0 else float("inf")
    st.evals = 1
    n_chains = sch.workers * sch.groups
    temps = []
    t = sch.t0
    while t >= sch.t_min:
        temps.append(t)
        t *= sch.cooling
    st.eval_cap = (sch.max_evals - 1 + n_chains - 1) // n_chains
    st.done = int(len(temps) == 0 or st.evals >= sch.max_evals)
    begin, end = rank * n_chains // world, (rank + 1) * n_chains // world
    trace = []
    sch_abi = sch.to_abi()
    for level, temp in enumerate(temps):
        if st.done:
            break
        rec = A.sabr_level_record()
        assert orc.lib.orc_level_record(obj, pred, lo_a, hi_a, dim, C.byref(sch_abi), C.byref(st),
                                        C.c_uint64(level), C.c_double(temp), C.c_int64(begin),
                                        C.c_int64(end), C.byref(rec)) == 0
        mine = torch.frombuffer(bytearray(bytes(rec)), dtype=torch.uint8)
        gathered = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(gathered, mine)
        recs = (A.sabr_level_record * world)()
        for r in range(world):
            C.memmove(C.addressof(recs[r]), bytes(gathered[r].numpy().tobytes()), C.sizeof(A.sabr_level_record))
        tf = C.c_double()
        assert lib.sabr_merge_level_records(C.byref(st), recs, world, n_chains, sch.max_evals, len(temps),
                                            C.byref(tf)) == 0
        trace.append((temp, tf.value))
    return list(st.best)[:dim], st.best_value, st.evals, trace


def worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = [sharded_run(rank, world, case) for case in CASES]
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2])
def test_sharded_annealer_equals_single_process(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    orc = Restate()
    for i, (obj, lo, hi, start, pred, kw) in enumerate(CASES):
        want = orc.minimize_builtin(obj, lo, hi, schedule(kw), start, predicate=pred)
        for r in range(world):
            best, value, evals, trace = results[r][i]
            assert evals == want.evals
            assert value == want.best_value
            assert best == want.best_point
            assert trace == want.temperature_trace
