"""Multi-process (world_size 2 and 3, gloo, CPU) tests of the sharded protocol.

The engine's multi-GPU scheme (paper_2511_01255_b200/distributed.py) is:
own-row trials -> fitness -> all-gather candidate fitness -> recompute the
trials other ranks accepted -> select + leaders -> own-row wolves -> fitness
-> all-gather candidate fitness and candidate sign rows -> select + stats.
Here the same protocol is driven with the CPU oracle's operators and real
torch.distributed all-gathers over gloo; every rank must reproduce the
single-process oracle trace bit for bit.  The NCCL-id bootstrap (rank 0
creates, torch.distributed broadcasts) is exercised over gloo too.
"""

import math
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2511_01255_b200 import tables as T
from paper_2511_01255_b200.distributed import shard_rows

MASK = (1 << 64) - 1


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def problem(D):
    t = T.build_tables("thg", 1.0, D, (0.3, 0.7))
    return O.Problem("thg", t.e1[None], t.b[None], np.array([t.w]), np.array([t.hconst]), t.normalization)


def allgather_f64(local: np.ndarray, world: int) -> np.ndarray:
    import torch

    src = torch.from_numpy(np.ascontiguousarray(local))
    out = [torch.empty_like(src) for _ in range(world)]
    dist.all_gather(out, src)
    return np.concatenate([o.numpy() for o in out])


def sharded_hybrid(rank, world, P, NP, D, G, seed):
    """One run_hybrid over `world` gloo ranks with the engine's exchange protocol."""
    s = O.RunSettings()
    lo, hi = shard_rows(NP, world, rank)
    pop = O.init_population(NP, D, s.x_min, s.x_max, seed)
    proj = np.where(pop >= 0.0, 1, -1).astype(np.int8)
    fit = O.evaluate_block(P, proj, threads=1)  # init is replicated
    mean0, std0 = O.mean_std(fit)
    trace = [[0.0, float(fit.max()), mean0, s.f_max, std0]]
    baseline, F, best_prev, window = std0, s.f_max, float(fit.max()), []
    k = s.leader_count
    for g in range(1, G + 1):
        keys = [O.fold_key(seed, g, i) for i in range(NP)]

        def trial(i):
            t, picks, m, jr = O.de_trial(keys[i], pop, i, F, s.cr)
            return t, m

        # DE: own rows, exchange candidate fitness, recompute accepted foreign trials
        own = {i: trial(i) for i in range(lo, hi)}
        cand_own = O.evaluate_block(P, np.stack([np.where(own[i][0] >= 0.0, 1, -1) for i in range(lo, hi)])
                                    .astype(np.int8), threads=1)
        cand = allgather_f64(cand_own, world)
        mcount = {}
        new_pop = pop.copy()
        for i in range(NP):
            if cand[i] > fit[i]:
                t, m = own[i] if lo <= i < hi else trial(i)
                new_pop[i] = t
            mcount[i] = own[i][1] if lo <= i < hi else O.de_trial(keys[i], pop, i, F, s.cr)[2]
        for i in range(NP):
            if cand[i] > fit[i]:
                fit[i] = cand[i]
        pop = new_pop
        proj = np.where(pop >= 0.0, 1, -1).astype(np.int8)
        # leaders and wolves: own rows, exchange fitness and candidate rows
        lead = O.reduce_best(fit, k)
        prog = g / G
        p_dist, p_sl, p_flip = s.p_dist0 * (1.0 - prog), s.p_sl0 * (1.0 - prog), s.p_flip0 * (1.0 - prog)
        early = prog < s.phase_split
        cands = np.zeros((NP, D))
        for i in range(lo, hi):
            if i not in lead:
                cands[i] = O.gwo_discrete(keys[i], mcount[i] + 1 + D, proj[lead], p_dist, p_sl, p_flip, 1.0, early)
        wolf_cand = np.full(hi - lo, -np.inf)
        movers = [i for i in range(lo, hi) if i not in lead]
        if movers:
            vals = O.evaluate_block(P, np.where(cands[movers] >= 0.0, 1, -1).astype(np.int8), threads=1)
            for i, v in zip(movers, vals):
                wolf_cand[i - lo] = v
        cand = allgather_f64(wolf_cand, world)
        rows = allgather_f64(cands[lo:hi].ravel(), world).reshape(NP, D)
        for i in range(NP):
            if i not in lead and cand[i] > fit[i]:
                pop[i] = rows[i]
                fit[i] = cand[i]
        mean, std = O.mean_std(fit)
        mx, mn = float(fit.max()), float(fit.min())
        window.append(mx > best_prev)
        window = window[-s.conv_window:]
        best_prev = mx
        conv = sum(window) / len(window)
        f = s.f_min + (s.f_max - s.f_min) * math.cos(0.5 * math.pi * prog)
        if std < s.theta_low_frac * baseline or conv < s.conv_threshold:
            f *= s.explore_boost
        if std > s.theta_high_frac * baseline or (mx - mn) < s.range_trigger_frac * baseline:
            f *= s.exploit_factor
        f *= 1.0 - s.decay_strength * prog * prog
        F = min(max(f, s.f_min), s.f_max)
        trace.append([float(g), mx, mean, F, std])
    return np.array(trace)


def _worker(rank, world, port, NP, D, G, seed, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        got = sharded_hybrid(rank, world, problem(D), NP, D, G, seed)
        q.put((rank, got))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_protocol_reproduces_single_process(world):
    NP, D, G, seed = 12, 40, 8, 5
    ref, *_ = O.run(problem(D), "hybrid", NP, G, seed)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, NP, D, G, seed, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        assert np.array_equal(results[r], ref), f"rank {r} trace differs from the single-process oracle"


def _id_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2511_01255_b200 import distributed as D

        uid = D.broadcast_unique_id()
        q.put((rank, uid))
    finally:
        dist.destroy_process_group()


def test_nccl_id_bootstrap_over_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_id_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert len(got[0]) == 128 and got[0] == got[1]


def test_shard_rows_partition():
    for NP, world in ((1024, 1), (1024, 8), (8192, 4), (12, 3)):
        spans = [shard_rows(NP, world, r) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == NP
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
        assert len({hi - lo for lo, hi in spans}) == 1
    with pytest.raises(ValueError, match="multiple"):
        shard_rows(10, 3, 0)
    with pytest.raises(ValueError):
        shard_rows(12, 3, 3)
