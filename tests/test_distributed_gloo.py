"""Multi-process (world_size 2 and 3, gloo, CPU) tests of the sharded protocol.

The engine's multi-GPU scheme (paper_2511_01255_b200/distributed.py) shards
the genes by columns: every rank runs the per-gene operators (DE trial and
crossover mask, wolf draws and leader vote, init) on its columns of all NP
rows, exchanges per-row fitness information, and runs selection, leaders and
statistics replicated.  Here the same protocol is driven with column-local
restatements of the operators (each pinned to the CPU oracle's full-row
operator below) and real torch.distributed all-gathers over gloo; the
exchange carries the candidates' sign columns and every rank scores full rows
with the oracle (the GPU engine exchanges fitness segment partials instead;
tests/test_gpu_sharded.py pins that path bit-exactly to one GPU).  Every rank
must reproduce the single-process oracle trace bit for bit.  The NCCL-id
bootstrap (rank 0 creates, torch.distributed broadcasts) is exercised over
gloo too.
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
from paper_2511_01255_b200.distributed import shard_columns


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def problem(D):
    t = T.build_tables("thg", 1.0, D, (0.3, 0.7))
    return O.Problem("thg", t.e1[None], t.b[None], np.array([t.w]), np.array([t.hconst]), t.normalization)


def allgather_cols(local: np.ndarray, world: int, D: int, spans) -> np.ndarray:
    """[rows, D] from every rank's [rows, g1 - g0] columns (gloo all-gather, padded to equal size)."""
    import torch

    width = max(g1 - g0 for g0, g1 in spans)
    pad = np.zeros((local.shape[0], width), dtype=local.dtype)
    pad[:, :local.shape[1]] = local
    src = torch.from_numpy(pad)
    out = [torch.empty_like(src) for _ in range(world)]
    dist.all_gather(out, src)
    full = np.empty((local.shape[0], D), dtype=local.dtype)
    for (g0, g1), o in zip(spans, out):
        full[:, g0:g1] = o.numpy()[:, :g1 - g0]
    return full


# column-local operators (stream positions of the global gene index g0 + j)
def trial_cols(key, cols, i, F, cr, picks, m, jr, g0):
    """de_mutate + de_crossover (optimizer.py:229-262) on columns [g0, g0 + cols.shape[1])."""
    r1, r2, r3 = picks
    u = O.uniform_fill(key, m + 1 + g0, cols.shape[1])  # mask positions m+1+j
    take = u <= cr
    if 0 <= jr - g0 < cols.shape[1]:
        take[jr - g0] = True
    return np.where(take, cols[r1] + F * (cols[r2] - cols[r3]), cols[i])


def wolf_cols(key, base, lead_cols, p_dist, p_sl, p_flip, early, g0, D):
    """gwo_discrete_update (optimizer.py:335-376) on columns; rows of the 6 x D block at base + r D + j."""
    k, n = lead_cols.shape
    u = [O.uniform_fill(key, base + r * D + g0, n) for r in range(6)]
    cp = (lead_cols > 0).sum(0)
    p_plus = cp / k
    pick = np.minimum((u[1] * k).astype(np.int64), k - 1)
    leader_state = lead_cols[pick, np.arange(n)]
    random_state = np.where(u[3] < 0.5, 1, -1)
    if early:
        sampled = np.where(u[4] < p_plus, 1, -1)
        basev = np.where(u[2] < p_dist, random_state, sampled)
    else:
        maj = np.where(2 * cp > k, 1, np.where(2 * cp < k, -1, random_state))
        basev = np.where(u[5] < p_flip, -maj, maj)
    return np.where(u[0] < p_sl, leader_state, basev).astype(np.float64)


def sharded_hybrid(rank, world, P, NP, D, G, seed):
    """One run_hybrid over `world` gloo ranks, genes sharded by columns."""
    s = O.RunSettings()
    spans = [shard_columns(D, world, r) for r in range(world)]
    g0, g1 = spans[rank]
    full0 = O.init_population(NP, D, s.x_min, s.x_max, seed)
    pop = full0[:, g0:g1].copy()  # this rank's columns (init positions are per gene)
    proj = np.where(pop >= 0.0, 1, -1).astype(np.int8)
    fit = O.evaluate_block(P, allgather_cols(proj, world, D, spans), threads=1)
    mean0, std0 = O.mean_std(fit)
    trace = [[0.0, float(fit.max()), mean0, s.f_max, std0]]
    baseline, F, best_prev, window = std0, s.f_max, float(fit.max()), []
    k = s.leader_count
    zeros = np.zeros((NP, D))
    for g in range(1, G + 1):
        keys = [O.fold_key(seed, g, i) for i in range(NP)]
        draws = [O.de_trial(keys[i], zeros, i, F, s.cr)[1:] for i in range(NP)]  # (picks, m, jr): key-only
        trials = np.stack([trial_cols(keys[i], pop, i, F, s.cr, *draws[i], g0) for i in range(NP)])
        tproj = allgather_cols(np.where(trials >= 0.0, 1, -1).astype(np.int8), world, D, spans)
        cand = O.evaluate_block(P, tproj, threads=1)
        acc = cand > fit
        pop[acc] = trials[acc]
        fit[acc] = cand[acc]
        proj = np.where(pop >= 0.0, 1, -1).astype(np.int8)
        lead = O.reduce_best(fit, k)
        prog = g / G
        p_dist, p_sl, p_flip = s.p_dist0 * (1.0 - prog), s.p_sl0 * (1.0 - prog), s.p_flip0 * (1.0 - prog)
        early = prog < s.phase_split
        movers = [i for i in range(NP) if i not in lead]
        cands = np.zeros_like(pop)
        for i in movers:
            cands[i] = wolf_cols(keys[i], draws[i][1] + 1 + D, proj[lead], p_dist, p_sl, p_flip, early, g0, D)
        cproj = allgather_cols(np.where(cands >= 0.0, 1, -1).astype(np.int8), world, D, spans)
        vals = O.evaluate_block(P, cproj[movers], threads=1)
        for i, v in zip(movers, vals):
            if v > fit[i]:
                pop[i] = cands[i]
                fit[i] = v
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


def test_column_operators_match_the_oracle():
    """The column-local restatements used by the protocol equal the oracle's
    full-row operators on every column split."""
    NP, D, seed = 9, 1300, 5
    pop = O.init_population(NP, D, -1.0, 1.0, seed)
    leaders = np.where(pop[:4] >= 0.0, 1, -1).astype(np.int8)
    for world in (1, 2, 3):
        for i in range(NP):
            key = O.fold_key(seed, 3, i)
            full, picks, m, jr = O.de_trial(key, pop, i, 0.07, 0.9)
            for early in (True, False):
                wfull = O.gwo_discrete(key, m + 1 + D, leaders, 0.3, 0.2, 0.25, 1.0, early)
                for r in range(world):
                    g0, g1 = shard_columns(D, world, r)
                    t = trial_cols(key, pop[:, g0:g1], i, 0.07, 0.9, picks, m, jr, g0)
                    assert np.array_equal(t, full[g0:g1])
                    w = wolf_cols(key, m + 1 + D, leaders[:, g0:g1], 0.3, 0.2, 0.25, early, g0, D)
                    assert np.array_equal(w, wfull[g0:g1])


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
    NP, D, G, seed = 12, 1300, 8, 5  # 3 fitness segments: 2 and 3 ranks get whole segments
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


def test_shard_columns_partition():
    for D, world in ((10_000, 1), (10_000, 8), (100_000, 8), (1300, 3), (5000, 4)):
        spans = [shard_columns(D, world, r) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == D
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
        assert all(g0 % 128 == 0 and g1 > g0 for g0, g1 in spans)  # whole segments (2 or 3 chunks)
        widths = [g1 - g0 for g0, g1 in spans]
        assert max(widths[:-1] or [0]) - min(widths[:-1] or [0]) <= 384
    assert [shard_columns(10_000, 8, r, seg_chunks=2)[1] - shard_columns(10_000, 8, r, seg_chunks=2)[0]
            for r in range(7)] == [1280] * 7
    with pytest.raises(ValueError, match="segments"):
        shard_columns(40, 2, 0)
    with pytest.raises(ValueError):
        shard_columns(5000, 3, 3)
