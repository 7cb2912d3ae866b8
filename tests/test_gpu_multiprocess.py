"""GPU, several processes: the real column-sharded CUDA engine run by separate
processes (torchrun, world 2 and 3, all on cuda:0) that exchange their fitness
partial slots over a gloo group through host memory
(distributed.HostExchangeShard, qpm_engine_partials_*).  Every rank must
reproduce the single-engine run bit for bit: trace, its columns of the
population and the assembled best individual.  This is the sharded protocol
across a real process boundary; the in-graph ncclAllGather transport is
covered by the 1-rank communicator tests (tests/test_gpu_sharded.py), since
NCCL cannot place two ranks on one GPU.  Replaces the reference's in-process
thread pool (/root/reference/pkg/src/qpmdesign/parexec.py:94-119).

Also: the failure-detection path of the NCCL transport (qpm_engine_wait): a
communicator aborted on timeout turns into QpmError, and the engine refuses
further steps.
"""

import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def q():
    import torch

    torch.cuda.set_device(0)
    import paper_2511_01255_b200 as pkg

    return pkg


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def launch(tmp_path, world, **kw):
    args = []
    for k, v in kw.items():
        args += [f"--{k}", str(v)]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           os.path.join(ROOT, "tests", "mp_shard_worker.py"), "--out", str(tmp_path)] + args
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    return [dict(np.load(os.path.join(tmp_path, f"rank{r}.npz"))) for r in range(world)]


@pytest.mark.parametrize("algorithm,world,D,nwl", [("hybrid", 2, 3000, 1), ("de", 2, 3000, 1), ("gwo", 2, 3000, 1),
                                                   ("hybrid", 3, 5000, 1), ("hybrid", 2, 3000, 3)])
def test_processes_match_single_engine(q, tmp_path, algorithm, world, D, nwl):
    NP, G, seed = 48, 25, 11
    ranks = launch(tmp_path, world, algorithm=algorithm, D=D, NP=NP, G=G, seed=seed, nwl=nwl)
    assert len({int(r["pid"]) for r in ranks}) == world  # really separate processes
    pumps = tuple(float(w) for w in np.linspace(1380.0, 1430.0, nwl)) if nwl > 1 else (1404.0,)
    spec = q.ObjectiveSpec("multi_thg" if nwl > 1 else "single_thg", pumps)
    obj = q.make_objective(spec, q.default_dispersion(), 1.0, D, mode="fast")
    gwo = q.GWOParams(a=0.1, a_final=0.01) if algorithm == "gwo" else q.GWOParams()
    single = q.Engine(obj, algorithm, pop_size=NP, generations=G, seed=seed, de=q.DEParams(), gwo=gwo,
                      sch=q.Schedules())
    single.init()
    single.step(G)
    single.finalize()
    want = single.trace()
    g_single, f_single = single.population()
    b = single.best()
    for r in ranks:
        assert np.array_equal(r["trace"], want)
        g0 = int(r["g0"])
        assert np.array_equal(r["genome"], g_single[:, g0:g0 + r["genome"].shape[1]])
        assert np.array_equal(r["fit"], f_single)
        assert float(r["best_fit"]) == b.fitness
        assert np.array_equal(r["best_genome"], b.genome) and np.array_equal(r["best_proj"], b.projection)
        assert int(r["exchanged"]) > 0
    cover = sorted((int(r["g0"]), int(r["g0"]) + r["genome"].shape[1]) for r in ranks)
    assert cover[0][0] == 0 and cover[-1][1] == D and all(a[1] == b_[0] for a, b_ in zip(cover, cover[1:]))


_TIMEOUT_CHILD = r"""
import os, sys
sys.path.insert(0, {root!r})
import torch
torch.cuda.set_device(0)
import paper_2511_01255_b200 as q
from paper_2511_01255_b200._native import QpmError
from paper_2511_01255_b200.distributed import ShardedEngine, nccl_unique_id
obj = q.make_objective(q.ObjectiveSpec("single_thg", (1404.0,)), q.default_dispersion(), 1.0, 20_000)
kw = dict(pop_size=2048, generations=300, seed=1, de=q.DEParams(), gwo=q.GWOParams(), sch=q.Schedules())
eng = ShardedEngine.create(obj, "hybrid", rank=0, world=1, nccl_id=nccl_unique_id(), **kw)
eng.init()
eng.step(5)
eng.wait(60.0)
print("WAIT-OK", flush=True)
eng.step(250)
try:
    eng.wait(0.0)
except QpmError as exc:
    print("TIMEOUT-RAISED", "timed out" in str(exc), flush=True)
try:
    eng.step(1)
except QpmError as exc:
    print("STEP-REFUSED", "collective failed" in str(exc), flush=True)
os._exit(0)  # the aborted communicator's queued work is not waited for
"""


def test_nccl_wait_timeout_aborts_and_refuses():
    """qpm_engine_wait on the collective path (a 1-rank communicator, in a
    child process): completion returns normally; a timeout aborts the
    communicator and raises QpmError; later steps are refused -- a stuck
    collective cannot block every later synchronize."""
    res = subprocess.run([sys.executable, "-c", _TIMEOUT_CHILD.format(root=ROOT)], capture_output=True, text=True,
                         timeout=300, cwd=ROOT)
    out = res.stdout
    assert "WAIT-OK" in out, out + res.stderr[-2000:]
    assert "TIMEOUT-RAISED True" in out, out + res.stderr[-2000:]
    assert "STEP-REFUSED True" in out, out + res.stderr[-2000:]


@pytest.mark.parametrize("algorithm,world", [("hybrid", 2), ("gwo", 3)])
def test_distributed_trials_match_single_process(q, tmp_path, algorithm, world):
    """run_trials(group=WORLD): each process runs its share of the seeds on the
    real engine (all on cuda:0 here; one GPU per rank in production) and every
    rank returns the single-process records and statistics bit for bit."""
    trials, seed, D, NP, G = 7, 3, 300, 24, 30
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           os.path.join(ROOT, "tests", "mp_trials_worker.py"), "--out", str(tmp_path), "--algorithm", algorithm,
           "--trials", str(trials), "--seed", str(seed), "--D", str(D), "--NP", str(NP), "--G", str(G)]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    ranks = [dict(np.load(os.path.join(tmp_path, f"rank{r}.npz"))) for r in range(world)]
    assert len({int(r["pid"]) for r in ranks}) == world
    obj = q.make_objective(q.ObjectiveSpec("single_thg", (1404.0,)), q.default_dispersion(), 1.0, D)
    stats, recs = q.run_trials(obj, algorithm, trials, seed, dimension=D, pop_size=NP, generations=G)
    for r in ranks:
        assert list(r["trial"]) == list(range(trials))
        assert list(r["final"]) == [x.final_fitness for x in recs]
        assert list(r["deff"]) == [x.deff_norm for x in recs]
        assert list(r["stats"]) == [stats.trials, stats.average, stats.maximum, stats.minimum, stats.std,
                                    stats.mean_deff_norm]
