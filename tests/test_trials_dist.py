"""run_trials over a process group (gloo, world 2 and 3, CPU): rank r runs
trials r, r + W, ...; the records are all-gathered in trial order and every
rank returns the statistics of the single-process call.  The device engine is
replaced by a seed-determined stand-in (tests/mp_trials_worker.py --fake);
tests/test_gpu_multiprocess.py runs the real engine the same way."""

import os
import socket
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def launch_trials(tmp_path, world, *extra):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           os.path.join(ROOT, "tests", "mp_trials_worker.py"), "--out", str(tmp_path), *extra]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    return [dict(np.load(os.path.join(tmp_path, f"rank{r}.npz"))) for r in range(world)]


@pytest.mark.parametrize("world,trials", [(2, 7), (3, 7), (3, 2)])
def test_distributed_trials_equal_single_process(tmp_path, world, trials):
    import mp_trials_worker as W

    stats, recs = W.fake_run(trials, 3, None)
    ranks = launch_trials(tmp_path, world, "--fake", "--trials", str(trials), "--seed", "3")
    for r in ranks:
        assert list(r["trial"]) == list(range(trials))
        assert list(r["seed"]) == [3 + t for t in range(trials)]
        assert list(r["final"]) == [x.final_fitness for x in recs]
        assert list(r["deff"]) == [x.deff_norm for x in recs]
        want = [stats.trials, stats.average, stats.maximum, stats.minimum, stats.std, stats.mean_deff_norm]
        assert list(r["stats"]) == want
