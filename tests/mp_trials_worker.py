"""One rank of a distributed run_trials (launched by torchrun from
tests/test_trials_dist.py and tests/test_gpu_multiprocess.py; not a test module).

Every rank calls run_trials(..., group=WORLD) and saves the statistics and the
gathered records to <out>/rank<r>.npz.  --fake swaps the device engine for a
seed-determined stand-in so the partition / gather / aggregate host logic runs
on CPU (gloo) without a GPU.
"""

import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


class FakeBest:
    def __init__(self, seed, D):
        r = np.random.default_rng(seed)
        self.fitness = float(r.random())
        self.projection = np.where(r.random(D) < 0.5, -1, 1).astype(np.int8)


class FakeEngine:
    def __init__(self, objective, algorithm, *, seed, **kw):
        self.seed, self.D = seed, objective.dimension

    def init(self):
        pass

    def step(self, n):
        pass

    def finalize(self):
        pass

    def best(self):
        return FakeBest(self.seed, self.D)


class FakeObjective:
    dimension = 16

    def normalized_gains(self, signs):
        return np.array([float(np.mean(signs == 1))])


def fake_run(trials, base_seed, group):
    import torch

    from paper_2511_01255_b200 import trials as T

    saved = T.Engine, torch.cuda.synchronize
    T.Engine, torch.cuda.synchronize = FakeEngine, (lambda *a, **k: None)
    try:
        return T.run_trials(FakeObjective(), "hybrid", trials, base_seed, dimension=16, pop_size=8, generations=5,
                            max_concurrent=3, group=group)
    finally:
        T.Engine, torch.cuda.synchronize = saved


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--fake", action="store_true")
    ap.add_argument("--algorithm", default="hybrid")
    ap.add_argument("--trials", type=int, default=7)
    ap.add_argument("--seed", type=int, default=3)
    ap.add_argument("--D", type=int, default=300)
    ap.add_argument("--NP", type=int, default=24)
    ap.add_argument("--G", type=int, default=30)
    args = ap.parse_args()
    import torch.distributed as dist

    dist.init_process_group("gloo")
    group = dist.group.WORLD
    if args.fake:
        stats, recs = fake_run(args.trials, args.seed, group)
    else:
        import torch

        torch.cuda.set_device(0)
        import paper_2511_01255_b200 as q

        obj = q.make_objective(q.ObjectiveSpec("single_thg", (1404.0,)), q.default_dispersion(), 1.0, args.D)
        stats, recs = q.run_trials(obj, args.algorithm, args.trials, args.seed, dimension=args.D, pop_size=args.NP,
                                   generations=args.G, group=group)
    np.savez(os.path.join(args.out, f"rank{dist.get_rank()}.npz"), pid=os.getpid(),
             trial=[r.trial for r in recs], seed=[r.seed for r in recs],
             final=[r.final_fitness for r in recs], deff=[r.deff_norm for r in recs],
             stats=[stats.trials, stats.average, stats.maximum, stats.minimum, stats.std, stats.mean_deff_norm])
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
