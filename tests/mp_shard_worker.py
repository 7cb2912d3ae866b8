"""One rank of a real multi-process sharded run (launched by torchrun from
tests/test_gpu_multiprocess.py; not a test module).

Every rank builds the real CUDA shard engine for its gene columns (all ranks
on cuda:0 -- NCCL cannot place two ranks on one GPU, so the partial slots
travel through host memory over a gloo group, qpm_engine_partials_*), runs the
whole run and saves its trace, population columns and the assembled best
individual to <out>/rank<r>.npz.
"""

import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--algorithm", default="hybrid")
    ap.add_argument("--D", type=int, default=3000)
    ap.add_argument("--NP", type=int, default=48)
    ap.add_argument("--G", type=int, default=25)
    ap.add_argument("--seed", type=int, default=11)
    ap.add_argument("--nwl", type=int, default=1)
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    dist.init_process_group("gloo")
    torch.cuda.set_device(0)
    import paper_2511_01255_b200 as q
    from paper_2511_01255_b200.distributed import HostExchangeShard

    pumps = tuple(float(w) for w in np.linspace(1380.0, 1430.0, args.nwl)) if args.nwl > 1 else (1404.0,)
    spec = q.ObjectiveSpec("multi_thg" if args.nwl > 1 else "single_thg", pumps)
    obj = q.make_objective(spec, q.default_dispersion(), 1.0, args.D, mode="fast")
    gwo = q.GWOParams(a=0.1, a_final=0.01) if args.algorithm == "gwo" else q.GWOParams()
    sh = HostExchangeShard(obj, args.algorithm, pop_size=args.NP, generations=args.G, seed=args.seed,
                           de=q.DEParams(), gwo=gwo, sch=q.Schedules())
    sh.init()
    sh.step(args.G)
    sh.finalize()
    trace = sh.trace()
    best = sh.best()
    genome, fit = sh.engine.population()
    np.savez(os.path.join(args.out, f"rank{sh.rank}.npz"), trace=trace, genome=genome, fit=fit,
             g0=sh.engine.g0, best_genome=best.genome, best_proj=best.projection, best_fit=best.fitness,
             exchanged=sh.exchanged_bytes, pid=os.getpid())
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
