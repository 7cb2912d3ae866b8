"""Per-rank GPU time of the sharded engine at world W, emulated on one GPU.

    python tools/shard_probe.py [--world 8] [--np-per-rank 1024] [--d 10000] [--gens 10]
W shard engines of one run (EmulatedShards protocol); after a warm-up, each
generation's phases of rank 0 are run alone between synchronisations and timed
with CUDA events on its stream.  The NCCL all-gathers are replaced by device
copies (not timed), so the result is the slowest rank's kernel time per
phase.  The exchange is reported as bytes (every rank's pre-stitched
super-block slot, qpm_engine_partials_info) and as modelled NCCL all-gather
time: NCCL_LAT_US + received bytes / NCCL_BW_GBS (defaults 12 us and 600
GB/s, a typical NVLink 5 / NVSwitch all-gather bus bandwidth; not measured
here -- one GPU).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, default=8)
    ap.add_argument("--np-per-rank", type=int, default=1024)
    ap.add_argument("--d", type=int, default=10_000)
    ap.add_argument("--warm", type=int, default=30)
    ap.add_argument("--gens", type=int, default=10)
    ap.add_argument("--np", type=int, default=0, help="total NP (strong scaling); default np-per-rank x world")
    ap.add_argument("--seg-chunks", type=int, default=0)
    ap.add_argument("--t", type=float, default=1.0)
    args = ap.parse_args()
    import numpy as np
    import torch

    import paper_2511_01255_b200 as q
    from paper_2511_01255_b200.distributed import EmulatedShards

    torch.cuda.set_device(0)
    NP = args.np or args.np_per_rank * args.world
    obj = q.make_objective(q.ObjectiveSpec("single_thg", (1404.0,)), q.default_dispersion(), args.t, args.d,
                           seg_chunks=args.seg_chunks or None)
    kw = dict(pop_size=NP, generations=1000, seed=0, de=q.DEParams(), gwo=q.GWOParams(), sch=q.Schedules())
    sh = EmulatedShards(obj, "hybrid", args.world, **kw)
    sh.init()
    sh.step(args.warm)
    engines = sh.engines
    phases = engines[0].phases
    W = len(engines)
    per = np.zeros((W, phases))
    for _ in range(args.gens):
        for ph in range(phases):
            if ph > 0:
                torch.cuda.synchronize()
                for dst in engines:
                    for src in engines:
                        if src is not dst:
                            dst.exchange_from(src, ph)
            for r, e in enumerate(engines):  # each rank's phase alone on the GPU
                torch.cuda.synchronize()
                s = e.stream
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                e.run_phase(ph)
                e1.record(s)
                torch.cuda.synchronize()
                per[r, ph] += e0.elapsed_time(e1) * 1e3
    torch.cuda.synchronize()
    per /= args.gens
    per_phase = per.max(axis=0)  # the slowest rank of each phase sets the pace
    single = q.Engine(obj, "hybrid", **kw)
    single.init()
    single.step(args.warm)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(single.stream)
    single.step(args.gens)
    e1.record(single.stream)
    torch.cuda.synchronize()
    one = e0.elapsed_time(e1) * 1e3 / args.gens
    slot_bytes = engines[0].partials_slot() * 8
    gathered = slot_bytes * W
    lat = float(os.environ.get("NCCL_LAT_US", "12"))
    bw = float(os.environ.get("NCCL_BW_GBS", "600"))
    x_us = lat + (gathered - slot_bytes) / (bw * 1e3)
    n_x = phases - 1
    print(json.dumps({"world": args.world, "NP": NP, "D": args.d, "seg_chunks": obj.seg_chunks,
                      "segments": obj.segments, "super_blocks": obj.super_blocks,
                      "exchange_bytes_per_allgather": gathered, "allgathers_per_gen": n_x,
                      "modelled_allgather_us": round(x_us, 2),
                      "modelled_us_per_gen_with_exchange": round(float(per_phase.sum()) + n_x * x_us, 1),
                      "exchange_model": f"{lat} us + received bytes / {bw} GB/s per all-gather (NCCL_LAT_US, "
                                        f"NCCL_BW_GBS; assumed, not measured)",
                      "columns": [e.Dl for e in engines], "max_rank_us_per_phase": per_phase.round(2).tolist(),
                      "max_rank_us_per_gen": float(per_phase.sum()),
                      "rank_us_per_gen": per.sum(axis=1).round(1).tolist(), "single_gpu_us_per_gen_same_NP": one,
                      "note": "eager phases (no graph, no PDL), exchanges untimed; per phase the slowest rank"}))


if __name__ == "__main__":
    main()
