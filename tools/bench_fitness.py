"""Microbenchmark of one fitness launch (bit rows resident on the device).

    python tools/bench_fitness.py [--rows 1024] [--d 10000] [--nwl 1] [--iters 200] [--mode fast]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=1024)
    ap.add_argument("--d", type=int, default=10_000)
    ap.add_argument("--nwl", type=int, default=1)
    ap.add_argument("--iters", type=int, default=200)
    ap.add_argument("--mode", default="fast")
    args = ap.parse_args()
    import numpy as np
    import torch

    import paper_2511_01255_b200 as q
    from paper_2511_01255_b200 import _native

    torch.cuda.set_device(0)
    pumps = tuple(float(w) for w in np.linspace(1380.0, 1430.0, args.nwl)) if args.nwl > 1 else (1404.0,)
    spec = q.ObjectiveSpec("multi_thg" if args.nwl > 1 else "single_thg", pumps)
    obj = q.make_objective(spec, q.default_dispersion(), 0.5 if args.nwl > 1 else 1.0, args.d, mode=args.mode)
    W = obj.row_words
    bits = torch.randint(0, 2**31 - 1, (args.rows, W), dtype=torch.int32, device="cuda")
    valid = args.d % 32
    # zero the padding bits
    cols = torch.arange(W * 32, device="cuda").reshape(W, 32)
    mask = (cols < args.d).to(torch.int64)
    weights = (2 ** torch.arange(32, device="cuda", dtype=torch.int64))
    wmask = (mask * weights).sum(1).to(torch.int64)
    bits = (bits.to(torch.int64) & wmask).to(torch.int32)
    out = torch.empty(args.rows, dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream()
    for _ in range(5):
        obj.evaluate_bits(bits, out, stream=s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(args.iters):
        obj.evaluate_bits(bits, out, stream=s)
    e1.record(s)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / args.iters
    evals = args.rows * args.d * args.nwl
    print(f"rows={args.rows} D={args.d} nwl={args.nwl} mode={args.mode} seg={'default'}"
          f" -> {us:.2f} us/launch, {evals / us * 1e-3:.3e} Gevals/s... {evals / (us * 1e-6):.3e} domain-evals/s")
    del valid


if __name__ == "__main__":
    main()
