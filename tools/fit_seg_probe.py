"""Fitness launches for several segment lengths in one process (for one ncu launch-list pass).

    python tools/fit_seg_probe.py [seg ...]
The segment length is a problem parameter (make_objective(seg_chunks=...)), so each setting gets its own problem.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import paper_2511_01255_b200 as q

    torch.cuda.set_device(0)
    segs = [int(a) for a in sys.argv[1:]] or [1, 2, 4]
    rows, d = 1024, 10_000
    for sc in segs:
        obj = q.make_objective(q.ObjectiveSpec("single_thg", (1404.0,)), q.default_dispersion(), 1.0, d,
                               seg_chunks=sc)
        W = obj.row_words
        g = torch.Generator(device="cuda").manual_seed(0)
        bits = torch.randint(0, 2**31 - 1, (rows, W), dtype=torch.int32, device="cuda", generator=g)
        bits[:, (d + 31) // 32:] = 0
        out = torch.empty(rows, dtype=torch.float64, device="cuda")
        s = torch.cuda.Stream()
        for _ in range(10):
            obj.evaluate_bits(bits, out, stream=s)
        torch.cuda.synchronize()
        print("seg", sc, "done", float(out[0]))


if __name__ == "__main__":
    main()
