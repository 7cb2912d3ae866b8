"""One fitness launch timed inside a CUDA graph of 50 launches (no CPU launch overhead)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch

    import paper_2511_01255_b200 as q

    torch.cuda.set_device(0)
    rows = int(os.environ.get("ROWS", "1024"))
    d = int(os.environ.get("DOM", "10000"))
    nwl = int(os.environ.get("NWL", "1"))
    pumps = tuple(float(w) for w in np.linspace(1380.0, 1430.0, nwl)) if nwl > 1 else (1404.0,)
    spec = q.ObjectiveSpec("multi_thg" if nwl > 1 else "single_thg", pumps)
    obj = q.make_objective(spec, q.default_dispersion(), 0.5 if nwl > 1 else 1.0, d)
    W = obj.row_words
    g = torch.Generator(device="cuda").manual_seed(0)
    bits = torch.randint(0, 2**31 - 1, (rows, W), dtype=torch.int32, device="cuda", generator=g)
    bits[:, (d + 31) // 32:] = 0
    if d % 32:
        bits[:, d // 32] &= (1 << (d % 32)) - 1
    out = torch.empty(rows, dtype=torch.float64, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            obj.evaluate_bits(bits, out, stream=s)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        for _ in range(50):
            obj.evaluate_bits(bits, out, stream=s)
    graph.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        graph.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / 500
    evals = rows * d * nwl
    print(f"rows={rows} D={d} nwl={nwl} seg={'default'}: {us:.2f} us/launch "
          f"(fast+finish), {evals / (us * 1e-6):.3e} domain-evals/s, "
          f"{evals * 10 / (us * 1e-6) / 1e12:.2f} TFLOP/s algorithmic")


if __name__ == "__main__":
    main()
