"""Phase timing of the public run_hybrid path at C2 (where the end-to-end seconds go)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import paper_2511_01255_b200 as q
    from paper_2511_01255_b200.optimizer import DEParams, Engine, GWOParams, Schedules

    torch.cuda.set_device(0)
    t = time.perf_counter()
    obj = q.make_objective(q.ObjectiveSpec("single_thg", (1404.0,)), q.default_dispersion(), 1.0, 10_000)
    torch.cuda.synchronize()
    print(f"objective {1e3 * (time.perf_counter() - t):8.2f} ms")
    G = int(sys.argv[1]) if len(sys.argv) > 1 else 950
    for rep in range(3):
        marks = []
        t0 = time.perf_counter()

        def mark(name):
            torch.cuda.synchronize()
            marks.append((name, time.perf_counter()))

        eng = Engine(obj, "hybrid", pop_size=1024, generations=G, seed=7, de=DEParams(), gwo=GWOParams(),
                     sch=Schedules())
        mark("create")
        eng.init()
        mark("init")
        eng.step(1)
        mark("capture+1")
        eng.step(G - 1)
        mark("steps")
        eng.finalize()
        mark("finalize")
        tr = eng.trace(0, G + 1)
        mark("trace")
        b = eng.best()
        mark("best")
        del eng
        mark("destroy")
        prev = t0
        parts = []
        for n, tt in marks:
            parts.append(f"{n}={1e3 * (tt - prev):.2f}")
            prev = tt
        print(f"rep {rep}: total {1e3 * (prev - t0):8.2f} ms  " + " ".join(parts))
        t1 = time.perf_counter()
        res = q.run_hybrid(obj, dimension=10_000, pop_size=1024, generations=G, seed=7)
        torch.cuda.synchronize()
        print(f"   run_hybrid {1e3 * (time.perf_counter() - t1):8.2f} ms")


if __name__ == "__main__":
    main()
