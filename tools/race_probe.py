"""Repeat one C2-shape run several times and print a digest of each trace (determinism probe).

    python tools/race_probe.py N 'QPM_WOLF=planner,QPM_PLAN_CTAS=592' [G] [SEG_CHUNKS]
"""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    os.environ.setdefault("QPM_DEV_KNOBS", "1")  # scheduling knobs are read only with this set
    import torch

    import paper_2511_01255_b200 as q

    n = int(sys.argv[1])
    for kv in filter(None, (sys.argv[2] if len(sys.argv) > 2 else "").split(",")):
        k, v = kv.split("=")
        os.environ[k] = v
    G = int(sys.argv[3]) if len(sys.argv) > 3 else 300
    seg = int(sys.argv[4]) if len(sys.argv) > 4 else None  # fitness segment length (chunks)
    torch.cuda.set_device(0)
    obj = q.make_objective(q.ObjectiveSpec("single_thg", (1404.0,)), q.default_dispersion(), 1.0, 10_000,
                           seg_chunks=seg)
    ref = None
    for r in range(n):
        eng = q.Engine(obj, "hybrid", pop_size=1024, generations=1000, seed=0, de=q.DEParams(), gwo=q.GWOParams(),
                       sch=q.Schedules())
        eng.init()
        eng.step(G, use_graph=os.environ.get("QPM_EAGER", "0") != "1")
        t = eng.trace(0, G + 1)
        h = hashlib.sha1(t.tobytes()).hexdigest()[:12]
        first = ""
        if ref is None:
            ref = t
        elif not (t == ref).all():
            g = int((t != ref).any(axis=1).argmax())
            first = f"first diff at g={g}: {t[g].tolist()} vs {ref[g].tolist()}"
        print(r, h, t[-1][1], first, flush=True)
        del eng


if __name__ == "__main__":
    main()
