"""Locate the first engine buffer whose contents differ between two identical runs (race probe)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    for kv in filter(None, (sys.argv[1] if len(sys.argv) > 1 else "").split(",")):
        k, v = kv.split("=")
        os.environ[k] = v
    G = int(sys.argv[2]) if len(sys.argv) > 2 else 80
    import numpy as np
    import torch
    import paper_2511_01255_b200 as q
    from paper_2511_01255_b200 import _native
    torch.cuda.set_device(0)
    L = _native.lib()
    L.qpm_engine_debug_hashes.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
    obj = q.make_objective(q.ObjectiveSpec("single_thg", (1404.0,)), q.default_dispersion(), 1.0, 10_000)
    runs = []
    for r in range(3):
        eng = q.Engine(obj, "hybrid", pop_size=1024, generations=1000, seed=0, de=q.DEParams(), gwo=q.GWOParams(),
                       sch=q.Schedules())
        eng.init()
        hs = []
        for g in range(G):
            eng.step(1, use_graph=False)
            out = np.zeros(64, dtype=np.uint64)
            n = ctypes.c_int()
            L.qpm_engine_debug_hashes(eng.handle, out.ctypes.data, 64, ctypes.byref(n))
            hs.append(out[:n.value].copy())
        runs.append(hs)
        del eng
    for r in (1, 2):
        for g in range(G):
            d = np.nonzero(runs[0][g] != runs[r][g])[0]
            if d.size:
                print(f"run {r}: first difference after generation {g + 1}: buffers {d.tolist()}", flush=True)
                break
        else:
            print(f"run {r}: identical through {G} generations", flush=True)


if __name__ == "__main__":
    main()
