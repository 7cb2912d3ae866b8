"""Race probe: per-stage buffer hashes of eager runs, first (generation, stage, buffer) that differs."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
NAMES = ["genome", "bits", "slot_bin", "planes", "cbits", "gthr", "slot_of", "spare_of", "jrand", "fit", "cand",
         "scratch", "tree_i", "tree_v", "keys", "picks", "sched", "trace", "st", "best_genome", "best_bits"]


def main():
    os.environ["QPM_WOLF"] = "planner"
    os.environ["QPM_DBG_STAGEHASH"] = "1"
    G = int(sys.argv[1]) if len(sys.argv) > 1 else 100
    R = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    import numpy as np
    import torch
    import paper_2511_01255_b200 as q
    from paper_2511_01255_b200 import _native
    torch.cuda.set_device(0)
    L = _native.lib()
    L.qpm_debug_stage_log.restype = ctypes.c_int64
    L.qpm_debug_stage_log.argtypes = [ctypes.c_void_p, ctypes.c_int64]
    L.qpm_debug_stage_name.restype = ctypes.c_char_p
    L.qpm_debug_stage_name.argtypes = [ctypes.c_int64]
    obj = q.make_objective(q.ObjectiveSpec("single_thg", (1404.0,)), q.default_dispersion(), 1.0, 10_000)
    logs = []
    for r in range(R):
        L.qpm_debug_stage_reset()
        eng = q.Engine(obj, "hybrid", pop_size=1024, generations=1000, seed=0, de=q.DEParams(), gwo=q.GWOParams(),
                       sch=q.Schedules())
        eng.init()
        eng.step(G, use_graph=False)
        torch.cuda.synchronize()
        names = []
        k = 0
        buf = np.zeros(50_000_000, dtype=np.uint64)
        n = L.qpm_debug_stage_log(buf.ctypes.data, buf.size)
        recs = np.split(buf[:n], np.nonzero(buf[:n] == np.uint64(2**64 - 1))[0] + 1)[:-1]
        while True:
            nm = L.qpm_debug_stage_name(k).decode()
            if not nm:
                break
            names.append(nm)
            k += 1
        logs.append((names, [x[:-1] for x in recs]))
        del eng
    names0, recs0 = logs[0]
    per_gen = len(recs0) // G if G else 0
    for r in range(1, R):
        names, recs = logs[r]
        for k, (a, b) in enumerate(zip(recs0, recs)):
            d = np.nonzero(a != b)[0]
            d = [NAMES[x] if x < len(NAMES) else f"buf{x}" for x in d if x < len(NAMES) + 1]
            d = [x for x in d if x not in ("scratch", "tree_v", "cbits") and not (x == "cand" and k < 4)]
            if d:
                print(f"run {r}: first difference before stage '{names0[k]}' (record {k}, generation ~{k // max(per_gen, 1) + 1}): {d}",
                      flush=True)
                if k > 0:
                    print(f"        previous stage: '{names0[k - 1]}'", flush=True)
                break
        else:
            print(f"run {r}: identical over {len(recs)} records", flush=True)


if __name__ == "__main__":
    main()
