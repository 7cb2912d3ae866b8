"""Two identical runs, generation 1 eager: which individuals differ and how."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    os.environ["QPM_WOLF"] = "planner"
    import numpy as np
    import torch
    import paper_2511_01255_b200 as q
    from paper_2511_01255_b200 import _native
    torch.cuda.set_device(0)
    L = _native.lib()
    L.qpm_engine_debug_read.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t]
    obj = q.make_objective(q.ObjectiveSpec("single_thg", (1404.0,)), q.default_dispersion(), 1.0, 10_000)
    NP, W = 1024, obj.row_words
    names = {6: ("slot_of", np.int32, NP), 7: ("spare_of", np.int32, NP), 9: ("fit", np.float64, NP),
             10: ("cand", np.float64, NP), 2: ("slot_bin", np.uint8, 2 * NP), 15: ("picks", np.int32, 8 * NP),
             14: ("keys", np.uint64, 2 * NP), 8: ("jrand", np.int32, 2 * NP), 18: ("st", np.uint8, 512)}
    GEN = int(os.environ.get("GEN", "100"))

    def snap(eng):
        d = {}
        for idx, (nm, dt, n) in names.items():
            a = np.zeros(n, dtype=dt)
            L.qpm_engine_debug_read(eng.handle, idx, a.ctypes.data, a.nbytes)
            d[nm] = a
        bits = np.zeros(2 * NP * W, dtype=np.uint32)
        L.qpm_engine_debug_read(eng.handle, 1, bits.ctypes.data, bits.nbytes)
        d["bits"] = bits.reshape(2 * NP, W)
        return d

    ref = []
    for r in range(6):
        eng = q.Engine(obj, "hybrid", pop_size=NP, generations=1000, seed=0, de=q.DEParams(), gwo=q.GWOParams(),
                       sch=q.Schedules())
        eng.init()
        for g in range(GEN):
            eng.step(1, use_graph=False)
            d = snap(eng)
            if r == 0:
                ref.append(d)
                continue
            a, b = ref[g], d
            diffs = {k: np.nonzero(a[k] != b[k])[0] for k in a if k != "bits"}
            diffs = {k: v for k, v in diffs.items() if v.size}
            bd = np.nonzero((a["bits"] != b["bits"]).any(axis=1))[0]
            if diffs or bd.size:
                print(f"run {r} gen {g + 1}:", {k: v[:8].tolist() for k, v in diffs.items()}, "bits slots",
                      bd[:8].tolist(), flush=True)
                for ii in diffs.get("fit", np.array([], int))[:3]:
                    print("   i", ii, "fit", a["fit"][ii], b["fit"][ii], "cand", a["cand"][ii], b["cand"][ii],
                          "slot", a["slot_of"][ii], b["slot_of"][ii], "spare", a["spare_of"][ii], b["spare_of"][ii],
                          flush=True)
                for s in bd[:4]:
                    print("   slot", s, "bin", a["slot_bin"][s], b["slot_bin"][s], "words differ",
                          np.nonzero(a["bits"][s] != b["bits"][s])[0][:10].tolist(),
                          "owner(a)", np.nonzero((a["slot_of"] == s) | (a["spare_of"] == s))[0].tolist(),
                          "owner(b)", np.nonzero((b["slot_of"] == s) | (b["spare_of"] == s))[0].tolist(), flush=True)
                break
        else:
            if r:
                print(f"run {r}: same for {GEN} generations", flush=True)
        del eng
    return


if __name__ == "__main__":
    main()
