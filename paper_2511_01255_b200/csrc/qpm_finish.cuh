// qpm_finish.cuh -- the stitch of a row's fitness segment partials and the
// objective (|w12 acc + h|, glibc hypot replica, normalisation, multi
// wavelength), shared by k_fit_finish (qpm_fitness.cu) and the engine's fused
// finish + selection kernels (qpm_engine.cu): one definition, so both give
// bit-identical fitness.
#pragma once

#include "qpm_common.cuh"
#include "qpm_internal.cuh"

namespace qpm {

// Segment concatenation: (a1, P1, T1) . (a2, P2, T2) = (a1 + a2 + P1 T2, P1 + P2, T1 + T2).
struct Seg {
    double ar, ai, pr, pi, tr, ti;
};

__device__ __forceinline__ Seg seg_cat(const Seg &x, const Seg &y) {
    Seg z;
    z.ar = (x.ar + y.ar) + fma(x.pr, y.tr, -x.pi * y.ti);
    z.ai = (x.ai + y.ai) + fma(x.pr, y.ti, x.pi * y.tr);
    z.pr = x.pr + y.pr;
    z.pi = x.pi + y.pi;
    z.tr = x.tr + y.tr;
    z.ti = x.ti + y.ti;
    return z;
}

// Column-sharded runs (multi-GPU): rank k scored the global segments
// [floor(k S / world), floor((k+1) S / world)) into its slot of the
// all-gathered partials, laid out [world][n_wl][rows][S_slot][6]; segment s
// lives in rank (world (s+1) - 1) / S.  One GPU: world = 1, S_slot = S.
__device__ __forceinline__ const double *seg_ptr(const double *part, int s, int lam, int64_t r, int64_t rows, int n_wl,
                                                 int S, int world, int S_slot) {
    int rk = 0, loc = s;
    if (world > 1) {
        rk = (world * (s + 1) - 1) / S;
        loc = s - (rk * S) / world;
    }
    return part + ((((int64_t)rk * n_wl + lam) * rows + r) * S_slot + loc) * kPartDoubles;
}

struct FinishArgs {
    const double *part;  // [n_wl][rows][S_slot][6] (one GPU) or [world][n_wl][rows][S_slot][6]
    int S, world, S_slot;
    int64_t rows;
    int n_wl;
    const double2 *w, *h;
    int thg;
    double scale;
    int multi;
    double g0, beta;
    double *gains;  // [rows][n_wl] scratch (multi)
};

// fitness of row r by one warp (every lane must call it; the value is lane 0's):
// lane l stitches the run of segments [l per, (l + 1) per), the 32 runs are
// stitched by a fixed shuffle tree (deterministic), then the objective
__device__ __forceinline__ double finish_row(const FinishArgs &f, int64_t r, int lane) {
    const int S = f.S;
    const int per = (S + 31) / 32;
    const int s0 = lane * per;
    const int s1 = s0 + per < S ? s0 + per : S;
    double gmax = 0.0, gmin = 0.0;
    for (int lam = 0; lam < f.n_wl; ++lam) {
        double ar, ai;
        if (S == 1) {
            const double *p = f.part + ((int64_t)lam * f.rows + r) * kPartDoubles;
            ar = __ldcg(p);  // exact mode: the row's sum, untouched
            ai = __ldcg(p + 1);
        } else {
            Seg acc = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
            for (int s = s0; s < s1; ++s) {
                const double *q = seg_ptr(f.part, s, lam, r, f.rows, f.n_wl, S, f.world, f.S_slot);
                const Seg y = {__ldcg(q), __ldcg(q + 1), __ldcg(q + 2), __ldcg(q + 3), __ldcg(q + 4), __ldcg(q + 5)};
                acc = s == s0 ? y : seg_cat(acc, y);
            }
            for (int off = 1; off < 32; off <<= 1) {
                Seg o;
                o.ar = __shfl_down_sync(0xffffffffu, acc.ar, off);
                o.ai = __shfl_down_sync(0xffffffffu, acc.ai, off);
                o.pr = __shfl_down_sync(0xffffffffu, acc.pr, off);
                o.pi = __shfl_down_sync(0xffffffffu, acc.pi, off);
                o.tr = __shfl_down_sync(0xffffffffu, acc.tr, off);
                o.ti = __shfl_down_sync(0xffffffffu, acc.ti, off);
                const bool has_other = lane + off < 32 && (lane + off) * per < S;
                if ((lane & (2 * off - 1)) == 0 && has_other) acc = seg_cat(acc, o);
            }
            ar = acc.ar;
            ai = acc.ai;
        }
        if (lane != 0) continue;
        const double2 ww = f.w[lam];
        double zr = ww.x * ar - ww.y * ai;
        double zi = ww.x * ai + ww.y * ar;
        if (f.thg) {
            const double2 hh = f.h[lam];
            zr += hh.x;
            zi += hh.y;
        }
        double g = hypot_glibc(zr, zi);
        if (f.scale != 1.0) g /= f.scale;
        if (!f.multi) return g;
        if (lam == 0 || g > gmax) gmax = g;
        if (lam == 0 || g < gmin) gmin = g;
        f.gains[r * f.n_wl + lam] = g;
    }
    if (lane != 0) return 0.0;
    double *dv = f.gains + r * f.n_wl;
    for (int lam = 0; lam < f.n_wl; ++lam) dv[lam] = fabs(f.g0 - dv[lam]);
    double fv = pairwise_sum_seq(dv, f.n_wl);
    fv += f.beta * (gmax - gmin);
    return -fv;
}

FinishArgs finish_args(const Problem *p, const double *part, int S, int world, int S_slot, int64_t rows,
                       double *gains);

}  // namespace qpm
