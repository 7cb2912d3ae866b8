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

// The stitch tree is fixed by the problem alone (D, wavelengths, segment
// length), never by the batch or the number of GPUs, so fitness is a pure
// function of the row bits: the S segments are grouped into nsb = min(8, S)
// contiguous super-blocks, super-block b = segments [sb_lo(b), sb_lo(b+1)),
// sb_lo(b) = floor(b S / nsb); a super-block is stitched sequentially, then
// the nsb super-block partials by a fixed 3-level shuffle tree.
// Multi-GPU (column shards): rank k of W owns super-blocks
// [floor(k nsb / W), floor((k+1) nsb / W)) and the genes under them; it
// pre-stitches its super-blocks (k_prestitch, the same sequential order) and
// only those partials are all-gathered, [W][n_wl][rows][SB_slot][6] --
// NP x nsb x 48 B per wavelength in total, whatever the segment count.
constexpr int kMaxSuperBlocks = 8;
__host__ __device__ __forceinline__ int super_blocks(int S) { return S < kMaxSuperBlocks ? S : kMaxSuperBlocks; }
__host__ __device__ __forceinline__ int sb_lo(int b, int S, int nsb) { return (int)((int64_t)b * S / nsb); }
// first super-block of rank k, and the rank owning super-block b
__host__ __device__ __forceinline__ int sb_first(int k, int nsb, int world) { return (int)((int64_t)k * nsb / world); }
__host__ __device__ __forceinline__ int sb_owner(int b, int nsb, int world) { return (world * (b + 1) - 1) / nsb; }

struct FinishArgs {
    const double *part;  // segment partials [n_wl][rows][S][6], or (pre) super-block partials
                         // [world][n_wl][rows][SB_slot][6]
    int S;               // segments per row (1: one exact sum per row)
    int nsb;             // super-blocks
    int pre;             // part holds pre-stitched super-blocks (multi-GPU)
    int world, SB_slot;
    int64_t rows;
    int n_wl;
    const double2 *w, *h;
    int thg;
    double scale;
    int multi;
    double g0, beta;
    double *gains;  // [rows][n_wl] scratch (multi)
};

__device__ __forceinline__ Seg seg_load(const double *q) {
    return Seg{__ldcg(q), __ldcg(q + 1), __ldcg(q + 2), __ldcg(q + 3), __ldcg(q + 4), __ldcg(q + 5)};
}

// super-block b of row r at wavelength lam from segment partials [n_wl][rows][S_stride][6]
// whose first entry is global segment s_base: sequential stitch (k_prestitch and finish_row)
__device__ __forceinline__ Seg stitch_super_block(const double *part, int b, int lam, int64_t r, int64_t rows,
                                                  int S, int nsb, int S_stride, int s_base) {
    const int s0 = sb_lo(b, S, nsb), s1 = sb_lo(b + 1, S, nsb);
    const double *q = part + (((int64_t)lam * rows + r) * S_stride + (s0 - s_base)) * kPartDoubles;
    Seg acc = seg_load(q);
    for (int s = s0 + 1; s < s1; ++s) acc = seg_cat(acc, seg_load(q + (s - s0) * kPartDoubles));
    return acc;
}

// fitness of row r by one warp (every lane must call it; the value is lane 0's):
// lane b < nsb forms super-block b, the nsb partials are stitched by a fixed
// shuffle tree, then the objective
__device__ __forceinline__ double finish_row(const FinishArgs &f, int64_t r, int lane) {
    const int S = f.S, nsb = f.nsb;
    double gmax = 0.0, gmin = 0.0;
    for (int lam = 0; lam < f.n_wl; ++lam) {
        double ar, ai;
        if (S == 1) {
            const double *p = f.part + ((int64_t)lam * f.rows + r) * kPartDoubles;
            ar = __ldcg(p);  // exact mode: the row's sum, untouched
            ai = __ldcg(p + 1);
        } else {
            Seg acc = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
            if (lane < nsb) {
                if (f.pre) {
                    const int rk = sb_owner(lane, nsb, f.world);
                    const int loc = lane - sb_first(rk, nsb, f.world);
                    acc = seg_load(f.part + ((((int64_t)rk * f.n_wl + lam) * f.rows + r) * f.SB_slot + loc) *
                                                kPartDoubles);
                } else {
                    acc = stitch_super_block(f.part, lane, lam, r, f.rows, S, nsb, S, 0);
                }
            }
#pragma unroll
            for (int off = 1; off < kMaxSuperBlocks; off <<= 1) {
                Seg o;
                o.ar = __shfl_down_sync(0xffffffffu, acc.ar, off);
                o.ai = __shfl_down_sync(0xffffffffu, acc.ai, off);
                o.pr = __shfl_down_sync(0xffffffffu, acc.pr, off);
                o.pi = __shfl_down_sync(0xffffffffu, acc.pi, off);
                o.tr = __shfl_down_sync(0xffffffffu, acc.tr, off);
                o.ti = __shfl_down_sync(0xffffffffu, acc.ti, off);
                if ((lane & (2 * off - 1)) == 0 && lane + off < nsb) acc = seg_cat(acc, o);
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

// one-GPU layout (segment partials), or the all-gathered super-block slots
FinishArgs finish_args(const Problem *p, const double *part, int S, int64_t rows, double *gains);
FinishArgs finish_args_pre(const Problem *p, const double *gpart, int world, int SB_slot, int64_t rows, double *gains);

}  // namespace qpm
