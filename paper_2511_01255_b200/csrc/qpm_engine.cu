// qpm_engine.cu -- device-resident HWSDA generation loop (run_hybrid /
// run_de / run_gwo, optimizer.py:400-592) on one B200, or on one column
// shard of a multi-GPU run.
//
// HBM layout (one engine; D, W, Dp are this engine's genes):
//   genome  f64 [2 NP][Dp]   slot pool; individual i lives in slot_of[i], its
//                            trial / candidate goes to spare_of[i] and
//                            acceptance swaps the two ids (no row copies)
//   bits    u32 [2 NP][W]    sign bits of each slot (bit 1 <=> gene < 0)
//   cbits   u32 [NP][W]      the generation's candidate sign rows, dense by
//                            individual (what the fitness scans)
//   slot_bin u8 [2 NP]       1 = the slot holds a wolf candidate whose genome is
//                            exactly +/-1 (optimizer.py:376): its f64 row is
//                            never written, readers expand the bits instead
//   planes  u32 [2][NP][W][4] per-gene wolf draw outcomes as bit-planes
//   fit, cand f64 [NP]; keys u64 [2][NP]; picks int4 [2][NP] (r1, r2, r3, m)
//   sched   f64 [G+1][8]     per-generation scalars, host-computed
//   trace   f64 [G+1][5]     (g, best, mean, F|a, pop_std)
//   state   EngineState      g, F, window, leaders, best-ever bookkeeping
//   gpart   f64 [W][n_wl][NP][SB_slot][6]  all-gathered fitness super-block
//                            partials (multi-GPU)
// Dp = W * 32 with W a multiple of 4, so rows start on 512-byte boundaries.
//
// One hybrid generation (ten per CUDA graph, everything reading g and F from
// device memory):
//   k_plan_rows     (side stream, one generation ahead) keys + DE indices
//   k_de_trial_tma  crossover mask, trial genome + bits, and the first two
//                   wolf draws of every gene as bit-planes, the source rows
//                   staged by TMA bulk copies (integer-issue bound, HBM
//                   traffic in its shadow); k_de_trial_rows for short rows
//                   (column shards), k_de_trial with global loads (QPM_DE_TMA=0)
//   k_fit_fast      segmented quad-table scan
//   k_finish_select<0>  stitch + greedy selection; the last CTA: top-k leaders
//   k_gwo_apply     leader vote per gene from the planes (+ the third draw
//                   where the outcome depends on it) -> candidate bits
//   k_fit_fast
//   k_finish_select<1>  stitch + wolf selection; the last CTA: np.max/mean/std
//                   replica, window, F update, trace row
// (NP > 2048: k_fit_finish + k_select_topk / k_select_stats instead of the
// fused finish/selection kernels.)  Multi-GPU (column shards): each rank
// pre-stitches its super-blocks (k_prestitch); the partials are all-gathered
// (NCCL, in the graph) and every rank finishes all rows.
// Decisions reproduce the reference bit-for-bit given the same fitness:
//   - stream positions follow SURVEY.md Appendix A (de_mutate rejection
//     draws 0..m-1, j_rand at m, mask m+1..m+D, wolf block from m+1+D), with
//     the global gene index on a shard;
//   - DE arithmetic x_r1 + F (x_r2 - x_r3) is unfused (-fmad=false);
//   - u < p comparisons are exact integer compares on the 53-bit mantissa;
//   - np.mean / np.std use a replica of numpy's pairwise summation.
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "qpm_common.cuh"
#include "qpm_internal.cuh"
#include "qpm_finish.cuh"

namespace qpm {

constexpr int kMaxLeaders = 8;
constexpr int kMaxWindow = 256;
constexpr int kRowThreads = 256;    // threads per row-block in the elementwise kernels
constexpr int kGenesPerThread = 4;  // genes per thread (strided by kRowThreads)
constexpr int kGenesPerBlock = kRowThreads * kGenesPerThread;
constexpr int kCtaThreads = 1024;   // single-CTA select / top-k / stats kernels
#ifndef QPM_DE_CHUNK
#define QPM_DE_CHUNK 4096
#endif
constexpr int kDeChunk = QPM_DE_CHUNK;  // genes per DE-trial CTA (multiple of 1024)
#ifndef QPM_APPLY_THREADS
#define QPM_APPLY_THREADS 128
#endif
constexpr int kApplyThreads = QPM_APPLY_THREADS;  // k_gwo_apply: 32-gene words per CTA
#ifndef QPM_DE_MINB
#define QPM_DE_MINB 4  // k_de_trial CTAs per SM the register budget is sized for
#endif      // genes per DE-trial CTA (amortizes the per-row setup)
constexpr int64_t kStatsSmemMaxNP = 12288;  // 2 x NP doubles of dynamic smem (<= 192 KB)

// ncclUniqueId layout (NCCL_UNIQUE_ID_BYTES = 128, nccl.h)
struct ncclUniqueIdPod {
    char internal[128];
};

struct EngineState {
    int64_t g;       // generation computed next (0 before init)
    int64_t g_plan;  // generation the planner draws next
    double F;
    double best_prev;
    double baseline_std;
    double best_fit;  // run_gwo best-ever fitness
    int32_t best_idx;
    int32_t best_flag;
    int32_t win_len;
    int32_t pad0;
    int32_t leaders[kMaxLeaders];
    uint64_t thr_plus[kMaxLeaders + 1];  // u_plus < p_plus(count) thresholds, nondecreasing
    uint8_t win[kMaxWindow];
};

// u < p as a compare on the raw 64-bit mix:  (mix >> 11) < T  <=>
// mix <= ((T - 1) << 11 | 0x7ff) for 1 <= T <= 2^53; T = 0 never passes.
struct Thr {
    uint64_t le;
    uint32_t never;
};
__host__ __device__ __forceinline__ Thr make_thr(uint64_t T) {
    Thr t;
    t.never = T == 0;
    if (T >= kTwo53)
        t.le = ~0ULL;  // p >= 1: every draw passes
    else
        t.le = T == 0 ? 0 : (((T - 1) << 11) | 0x7ffULL);
    return t;
}
__device__ __forceinline__ bool passes(const Thr &t, uint64_t mix) { return !t.never && mix <= t.le; }

struct RunConsts {
    int algorithm;
    // D, Dp, W: this engine's genes (a column shard [g0, g0 + D) of the run's
    // Dg genes on a multi-GPU run; g0 = 0, D = Dg on one GPU).  Stream
    // positions always use the global gene index g0 + j and Dg.
    int64_t NP, D, Dp, W, G;
    int64_t Dg, g0;
    uint64_t seed;
    double f_max, f_min;
    uint64_t cr_thr;
    double x_lo, x_span;
    int k;  // leader count (hybrid) / 3 (gwo)
    int divide;
    double theta_low_frac, theta_high_frac, range_trigger_frac;
    double explore_boost, exploit_factor, conv_threshold;
    int conv_window;
    int adaptive;
    double gwo_a0;
    // numpy pairwise-sum tree of an NP-vector: leaves, then internal nodes by height
    int32_t n_leaf, n_levels;
    Thr thr_cr;      // u <= CR (de_crossover)
    int plus_dyadic; // K = 4 and p_plus(c) = c/4 exactly: plus level = 1 + floor(4u)
    int plus_ends;   // p_plus(0) = 0 and p_plus(K) = 1 (discreteness 1)
    uint32_t m4, m32, m2;  // = 4, 32, 2: runtime constants (see xs_fma)
    Thr thr_plus[5]; // u_plus < p_plus(count), count = 0..K (hybrid K <= 4)
};

// pairwise-sum tree (host-built, see build_tree): leaf l covers
// [leaf_off[l], leaf_off[l+1]); internal node t (id n_leaf + t) adds nodes
// kid[2t] + kid[2t+1]; level h holds internal nodes [lvl[h], lvl[h+1]).
struct SumTree {
    const int32_t *leaf_off;
    const int32_t *kid;
    const int32_t *lvl;
    double *val;  // [2 n_leaf - 1]
};
// The same tree by value (leaf_off, kid, lvl concatenated) when it fits: a
// kernel parameter sits in the constant bank at launch, so staging it costs no
// global round trip on the critical path (NP <= 8192 -> at most 64 leaves)
#ifndef QPM_TREE_INLINE
#define QPM_TREE_INLINE 1
#endif
constexpr int kTreeInline = 256;
struct SumTreeInline {
    int32_t n;  // 0: use the global copy
    int32_t v[kTreeInline];
};

// ---------------------------------------------------------------- helpers
// draw at counter position p1 = pos + 1 (< 2^32): mix(key + p1 * GOLD).  The
// 32 x 64 product is one IMAD.WIDE.U32 (key as addend) plus one IMAD on the
// FMA pipe; the ALU pipe, which the xorshifts saturate, is left alone.
__device__ __forceinline__ uint64_t mix_at(uint64_t key, uint32_t p1) { return mix64(key + (uint64_t)p1 * kGold); }

// per-generation wolf thresholds (host-built from the schedule table)
struct GenThr {
    Thr sl, dist, flip;
    uint32_t early;
    uint32_t pad;
};

// a genome row that is either f64 or, for wolf candidates, +/-1 bits (one
// pointer and a flag: the trial kernel keeps four of these in registers)
struct RowRef {
    const void *p;
    uint32_t bin;
    __device__ __forceinline__ const double *f() const { return static_cast<const double *>(p); }
    __device__ __forceinline__ const uint32_t *b() const { return static_cast<const uint32_t *>(p); }
    __device__ __forceinline__ double at(int j) const {
        if (!bin) return f()[j];
        return ((b()[j >> 5] >> (j & 31)) & 1u) ? -1.0 : 1.0;
    }
};

__device__ __forceinline__ RowRef row_ref(const RunConsts &c, int64_t slot, const uint8_t *slot_bin,
                                          const double *genome, const uint32_t *bits) {
    RowRef r;
    r.bin = slot_bin[slot] ? 1u : 0u;
    r.p = r.bin ? static_cast<const void *>(bits + slot * c.W) : static_cast<const void *>(genome + slot * c.Dp);
    return r;
}

// the same from a slot tag (slot | bin << 31)
constexpr uint32_t kBinTag = 0x80000000u;
#ifndef QPM_SLOT_TAG
#define QPM_SLOT_TAG 1
#endif
__device__ __forceinline__ RowRef row_ref_tag(const RunConsts &c, uint32_t tag, const double *genome,
                                              const uint32_t *bits) {
    const int64_t slot = (int64_t)(tag & ~kBinTag);
    RowRef r;
    r.bin = (tag & kBinTag) ? 1u : 0u;
    r.p = r.bin ? static_cast<const void *>(bits + slot * c.W) : static_cast<const void *>(genome + slot * c.Dp);
    return r;
}

// de_mutate index draws (optimizer.py:229-247) and j_rand (optimizer.py:258)
__device__ void de_row_draws(const RunConsts &c, uint64_t key, int64_t i, int4 &pk, int32_t &jr) {
    int64_t r[3];
    int n = 0;
    uint64_t m = 0;
    while (n < 3) {
        const int64_t cand = randint(key, m, c.NP);
        ++m;
        bool dup = cand == i;
        for (int t = 0; t < n; ++t) dup |= cand == r[t];
        if (!dup) r[n++] = cand;
    }
    pk = make_int4((int)r[0], (int)r[1], (int)r[2], (int)m);
    jr = (int32_t)randint(key, m, c.Dg);
}


// ---------------------------------------------------------------- wolf planes
// gwo_discrete_update (optimizer.py:335-376) needs, per gene, the outcome of
// at most three draws of the 6 x D block:
//   row 0 social;  row 1 pick (social) | 2 disturb (early) | 5 flip (late);
//   row 3 state | 4 plus (early, not disturbed).
// Since social and non-social genes use disjoint outcomes, they share
// bit-planes (one ballot each per 32-gene word):
//   P0 social
//   P1 social ? pick bit 0 : disturbed (early) | flipped (late)
//   P2 social ? pick bit 1 : state (+1)       -- early & !disturbed: L bit 0
//   P3, P4 (early, !social, !disturbed) L bits 1, 2, with the plus level
//      L = #{c <= K : u_plus >= p_plus(c)}  (p_plus is nondecreasing in c, so
//      u_plus < p_plus(count) <=> count >= L)
// so a late generation writes 3 planes and an early one 5.  The leader vote
// is then evaluated 32 genes at a time with bit-sliced logic.
#ifndef QPM_PLANES
#define QPM_PLANES 4
#endif
// stored plane slots per 32-gene word: P0..P2 (P3, P4 live in k_gwo_apply's
// registers only), one 16-byte store / load per word
constexpr int kPlanes = QPM_PLANES;

// bit-sliced leader vote of one 32-gene word.  ld[t]: leader t's sign bits
// (1 = -1); pl: the word's planes.  Returns the candidate's sign bits.
template <int K>
__device__ __forceinline__ uint32_t wolf_word(const uint32_t *ld, const uint32_t *pl, bool early) {
    // count of +1 leaders per gene, as bits s2 s1 s0
    const uint32_t z0 = ~ld[0], z1 = ~ld[1], z2 = ~ld[2];
    uint32_t s0 = z0 ^ z1 ^ z2;
    uint32_t s1 = (z0 & z1) | (z0 & z2) | (z1 & z2);
    uint32_t s2 = 0;
    if (K == 4) {
        const uint32_t z3 = ~ld[3];
        const uint32_t cy = s0 & z3;
        s0 ^= z3;
        s2 = s1 & cy;
        s1 ^= cy;
    }
    const uint32_t soc = pl[0], a = pl[1], bb = pl[2];
    uint32_t plus;
    if (early) {
        // count >= L (three-bit unsigned compare), L = (P4 P3 P2)
        const uint32_t l0 = bb, l1 = pl[3], l2 = pl[4];
        const uint32_t ge0 = s0 | ~l0;
        const uint32_t ge1 = (s1 & ~l1) | (~(s1 ^ l1) & ge0);
        const uint32_t ge2 = (s2 & ~l2) | (~(s2 ^ l2) & ge1);
        plus = (a & bb) | (~a & ge2);  // disturbed: state, else sampled
    } else {
        uint32_t maj;
        if (K == 4)
            maj = s2 | (s1 & s0) | (s1 & ~s0 & ~s2 & bb);  // >= 3 of 4, or a 2-2 tie broken by state
        else
            maj = s1;  // >= 2 of 3
        plus = maj ^ a;
    }
    const uint32_t l3 = K == 4 ? ld[3] : ld[0];
    const uint32_t lp = (bb & ((a & l3) | (~a & ld[2]))) | (~bb & ((a & ld[1]) | (~a & ld[0])));
    return (soc & lp) | (~soc & ~plus);
}

// ---------------------------------------------------------------- planner
// Everything random in generation g depends only on (seed, g, i, position):
// the planner draws generation g+1's per-row keys and DE indices (rejection
// sampling) on a low-priority side stream while generation g's dependent
// chain runs on the main stream (buffers alternate by g & 1).  The per-gene
// draws (crossover mask, wolf planes) are made inside k_de_trial, whose HBM
// stream leaves most issue slots free.
//
// Draw arithmetic is trimmed to what each decision needs: splitmix64's last
// step z ^= z >> 31 leaves bits 63..33 untouched, so top-bit decisions (state,
// pick, dyadic plus level) read the high word of the second product only,
// and u < p compares decide on the high word, falling back to the full
// 64-bit value only when the high words tie (probability 2^-32).
struct PlanArgs {
    EngineState *st;
    const GenThr *gthr;
    int64_t row_lo, n_rows;  // this rank's rows
    uint64_t *keys;    // [2][NP]
    int4 *picks;       // [2][NP]  r1, r2, r3, m
    int32_t *jrand;    // [2][NP]
    uint32_t *planes;  // [2][NP][W][kPlanes]
};

// z ^= z >> s with the shifts done as multiplies on the FMA pipe (the ALU
// pipe is the binding one in the draw-heavy kernels): m = 2^(32-s) is a
// runtime value so ptxas cannot turn the multiplies back into shifts.
__device__ __forceinline__ uint64_t xs_fma(uint64_t z, uint32_t m) {
    const uint32_t lo = (uint32_t)z, hi = (uint32_t)(z >> 32);
    const uint32_t nlo = lo ^ __umulhi(lo, m) ^ (hi * m);
    const uint32_t nhi = hi ^ __umulhi(hi, m);
    return ((uint64_t)nhi << 32) | nlo;
}
// z ^= z >> s, pipe placement by MODE.  ncu (C2 late generation): IMAD.HI and
// IMAD.WIDE occupy the FMA-heavy pipe twice as long as a plain IMAD, and
// with every xorshift there (MODE 2) FMA-heavy was the busiest pipe (61 % of
// elapsed vs ALU 41 %).  MODE 0: all ALU (two SHF, two LOP3); MODE 1: low
// word by a funnel shift on the ALU, high word by IMAD.HI; MODE 2: xs_fma.
#ifndef QPM_XS30
#define QPM_XS30 0
#endif
#ifndef QPM_XS27
#define QPM_XS27 0
#endif
template <int MODE>
__device__ __forceinline__ uint64_t xs_mode(uint64_t z, int s, uint32_t m) {
    if (MODE == 0) return z ^ (z >> s);
    if (MODE == 2) return xs_fma(z, m);
    const uint32_t lo = (uint32_t)z, hi = (uint32_t)(z >> 32);
    const uint32_t nlo = lo ^ __funnelshift_r(lo, hi, s);
    const uint32_t nhi = hi ^ __umulhi(hi, m);
    return ((uint64_t)nhi << 32) | nlo;
}
// splitmix64 up to (excluding) the last multiply, from the counter state
// z = key + (pos + 1) * GOLD
__device__ __forceinline__ uint64_t mix_pre2z(uint64_t z, const RunConsts &c) {
    z = xs_mode<QPM_XS30>(z, 30, c.m4) * kMix1;  // z ^= z >> 30
    return xs_mode<QPM_XS27>(z, 27, c.m32);      // z ^= z >> 27
}
// the same at position p1 = pos + 1
__device__ __forceinline__ uint64_t mix_pre2(uint64_t key, uint32_t p1, const RunConsts &c) {
    return mix_pre2z(key + (uint64_t)p1 * kGold, c);
}
__device__ __forceinline__ uint32_t mix_hi2(uint64_t x) {  // high word of x * kMix2
    const uint32_t lo = (uint32_t)x, hi = (uint32_t)(x >> 32);
    return __umulhi(lo, (uint32_t)kMix2) + lo * (uint32_t)(kMix2 >> 32) + hi * (uint32_t)kMix2;
}
// u < p for the draw whose pre-product state is x and product high word h
__device__ __forceinline__ bool passes_hi(const Thr &t, uint64_t x, uint32_t h) {
    const uint32_t ho = h ^ (h >> 31);
    const uint32_t hl = (uint32_t)(t.le >> 32);
    bool r = ho < hl;
    if (ho == hl) {
        const uint64_t z = x * kMix2;
        r = (z ^ (z >> 31)) <= t.le;
    }
    return !t.never && r;
}

// branch-free variant: decides on the high word and flags a tie (probability
// 2^-32 per compare) for the caller's warp-level exact fallback, so two
// independent draws interleave without per-compare branches
// (a never-passing threshold has le = 0, so its high word decides "no"; a
// tie there is resolved by the exact path like any other)
__device__ __forceinline__ bool lt_hi(const Thr &t, uint32_t h, bool &tie, uint32_t m2) {
    const uint32_t ho = h ^ __umulhi(h, m2);  // h ^ (h >> 31)
    const uint32_t hl = (uint32_t)(t.le >> 32);
    tie |= ho == hl;
    return ho < hl;
}
// the same decision without forming h ^ (h >> 31): that xor only touches bit
// 0, so with H = hl & ~1 the high-word compare ho < hl is h < H whenever the
// top 31 bits differ; equal top bits (h in {H, H + 1}, probability 2^-31)
// count as a tie and go to the exact path.  Three ALU ops, no IMAD.HI.
__device__ __forceinline__ bool lt_top(uint32_t H, uint32_t h, bool &tie) {
    tie |= h - H < 2u;
    return h < H;
}
__device__ __forceinline__ uint32_t top_thr(const Thr &t) { return (uint32_t)(t.le >> 32) & ~1u; }

__global__ void k_plan_rows(RunConsts c, PlanArgs a) {
    QTRACE(6);
    const int64_t g = a.st->g_plan;
    if (g > c.G) return;
    const int64_t b = g & 1;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < c.NP; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t key = fold_key3(c.seed, (uint64_t)g, (uint64_t)i);
        int4 pk;
        int32_t jr;
        de_row_draws(c, key, i, pk, jr);
        a.keys[b * c.NP + i] = key;
        a.picks[b * c.NP + i] = pk;
        a.jrand[b * c.NP + i] = jr;
    }
}

template <bool EXACT>
__device__ __forceinline__ bool draw_lt(const RunConsts &c, const Thr &t, uint64_t x, uint32_t h, bool &tie) {
    return EXACT ? passes_hi(t, x, h) : lt_top(top_thr(t), h, tie);
}

// The first two wolf draws of one gene as plane bits P0..P2: social; then
// pick (social) or disturbed / flipped (row 2 early, row 5 late).  The third
// draw (state or plus level) matters only for a minority of genes, and which
// ones depends on the leaders, so k_gwo_apply draws it for exactly those
// genes.  Straight-line code (selects only), so the draws of several genes
// interleave.  EXACT = false decides every compare on the high word and sets
// `tie` when one tied; the caller then redoes the gene with EXACT = true.
// zs is the social draw's counter state key + p0 * GOLD (p0 = m + 1 + D + j,
// plus one); the second draw sits gsoc = D * GOLD (social: pick row) or gnon =
// 2D * GOLD (early: disturb row) / 5D * GOLD (late: flip row) further on.
template <int K, bool EXACT>
__device__ __forceinline__ uint32_t wolf_code_z(const RunConsts &c, const GenThr &t, uint64_t zs, uint64_t gsoc,
                                                uint64_t gnon, bool early, bool &tie) {
    const uint64_t x1 = mix_pre2z(zs, c);
    const bool soc = draw_lt<EXACT>(c, t.sl, x1, mix_hi2(x1), tie);
    const uint64_t x2 = mix_pre2z(zs + (soc ? gsoc : gnon), c);
    const uint32_t h2 = mix_hi2(x2);
    uint32_t pick;
    if (K == 4) {
        pick = h2 >> 30;  // int(u * 4) = top two bits
    } else {
        const uint64_t z = x2 * kMix2;
        const int pv = (int)((double)((z ^ (z >> 31)) >> 11) * kTwoM53 * (double)K);
        pick = (uint32_t)min(pv, K - 1);
    }
    const bool f2 = draw_lt<EXACT>(c, early ? t.dist : t.flip, x2, h2, tie);
    return soc ? 1u | (pick << 1) : (f2 ? 2u : 0u);
}
template <int K, bool EXACT>
__device__ __forceinline__ uint32_t wolf_code(const RunConsts &c, const GenThr &t, uint64_t key, uint32_t p0,
                                              uint32_t D, bool early, bool &tie) {
    return wolf_code_z<K, EXACT>(c, t, key + (uint64_t)p0 * kGold, (uint64_t)D * kGold,
                                 (uint64_t)(early ? 2 * D : 5 * D) * kGold, early, tie);
}

// planes P0..P2 of one 32-gene word from each lane's code; lane `writer`
// stores them (P3 cleared; k_gwo_apply completes P2..P4)
__device__ __forceinline__ void store_planes(uint32_t *dst_word, uint32_t code, int lane, int writer) {
    const uint32_t p0 = __ballot_sync(0xffffffffu, code & 1u);
    const uint32_t p1 = __ballot_sync(0xffffffffu, code & 2u);
    const uint32_t p2 = __ballot_sync(0xffffffffu, code & 4u);
    if (lane == writer) *reinterpret_cast<uint4 *>(dst_word) = make_uint4(p0, p1, p2, 0u);
}

// The wolf planes of row genes [jc, jc + len) (len a multiple of
// 2 * kRowThreads) by one CTA: each thread draws two genes at a time
// (independent chains), warps ballot the plane words.
template <int K>
__device__ __forceinline__ void wolf_chunk(const RunConsts &c, const GenThr &t, uint64_t key, uint32_t p_wolf,
                                           uint32_t *prow, int jc, int len) {
    const uint32_t Dg = (uint32_t)c.Dg;  // stream layout
    const int D = (int)c.D;              // this shard's genes
    const bool early = t.early != 0;
    const int lane = threadIdx.x & 31;
#pragma unroll 1
    for (int it = 0; it < len; it += 2 * kRowThreads) {
        int j[2];
        uint32_t code[2];
        bool tie[2] = {false, false};
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            j[h] = jc + it + h * kRowThreads + (int)threadIdx.x;
            code[h] = wolf_code<K, false>(c, t, key, p_wolf + (uint32_t)j[h], Dg, early, tie[h]);
            if (j[h] >= D) code[h] = 0u, tie[h] = false;
        }
        if (__any_sync(0xffffffffu, tie[0] || tie[1])) {
#pragma unroll
            for (int h = 0; h < 2; ++h)
                if (tie[h]) code[h] = wolf_code<K, true>(c, t, key, p_wolf + (uint32_t)j[h], Dg, early, tie[h]);
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            if (j[h] - lane >= (int)c.Dp) break;  // warp-uniform
            store_planes(prow + ((j[h] - lane) >> 5) * kPlanes, code[h], lane, 0);
        }
    }
}

// the wolf planes of generation g_plan for this rank's rows on the side
// stream (QPM_WOLF=planner)
// NOW: the current generation's planes instead (QPM_WOLF=side: forked after
// the trial, joined before k_gwo_apply)
template <int K, bool NOW = false>
__global__ void __launch_bounds__(kRowThreads) k_plan_wolf(RunConsts c, PlanArgs a) {
    QTRACE(8);
    const int64_t g = NOW ? a.st->g : a.st->g_plan;
    if (g > c.G) return;
    const int64_t b = g & 1;
    const GenThr t = a.gthr[g];
    const int nchunk = (int)((c.Dp + kGenesPerBlock - 1) / kGenesPerBlock);
    const int64_t items = a.n_rows * nchunk;
    for (int64_t item = blockIdx.x; item < items; item += gridDim.x) {
        const int64_t i = a.row_lo + item / nchunk;
        const int jc = (int)(item % nchunk) * kGenesPerBlock;
        const uint32_t p_wolf = (uint32_t)a.picks[b * c.NP + i].w + 2 + (uint32_t)(c.Dg + c.g0);  // m + 1 + Dg + (g0 + j), plus one
        wolf_chunk<K>(c, t, a.keys[b * c.NP + i], p_wolf, a.planes + (b * c.NP + i) * c.W * kPlanes, jc,
                            kGenesPerBlock);
    }
}

__global__ void k_plan_bump(EngineState *st) {
    QTRACE(7);
    st->g_plan += 1;
}

// ---------------------------------------------------------------- init
__global__ void __launch_bounds__(kRowThreads) k_init_population(RunConsts c, double *__restrict__ genome,
                                                                 uint32_t *__restrict__ bits,
                                                                 int32_t *__restrict__ slot_of,
                                                                 int32_t *__restrict__ spare_of,
                                                                 uint32_t *__restrict__ slot_tag) {
    const int64_t i = blockIdx.y;
    const uint64_t key = fold_key3(c.seed, 0, (uint64_t)i);  // stream (seed, 0, i), optimizer.py:223
    double *row = genome + i * c.Dp;
    uint32_t *brow = bits + i * c.W;
    for (int jb = 0; jb < (int)c.Dp; jb += kGenesPerBlock)
#pragma unroll
        for (int it = 0; it < kGenesPerThread; ++it) {
            const int j = jb + it * kRowThreads + threadIdx.x;
            bool neg = false;
            if (j < (int)c.D) {
                const double x = c.x_lo + (double)(mix_at(key, (uint32_t)(c.g0 + j) + 1) >> 11) * kTwoM53 * c.x_span;
                row[j] = x;
                neg = !(x >= 0.0);
            }
            const uint32_t word = __ballot_sync(0xffffffffu, neg);
            if ((threadIdx.x & 31) == 0 && j < (int)c.Dp) brow[j >> 5] = word;
        }
    if (threadIdx.x == 0) {
        slot_of[i] = (int32_t)i;
        if (slot_tag) slot_tag[i] = (uint32_t)i;
        spare_of[i] = (int32_t)(c.NP + i);
    }
}

// ---------------------------------------------------------------- DE trial
// de_mutate + de_crossover (optimizer.py:229-262) with the planner's indices
// and mask: trial_j = take_j ? x_r1 + F (x_r2 - x_r3) : x_i, written to the
// spare slot with its sign bits.  No random draws left here: the kernel
// streams the genome rows it needs (HBM-bound).  Work items are
// (row, 1024-gene chunk) over a persistent grid.
struct TrialArgs {
    const EngineState *st;
    const GenThr *gthr;
    int64_t row_lo, n_rows;
    const int4 *picks;       // [2][NP]
    const uint64_t *keys;    // [2][NP]
    const int32_t *jrand;    // [2][NP]
    uint32_t *planes;        // [2][NP][W][kPlanes] wolf planes (P0..P2 stored)
    const int32_t *slot_of, *spare_of;
    const uint32_t *slot_tag;  // [NP] slot_of[i] | slot_bin[slot_of[i]] << 31 (QPM_SLOT_TAG)
    uint8_t *slot_bin;
    double *genome;
    uint32_t *bits;
    uint32_t *cbits;  // [NP][W] the generation's candidate sign rows, dense by individual: scored from
                      // here (no slot indirection) and, multi-GPU, all-gathered from here
};



// The trial of row i over genes [jc, jc + kDeChunk) with the crossover mask
// drawn inline (one splitmix64 per gene).  For K > 0 (run_hybrid)
// the same pass draws the row's wolf planes for this generation (three
// draws per gene): the trial is HBM-bound (~30 B per gene) and the integer
// work of the draws runs while the genome loads are in flight.
// Per-row operands of a trial CTA, resolved once by thread 0 and shared
// through shared memory (the slot lookups and pointer arithmetic would
// otherwise be repeated by all eight warps).
struct TrialRow {
    RowRef xi, x1, x2, x3;
    double *out;
    uint32_t *bout, *prow;
    uint32_t *dout;  // the candidate's dense row
    uint64_t key;
    int64_t out_slot;
    double F;
    GenThr t;
    uint32_t p_mask;
    int jr;
    int bin;  // a source row is a +/-1 (bits-only) slot
};

__device__ __forceinline__ void trial_row_setup(const RunConsts &c, const TrialArgs &a, int64_t g, int64_t i,
                                                TrialRow &r) {
    const int64_t b = g & 1;
    const int4 pk = a.picks[b * c.NP + i];
    r.key = a.keys[b * c.NP + i];
    r.jr = a.jrand[b * c.NP + i];
    if (a.slot_tag) {  // slot and +/-1 flag in one load: picks -> tag, no slot_bin level
        r.xi = row_ref_tag(c, a.slot_tag[i], a.genome, a.bits);
        r.x1 = row_ref_tag(c, a.slot_tag[pk.x], a.genome, a.bits);
        r.x2 = row_ref_tag(c, a.slot_tag[pk.y], a.genome, a.bits);
        r.x3 = row_ref_tag(c, a.slot_tag[pk.z], a.genome, a.bits);
    } else {
        r.xi = row_ref(c, a.slot_of[i], a.slot_bin, a.genome, a.bits);
        r.x1 = row_ref(c, a.slot_of[pk.x], a.slot_bin, a.genome, a.bits);
        r.x2 = row_ref(c, a.slot_of[pk.y], a.slot_bin, a.genome, a.bits);
        r.x3 = row_ref(c, a.slot_of[pk.z], a.slot_bin, a.genome, a.bits);
    }
    r.bin = r.xi.bin | r.x1.bin | r.x2.bin | r.x3.bin;
    r.out_slot = a.spare_of[i];
    r.out = a.genome + r.out_slot * c.Dp;
    r.bout = a.bits + r.out_slot * c.W;
    r.dout = a.cbits ? a.cbits + i * c.W : nullptr;
    r.prow = a.planes + (b * c.NP + i) * c.W * kPlanes;
    r.p_mask = (uint32_t)(pk.w + 2 + c.g0);  // m + 1 + (g0 + j), plus one: j counts this shard's genes
    r.jr -= (int)c.g0;                      // j_rand relative to the shard (never matches outside it)
    r.F = a.st->F;
    r.t = a.gthr[g];
}

constexpr int kDeSteps = 2;  // 64-gene warp steps per k_de_trial batch (registers)
#ifndef QPM_TRIAL_LOADS
#define QPM_TRIAL_LOADS 1  // f64-row trials: branch-free base-row select (1) or take-branched loads (0)
#endif

// L2 policy of the trial's genome traffic (QPM_L2_HINTS): the current
// population (NP rows, 82 MB at C2) is read ~4 times per generation as
// donors / targets and fits the 126 MB L2; the trial rows written to the
// spare slots are not read again this generation.  Donor loads ask L2 to
// keep their lines (evict_last), trial stores to drop theirs first
// (st.global.cs), so the written stream does not push the donors out.
#ifndef QPM_L2_HINTS
#define QPM_L2_HINTS 1
#endif
__device__ __forceinline__ double ld_keep(const double *p) {
#if QPM_L2_HINTS
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    double v;
    asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
#else
    return *p;
#endif
}
__device__ __forceinline__ void st_stream(double *p, double v) {
#if QPM_L2_HINTS && !defined(QPM_NO_STCS)
    __stcs(p, v);
#else
    *p = v;
#endif
}

// +1.0 / -1.0 from a sign bit (bit 0 of b; 1 = -1): built on the high word
__device__ __forceinline__ double pm1(uint32_t b) { return __hiloint2double((int)(0x3FF00000u | (b << 31)), 0); }

// One warp's share of a row: nb batches of kDeSteps 64-gene steps, step st of
// batch bt at genes j0 + (bt kDeSteps + st) SPAN (SPAN = 512: the eight warps of
// a CTA interleave over a chunk; SPAN = 64: one warp walks a whole row).
template <bool BIN, bool FULL, int K, int SPAN>
__device__ __forceinline__ void de_trial_chunk(const RunConsts &c, const TrialArgs &a, const TrialRow &r, int j0,
                                               int nb) {
    // A warp covers 64 genes per step: lane l owns genes l and l+32, so every
    // load/store is one coalesced 256-byte warp access and the two sign words
    // are plain ballots.
    const RowRef xi = r.xi, x1 = r.x1, x2 = r.x2, x3 = r.x3;
    double *out = r.out;
    uint32_t *bout = r.bout, *prow = r.prow;
    const uint64_t key = r.key;
    const int jr = r.jr;
    const double F = r.F;
    const GenThr t = r.t;
    const bool early = t.early != 0;
    const uint32_t p_mask = r.p_mask;
    const int D = (int)c.D;
    // counter states advance by constant multiples of GOLD: one 64-bit add
    // per draw instead of a 32 x 64 product (the wolf block starts D later)
    const uint64_t gD = (uint64_t)(uint32_t)c.Dg * kGold;
    const uint64_t gnon = (uint64_t)(uint32_t)(early ? 2 * c.Dg : 5 * c.Dg) * kGold;
    const uint32_t Hcr = top_thr(c.thr_cr);
    const int lane = threadIdx.x & 31;
    constexpr int kSpan = SPAN;
#pragma unroll 1
    for (int bt = 0; bt < nb; ++bt) {
        const int jb = j0 + bt * kSpan * kDeSteps;
        if (!FULL && jb >= (int)c.Dp) break;
        // mask bits, then every genome load of the batch, the math and the
        // stores, then the wolf draws (other warps' loads are in flight)
        uint32_t mb[kDeSteps];
        bool tie = false;
        const uint64_t zb = key + (uint64_t)(p_mask + (uint32_t)(jb + lane)) * kGold;  // mask draw of gene jb + lane
#pragma unroll
        for (int st = 0; st < kDeSteps; ++st) {
            mb[st] = 0u;
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const int jj = jb + st * kSpan + lane + 32 * q;
                bool ti = false;
                const uint64_t x = mix_pre2z(zb + (uint64_t)(st * kSpan + 32 * q) * kGold, c);
                const bool take = lt_top(Hcr, mix_hi2(x), ti) || jj == jr;
                if (FULL || jj < D) {
                    mb[st] |= take ? 1u << q : 0u;
                    tie |= ti;
                }
            }
        }
        if (__any_sync(0xffffffffu, tie) && tie) {  // a high-word tie (p = 2^-32): exact compares
#pragma unroll
            for (int st = 0; st < kDeSteps; ++st) {
                mb[st] = 0u;
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const int jj = jb + st * kSpan + lane + 32 * q;
                    const uint64_t x = mix_pre2(key, p_mask + (uint32_t)jj, c);
                    if ((FULL || jj < D) && (passes_hi(c.thr_cr, x, mix_hi2(x)) || jj == jr)) mb[st] |= 1u << q;
                }
            }
        }
        double y[kDeSteps][2], p1[kDeSteps][2], p2[kDeSteps][2], p3[kDeSteps][2];
#pragma unroll
        for (int st = 0; st < kDeSteps; ++st) {
            const int j64 = jb + st * kSpan;
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const int j = j64 + lane + 32 * q;
                if (!FULL || BIN || !QPM_TRIAL_LOADS) y[st][q] = p1[st][q] = p2[st][q] = p3[st][q] = 0.0;
                if (!FULL && j >= D) continue;
                if (!BIN && QPM_TRIAL_LOADS) {
                    // f64 rows: the base (x_r1 where the mask takes the
                    // mutant, x_i elsewhere) by a per-lane row select, and
                    // both difference rows unconditionally -- three loads per
                    // gene, no divergent branch; the lanes that do not take
                    // the mutant add no DRAM sectors (their neighbours' loads
                    // of x_r2, x_r3 already fetch them)
                    const bool tk = (mb[st] >> q) & 1u;
                    y[st][q] = ld_keep((tk ? x1.f() : xi.f()) + j);
                    p1[st][q] = y[st][q];
                    p2[st][q] = ld_keep(x2.f() + j);
                    p3[st][q] = ld_keep(x3.f() + j);
                } else if (BIN) {
                    // +/-1 rows: one broadcast word load per 32 genes
                    const int w = (j64 >> 5) + q;
                    y[st][q] = !xi.bin ? xi.f()[j] : pm1(xi.b()[w] >> lane);
                    p1[st][q] = !x1.bin ? x1.f()[j] : pm1(x1.b()[w] >> lane);
                    p2[st][q] = !x2.bin ? x2.f()[j] : pm1(x2.b()[w] >> lane);
                    p3[st][q] = !x3.bin ? x3.f()[j] : pm1(x3.b()[w] >> lane);
                } else if ((mb[st] >> q) & 1u) {
                    p1[st][q] = ld_keep(x1.f() + j);
                    p2[st][q] = ld_keep(x2.f() + j);
                    p3[st][q] = ld_keep(x3.f() + j);
                } else {
                    y[st][q] = ld_keep(xi.f() + j);
                }
            }
        }
#pragma unroll
        for (int st = 0; st < kDeSteps; ++st) {
            const int j64 = jb + st * kSpan;  // this warp's 64-gene span
            if (!FULL && j64 >= (int)c.Dp) break;
            bool neg[2];
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const int j = j64 + lane + 32 * q;
                neg[q] = false;
                if (FULL || j < D) {
                    const double v = ((mb[st] >> q) & 1u) ? p1[st][q] + F * (p2[st][q] - p3[st][q]) : y[st][q];
                    st_stream(out + j, v);
                    neg[q] = !(v >= 0.0);
                } else if (j < (int)c.Dp) {
                    out[j] = 0.0;
                }
            }
            const uint32_t w0 = __ballot_sync(0xffffffffu, neg[0]);
            const uint32_t w1 = __ballot_sync(0xffffffffu, neg[1]);
            if (lane < 2) {
                bout[(j64 >> 5) + lane] = lane ? w1 : w0;
                if (r.dout) r.dout[(j64 >> 5) + lane] = lane ? w1 : w0;
            }
        }
        if (K > 0) {  // after the stores: the load registers are free again
            uint32_t code[kDeSteps][2];
            bool wtie = false;
#pragma unroll
            for (int st = 0; st < kDeSteps; ++st) {
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const int jj = jb + st * kSpan + lane + 32 * q;
                    bool ti = false;
                    code[st][q] = wolf_code_z<K, false>(c, t, zb + (uint64_t)(st * kSpan + 32 * q) * kGold + gD, gD,
                                                        gnon, early, ti);
                    if (!FULL && jj >= D) code[st][q] = 0u, ti = false;
                    wtie |= ti;
                }
            }
            if (__any_sync(0xffffffffu, wtie) && wtie) {
#pragma unroll
                for (int st = 0; st < kDeSteps; ++st) {
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                        const int jj = jb + st * kSpan + lane + 32 * q;
                        bool ti = false;
                        if (FULL || jj < D)
                            code[st][q] = wolf_code_z<K, true>(
                                c, t, zb + (uint64_t)(st * kSpan + 32 * q) * kGold + gD, gD, gnon, early, ti);
                    }
                }
            }
#pragma unroll
            for (int st = 0; st < kDeSteps; ++st) {
                const int j64 = jb + st * kSpan;
                if (!FULL && j64 >= (int)c.Dp) break;
#pragma unroll
                for (int q = 0; q < 2; ++q)
                    store_planes(prow + ((j64 >> 5) + q) * kPlanes, code[st][q], lane, q);
            }
        }
    }
}

template <int K>
__device__ __forceinline__ void de_trial_dispatch(const RunConsts &c, const TrialArgs &a, const TrialRow &r, int jc) {
    constexpr int kSpan = kRowThreads * 2;  // genes per CTA step
    constexpr int kBatches = kDeChunk / (kSpan * kDeSteps);
    const bool full = jc + kDeChunk <= (int)c.D;
    const int j0 = jc + (int)(threadIdx.x >> 5) * 64;
    if (r.bin) {
        if (full)
            de_trial_chunk<true, true, K, kSpan>(c, a, r, j0, kBatches);
        else
            de_trial_chunk<true, false, K, kSpan>(c, a, r, j0, kBatches);
    } else {
        if (full)
            de_trial_chunk<false, true, K, kSpan>(c, a, r, j0, kBatches);
        else
            de_trial_chunk<false, false, K, kSpan>(c, a, r, j0, kBatches);
    }
    if (jc == 0 && threadIdx.x == 0) a.slot_bin[r.out_slot] = 0;
}

// Warp items (short rows -- a column shard of a multi-GPU run, Dp <=
// kDeRowsDefaultDp -- or QPM_DE_ROWS): each warp walks the genes [ch k, ch (k+1))
// of one row (ch = whole row for short rows), eight items per CTA.  Each
// warp resolves its own row (lane 0, broadcast through shared memory) with no
// CTA barrier, so a row's setup latency hides under the other warps' work.
constexpr int kDeRowsMaxDp = 4096;
// the default switch to warp items: the TMA-staged row kernel wins above it
// (emulated C2-shape shards, tools/shard_probe.py: W = 4 (2,560 genes) trial +
// scan phase 129.5 -> 109.6 us with TMA; W = 8 (1,280 genes) 117.5 -> 135.3 us)
constexpr int kDeRowsDefaultDp = 2048;
template <int K>
__global__ void __launch_bounds__(kRowThreads, QPM_DE_MINB) k_de_trial_rows(RunConsts c, TrialArgs a, int ch) {
    QTRACE(0);
    pdl_wait();
    pdl_trigger<1>();
    QTRACE_STARTED();
    constexpr int kWarps = kRowThreads / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nch = (int)((c.Dp + ch - 1) / ch);
    const int64_t item = (int64_t)blockIdx.x * kWarps + warp;
    if (item >= a.n_rows * nch) return;  // warp-uniform
    const int64_t i = a.row_lo + item / nch;
    const int j0 = (int)(item % nch) * ch, j1 = min(j0 + ch, (int)c.Dp);
    __shared__ TrialRow s_rows[kWarps];
    if (lane == 0) trial_row_setup(c, a, a.st->g, i, s_rows[warp]);
    __syncwarp();
    const TrialRow &r = s_rows[warp];
    constexpr int kB = 64 * kDeSteps;  // genes per warp batch (ch is a multiple)
    const int jf = max(j0, min(j1, (int)c.D / kB * kB));  // batches below jf lie inside D
    const int nfull = (jf - j0) / kB, ntail = (j1 - jf + kB - 1) / kB;
    if (r.bin) {
        de_trial_chunk<true, true, K, 64>(c, a, r, j0, nfull);
        de_trial_chunk<true, false, K, 64>(c, a, r, jf, ntail);
    } else {
        de_trial_chunk<false, true, K, 64>(c, a, r, j0, nfull);
        de_trial_chunk<false, false, K, 64>(c, a, r, jf, ntail);
    }
    if (lane == 0 && j0 == 0) a.slot_bin[r.out_slot] = 0;
}

// one CTA per (row, kDeChunk genes).  K = leader count when the CTA also
// draws the wolf planes (run_hybrid), 0 otherwise
template <int K>
__global__ void __launch_bounds__(kRowThreads, QPM_DE_MINB) k_de_trial(RunConsts c, TrialArgs a) {
    QTRACE(0);
    pdl_wait();
    pdl_trigger<1>();
    QTRACE_STARTED();
    const int nchunk = (int)((c.Dp + kDeChunk - 1) / kDeChunk);
    const int64_t i = a.row_lo + blockIdx.x / nchunk;
    const int jc = (int)(blockIdx.x % nchunk) * kDeChunk;
    __shared__ TrialRow s_row;
    if (threadIdx.x == 0) trial_row_setup(c, a, a.st->g, i, s_row);
    __syncthreads();
    de_trial_dispatch<K>(c, a, s_row, jc);
}

// ---------------------------------------------------------------- DE trial, TMA-staged
// The same trial with its four source rows (x_i, x_r1, x_r2, x_r3) streamed
// into shared memory by the bulk-copy engine (cp.async.bulk, one elected
// thread, an mbarrier per stage) kTmaBufs stages ahead of the warps.  The
// global-load version keeps at most 12 doubles per lane in flight and stalls
// on them (long scoreboard, 64-register spills of the row pointers); here
// 4 x 4 KB per stage and kTmaBufs stages per CTA are in flight while the warps
// compute the stage's mask and wolf draws, which do not depend on the data.
// A stage is 512 genes: warp w owns genes [64 w, 64 w + 64), lane l genes l
// and l + 32, exactly the global-load kernel's per-warp step, so every draw,
// every rounding and every stored word is the same.  Rows that are +/-1 slots
// (bits only) are staged as their bit words (128 B per 1024 genes).
#ifndef QPM_DE_TMA
#define QPM_DE_TMA 1
#endif
#ifndef QPM_DE_TMA_STEPS
#define QPM_DE_TMA_STEPS 2  // 64-gene warp steps per stage (a stage is 512 x this genes)
#endif
#ifndef QPM_DE_TMA_BUFS
#define QPM_DE_TMA_BUFS 2
#endif
#ifndef QPM_DE_TMA_MINB
#define QPM_DE_TMA_MINB 3  // CTAs per SM: 3 x (BUFS x 32 KB) of stage ring
#endif
constexpr int kTmaSteps = QPM_DE_TMA_STEPS;
constexpr int kTmaStage = 512 * kTmaSteps;  // genes per stage
constexpr int kTmaBufs = QPM_DE_TMA_BUFS;
constexpr size_t kTmaSmem = (size_t)kTmaBufs * 4 * kTmaStage * sizeof(double);
constexpr int64_t kTmaLongRows = 32768;  // rows at least this long take 8,192-gene items

__device__ __forceinline__ uint32_t de_smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void de_mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(de_smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void de_mbar_expect(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(de_smem_addr(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void de_bulk(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            de_smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(de_smem_addr(bar))
        : "memory");
}
__device__ __forceinline__ void de_mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(de_smem_addr(bar)),
        "r"(parity)
        : "memory");
}

// the row's operands in registers for the whole item (the global-load kernel
// reads them from the shared TrialRow per batch)
struct TmaRow {
    const void *src[4];  // x_i, x_r1, x_r2, x_r3: f64 rows, or bit rows for +/-1 slots (bit k of bin)
    uint32_t bin;
    double *out;
    uint32_t *bout, *dout, *prow;
    uint64_t key;
    uint32_t p_mask;
    int jr;
    double F;
    uint32_t Hsl, H2;  // top-31-bit thresholds of the social draw and of the second draw
    bool early;
};

// wolf code of one gene on the high-word fast path (wolf_code_z<K, false>
// with the thresholds pre-shifted); K = 4 only (the pick is the top two bits)
__device__ __forceinline__ uint32_t wolf_code_fast4(const RunConsts &c, const TmaRow &w, uint64_t zs, uint64_t gsoc,
                                                    uint64_t gnon, bool &tie) {
    const uint64_t x1 = mix_pre2z(zs, c);
    const bool soc = lt_top(w.Hsl, mix_hi2(x1), tie);
    const uint64_t x2 = mix_pre2z(zs + (soc ? gsoc : gnon), c);
    const uint32_t h2 = mix_hi2(x2);
    const bool f2 = lt_top(w.H2, h2, tie);
    return soc ? 1u | ((h2 >> 30) << 1) : (f2 ? 2u : 0u);
}

// one warp's kTmaSteps x 64 genes of a landed stage: genes j64 + 512 s + lane
// + 32 q (s < kTmaSteps, q < 2), the global-load kernel's layout
// a lane's gene of a staged row: the f64 value at offset o, or +/-1 from bit
// `lane` of the staged bit word wi (warp-uniform: one broadcast load per 32 genes)
__device__ __forceinline__ double tma_gene(const double *srow, uint32_t binrow, int o, int wi, int lane) {
    if (!binrow) return srow[o];
    return pm1(reinterpret_cast<const uint32_t *>(srow)[wi] >> lane);
}

// the draws of one warp's kTmaSteps x 64 genes (mask bits returned, wolf
// planes stored): no data dependence, so they run while the stage lands
template <bool FULL, int K>
__device__ __forceinline__ uint32_t de_tma_draws(const RunConsts &c, const TrialRow &r, const TmaRow &w, int j64,
                                                 uint64_t gD, uint64_t gnon, uint32_t Hcr) {
    const int lane = threadIdx.x & 31;
    const int D = (int)c.D;
    const uint64_t zb = w.key + (uint64_t)(w.p_mask + (uint32_t)(j64 + lane)) * kGold;
    uint32_t mb = 0u;  // bit 2 s + q: take the mutant
    bool tie = false;
#pragma unroll
    for (int st = 0; st < kTmaSteps; ++st)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const int jj = j64 + 512 * st + lane + 32 * q;
            bool ti = false;
            const uint64_t x = mix_pre2z(zb + (uint64_t)(512 * st + 32 * q) * kGold, c);
            const bool take = lt_top(Hcr, mix_hi2(x), ti) || jj == w.jr;
            if (FULL || jj < D) {
                mb |= take ? 1u << (2 * st + q) : 0u;
                tie |= ti;
            }
        }
    if (__any_sync(0xffffffffu, tie) && tie) {
        mb = 0u;
#pragma unroll
        for (int st = 0; st < kTmaSteps; ++st)
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const int jj = j64 + 512 * st + lane + 32 * q;
                const uint64_t x = mix_pre2(w.key, w.p_mask + (uint32_t)jj, c);
                if ((FULL || jj < D) && (passes_hi(c.thr_cr, x, mix_hi2(x)) || jj == w.jr)) mb |= 1u << (2 * st + q);
            }
    }
    if (K > 0) {  // wolf planes of the same genes: no data dependence, drawn while the stage lands
        uint32_t code[kTmaSteps][2];
        bool wtie = false;
#pragma unroll
        for (int st = 0; st < kTmaSteps; ++st)
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const int jj = j64 + 512 * st + lane + 32 * q;
                const uint64_t zs = zb + (uint64_t)(512 * st + 32 * q) * kGold + gD;
                bool ti = false;
                if (K == 4)
                    code[st][q] = wolf_code_fast4(c, w, zs, gD, gnon, ti);
                else
                    code[st][q] = wolf_code_z<K, false>(c, r.t, zs, gD, gnon, w.early, ti);
                if (!FULL && jj >= D) code[st][q] = 0u, ti = false;
                wtie |= ti;
            }
        if (__any_sync(0xffffffffu, wtie) && wtie) {
#pragma unroll
            for (int st = 0; st < kTmaSteps; ++st)
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const int jj = j64 + 512 * st + lane + 32 * q;
                    bool ti = false;
                    if (FULL || jj < D)
                        code[st][q] = wolf_code_z<K, true>(c, r.t, zb + (uint64_t)(512 * st + 32 * q) * kGold + gD, gD,
                                                           gnon, w.early, ti);
                }
        }
#pragma unroll
        for (int st = 0; st < kTmaSteps; ++st) {
            if (!FULL && j64 + 512 * st >= (int)c.Dp) break;  // (a 64-gene span lies wholly inside or outside Dp)
#pragma unroll
            for (int q = 0; q < 2; ++q)
                store_planes(w.prow + (((j64 + 512 * st) >> 5) + q) * kPlanes, code[st][q], lane, q);
        }
    }
    return mb;
}

// the trial values of the same genes from the landed stage sx
template <bool FULL, bool BIN>
__device__ __forceinline__ void de_tma_data(const RunConsts &c, const TmaRow &w, const double *sx, int j64,
                                            uint32_t mb) {
    const int lane = threadIdx.x & 31;
    const int D = (int)c.D;
    const double *s0 = sx + (j64 & 511) + lane;  // this lane's first gene in the stage
#pragma unroll
    for (int st = 0; st < kTmaSteps; ++st) {
        if (!FULL && j64 + 512 * st >= (int)c.Dp) break;
        bool neg[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const int j = j64 + 512 * st + lane + 32 * q;
            const int o = 512 * st + 32 * q;
            const bool tk = (mb >> (2 * st + q)) & 1u;
            double y, p2, p3;
            if (!BIN) {
                y = s0[(tk ? kTmaStage : 0) + o];  // x_r1 where the mask takes the mutant, else x_i
                p2 = s0[2 * kTmaStage + o];
                p3 = s0[3 * kTmaStage + o];
            } else {  // some rows are +/-1 slots: each row from its staged f64 values or bits
                const int og = (j64 & 511) + lane + o;       // gene offset in the stage
                const int wi = ((j64 & 511) >> 5) + 16 * st + q;  // its bit word (lane = bit)
                const double yi = tma_gene(sx, w.bin & 1u, og, wi, lane);
                const double y1 = tma_gene(sx + kTmaStage, w.bin & 2u, og, wi, lane);
                y = tk ? y1 : yi;
                p2 = tma_gene(sx + 2 * kTmaStage, w.bin & 4u, og, wi, lane);
                p3 = tma_gene(sx + 3 * kTmaStage, w.bin & 8u, og, wi, lane);
            }
            neg[q] = false;
            if (FULL || j < D) {
                const double v = tk ? y + w.F * (p2 - p3) : y;
                st_stream(w.out + j, v);
                neg[q] = !(v >= 0.0);
            } else {
                w.out[j] = 0.0;  // padding genes [D, Dp)
            }
        }
        const uint32_t w0 = __ballot_sync(0xffffffffu, neg[0]);
        const uint32_t w1 = __ballot_sync(0xffffffffu, neg[1]);
        if (lane < 2) {
            const int wi = ((j64 + 512 * st) >> 5) + lane;
            w.bout[wi] = lane ? w1 : w0;
            if (w.dout) w.dout[wi] = lane ? w1 : w0;
        }
    }
}

// CHUNK: genes per CTA item (4,096; 8,192 for rows of >= 32,768 genes: C3
// 6.67 -> 6.60 ms/gen, while C2's 10,112-gene rows keep 4,096 -- 8,192 would
// leave a 1,920-gene second item per row)
template <int K, int CHUNK = kDeChunk>
__global__ void __launch_bounds__(kRowThreads, QPM_DE_TMA_MINB) k_de_trial_tma(RunConsts c, TrialArgs a) {
    QTRACE(0);
    pdl_wait();
    pdl_trigger<1>();
    QTRACE_STARTED();
    QSTAMP(0);
    extern __shared__ __align__(128) double s_stage[];  // [kTmaBufs][4 rows][kTmaStage]
    __shared__ __align__(8) uint64_t full[kTmaBufs];
    __shared__ uint32_t done[kTmaBufs];
    __shared__ TrialRow s_row;
    const int nchunk = (int)((c.Dp + CHUNK - 1) / CHUNK);
    const int64_t i = a.row_lo + blockIdx.x / nchunk;
    const int jc = (int)(blockIdx.x % nchunk) * CHUNK;
    // Two-phase setup by thread 0.  Phase A (st->g -> keys / picks / thresholds)
    // is all the draws need: the warps start drawing after it.  Phase B (the
    // picked rows' slot tags, one dependent load later) gives the source rows;
    // thread 0 then issues the first stages.  The other warps read the row
    // pointers only after waiting on a stage's barrier, which orders thread 0's
    // shared-memory writes (mbarrier arrive: release; wait: acquire).
    int4 pk = make_int4(0, 0, 0, 0);
    uint32_t tag_i = 0u;
    if (threadIdx.x == 0) {
        for (int b = 0; b < kTmaBufs; ++b) {
            de_mbar_init(&full[b], 1);
            done[b] = 0u;
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        const int64_t g = a.st->g;
        const int64_t b = g & 1;
        pk = a.picks[b * c.NP + i];
        TrialRow &r = s_row;
        r.key = a.keys[b * c.NP + i];
        r.jr = a.jrand[b * c.NP + i] - (int)c.g0;  // j_rand relative to the shard (never matches outside it)
        tag_i = a.slot_tag ? a.slot_tag[i] : 0u;
        r.out_slot = a.spare_of[i];
        r.out = a.genome + r.out_slot * c.Dp;
        r.bout = a.bits + r.out_slot * c.W;
        r.dout = a.cbits ? a.cbits + i * c.W : nullptr;
        r.prow = a.planes + (b * c.NP + i) * c.W * kPlanes;
        r.p_mask = (uint32_t)(pk.w + 2 + c.g0);  // m + 1 + (g0 + j), plus one: j counts this shard's genes
        r.F = a.st->F;
        r.t = a.gthr[g];
    }
    __syncthreads();
    if (threadIdx.x == 0) {  // phase B
        TrialRow &r = s_row;
        if (a.slot_tag) {
            r.xi = row_ref_tag(c, tag_i, a.genome, a.bits);
            r.x1 = row_ref_tag(c, a.slot_tag[pk.x], a.genome, a.bits);
            r.x2 = row_ref_tag(c, a.slot_tag[pk.y], a.genome, a.bits);
            r.x3 = row_ref_tag(c, a.slot_tag[pk.z], a.genome, a.bits);
        } else {
            r.xi = row_ref(c, a.slot_of[i], a.slot_bin, a.genome, a.bits);
            r.x1 = row_ref(c, a.slot_of[pk.x], a.slot_bin, a.genome, a.bits);
            r.x2 = row_ref(c, a.slot_of[pk.y], a.slot_bin, a.genome, a.bits);
            r.x3 = row_ref(c, a.slot_of[pk.z], a.slot_bin, a.genome, a.bits);
        }
    }
    QSTAMP(1);  // setup phase A done (CTA 0)
    const TrialRow &r = s_row;
    TmaRow w;
    w.out = r.out;
    w.bout = r.bout;
    w.dout = r.dout;
    w.prow = r.prow;
    w.key = r.key;
    w.p_mask = r.p_mask;
    w.jr = r.jr;
    w.F = r.F;
    w.early = r.t.early != 0;
    w.Hsl = top_thr(r.t.sl);
    w.H2 = top_thr(w.early ? r.t.dist : r.t.flip);
    const int jend = min(jc + CHUNK, (int)c.Dp);
    const int nst = (jend - jc + kTmaStage - 1) / kTmaStage;
    // the source rows (valid in thread 0 after phase B, elsewhere after a stage wait)
    auto load_src = [&]() {
        w.src[0] = r.xi.p;
        w.src[1] = r.x1.p;
        w.src[2] = r.x2.p;
        w.src[3] = r.x3.p;
        w.bin = r.xi.bin | r.x1.bin << 1 | r.x2.bin << 2 | r.x3.bin << 3;
    };
    auto issue = [&](int st) {
        const int b = st % kTmaBufs;
        const int j = jc + st * kTmaStage;
        const int n = min(kTmaStage, jend - j);  // a multiple of 128 genes
        const uint32_t fb = (uint32_t)(n * (int)sizeof(double)), bb = (uint32_t)(n / 8);  // f64 / bit bytes
        double *dst = s_stage + (size_t)b * 4 * kTmaStage;
        const int nb = __popc(w.bin);
        de_mbar_expect(&full[b], (uint32_t)(4 - nb) * fb + (uint32_t)nb * bb);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if ((w.bin >> k) & 1u)
                de_bulk(dst + k * kTmaStage, static_cast<const uint32_t *>(w.src[k]) + (j >> 5), bb, &full[b]);
            else
                de_bulk(dst + k * kTmaStage, static_cast<const double *>(w.src[k]) + j, fb, &full[b]);
        }
    };
    if (threadIdx.x == 0) {
        load_src();
        for (int st = 0; st < min(nst, kTmaBufs); ++st) issue(st);
    }
    const uint64_t gD = (uint64_t)(uint32_t)c.Dg * kGold;
    const uint64_t gnon = (uint64_t)(uint32_t)(w.early ? 2 * c.Dg : 5 * c.Dg) * kGold;
    const uint32_t Hcr = top_thr(c.thr_cr);
    const int warp = threadIdx.x >> 5;
#pragma unroll 1
    for (int st = 0; st < nst; ++st) {
        const int b = st % kTmaBufs;
        const uint32_t parity = (uint32_t)((st / kTmaBufs) & 1);
        const int j64 = jc + st * kTmaStage + warp * 64;
        const double *sx = s_stage + (size_t)b * 4 * kTmaStage;
        const bool fullw = j64 + 512 * (kTmaSteps - 1) + 64 <= (int)c.D;
        const uint32_t mb = fullw ? de_tma_draws<true, K>(c, r, w, j64, gD, gnon, Hcr)
                                  : de_tma_draws<false, K>(c, r, w, j64, gD, gnon, Hcr);
        de_mbar_wait(&full[b], parity);
        if (st == 0) load_src();
        if (w.bin) {
            if (fullw)
                de_tma_data<true, true>(c, w, sx, j64, mb);
            else
                de_tma_data<false, true>(c, w, sx, j64, mb);
        } else if (fullw) {
            de_tma_data<true, false>(c, w, sx, j64, mb);
        } else {
            de_tma_data<false, false>(c, w, sx, j64, mb);
        }
        // the last warp done with the buffer refills it (its reads are in
        // registers; the bulk copy is ordered after them by the shared atomic)
        if (st + kTmaBufs < nst) {
            __syncwarp();
            if ((threadIdx.x & 31) == 0) {
                __threadfence_block();
                if (atomicAdd(&done[b], 1u) == kRowThreads / 32 - 1) {
                    done[b] = 0u;
                    issue(st + kTmaBufs);
                }
            }
        }
    }
    QSTAMP(2);  // CTA 0 thread 0 done
    if (jc == 0 && threadIdx.x == 0) a.slot_bin[r.out_slot] = 0;
}

// Horizontal fusion (QPM_WOLF=mixed): even CTAs run the trial
// of a (row, kDeChunk) item (HBM-bound), odd CTAs draw the same item's wolf
// planes (integer-ALU-bound).  The block scheduler keeps both kinds resident
// on every SM, so the draws fill the issue slots the trial's loads leave idle.
template <int K>
__global__ void __launch_bounds__(kRowThreads, QPM_DE_MINB) k_de_trial_mixed(RunConsts c, TrialArgs a) {
    pdl_wait();
    const int64_t g = a.st->g;
    const int64_t b = g & 1;
    const int nchunk = (int)((c.Dp + kDeChunk - 1) / kDeChunk);
    const int64_t item = blockIdx.x >> 1;
    const int64_t i = a.row_lo + item / nchunk;
    const int jc = (int)(item % nchunk) * kDeChunk;
    const GenThr t = a.gthr[g];
    if (blockIdx.x & 1) {
        const uint32_t p_wolf = (uint32_t)a.picks[b * c.NP + i].w + 2 + (uint32_t)(c.Dg + c.g0);  // m + 1 + Dg + (g0 + j), plus one
        wolf_chunk<K>(c, t, a.keys[b * c.NP + i], p_wolf, a.planes + (b * c.NP + i) * c.W * kPlanes, jc,
                            kDeChunk);
        return;
    }
    __shared__ TrialRow s_row;
    if (threadIdx.x == 0) trial_row_setup(c, a, g, i, s_row);
    __syncthreads();
    de_trial_dispatch<0>(c, a, s_row, jc);
}

// ---------------------------------------------------------------- wolf update
// One thread per (row, 32-gene word), one CTA row per individual: the candidate's sign word from the
// leaders' words and the row's stored planes P0..P2 (bit-sliced, ~30 logic ops per 32
// genes).  Leaders do not move (optimizer.py:454).
#ifndef QPM_APPLY_ILP
#define QPM_APPLY_ILP 2
#endif
constexpr int kApplyIlp = QPM_APPLY_ILP;  // third draws in flight per thread
template <int K>
__global__ void __launch_bounds__(kApplyThreads) k_gwo_apply(RunConsts c, TrialArgs a) {
    QTRACE(4);
    pdl_wait();
    pdl_trigger<8>();
    QTRACE_STARTED();
    // one thread per (individual, 32-gene word), flattened: short rows (a
    // column shard of a multi-GPU run) leave no idle lanes
    const int64_t idx = (int64_t)blockIdx.x * kApplyThreads + threadIdx.x;
    if (idx >= a.n_rows * c.W) return;
    const int64_t i = a.row_lo + idx / c.W;
    const int w = (int)(idx % c.W);
    int32_t lead[K];
#pragma unroll
    for (int t = 0; t < K; ++t) lead[t] = a.st->leaders[t];
    bool skip = false;
#pragma unroll
    for (int t = 0; t < K; ++t) skip |= lead[t] == i;
    if (skip || w >= (int)c.W) return;
    const int64_t g = a.st->g;
    const bool early = a.gthr[g].early != 0;
    uint32_t ld[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) ld[t] = t < K ? a.bits[(int64_t)a.slot_of[lead[t]] * c.W + w] : 0u;
    const uint32_t *pw = a.planes + (((g & 1) * c.NP + i) * c.W + w) * kPlanes;
    const uint4 q0 = *reinterpret_cast<const uint4 *>(pw);
    uint32_t pl[5] = {q0.x, q0.y, q0.z, 0u, 0u};  // P0..P2 from k_de_trial
    const int rem = (int)c.D - w * 32;
    const uint32_t valid = rem >= 32 ? 0xffffffffu : (rem <= 0 ? 0u : ((1u << rem) - 1u));
    // the third draw (row 3 state / row 4 plus) for the non-social genes whose
    // outcome depends on it: early, disturbed genes (state) and undisturbed
    // genes whose leaders disagree (plus level); late, 2-2 ties of 4 leaders
    const uint32_t z0 = ~ld[0], z1 = ~ld[1], z2 = ~ld[2], z3 = K == 4 ? ~ld[3] : 0u;
    const uint32_t a3 = z0 ^ z1 ^ z2, c3 = (z0 & z1) | (z0 & z2) | (z1 & z2);
    const uint32_t s0 = a3 ^ z3, s1 = c3 ^ (a3 & z3), s2 = c3 & (a3 & z3);  // count of +1 leaders
    const uint32_t nsoc = ~pl[0] & valid;
    const uint32_t f2 = pl[1] & nsoc;
    uint32_t need;
    if (early) {
        const uint32_t none = ~(s0 | s1 | s2);
        const uint32_t all = K == 4 ? (s2 & ~s1 & ~s0) : (s1 & s0);
        const uint32_t agree = c.plus_ends ? (none | all) : 0u;
        // agreeing leaders decide "plus" for any level L in [1, K]: take L = 1
        pl[2] |= nsoc & ~f2 & agree;
        need = nsoc & (f2 | ~agree);
    } else {
        need = K == 4 ? nsoc & s1 & ~s0 & ~s2 : 0u;  // count == 2
    }
    if (need) {
        const int64_t b = g & 1;
        const uint64_t key = a.keys[b * c.NP + i];
        const uint32_t base = (uint32_t)a.picks[b * c.NP + i].w + 2 + (uint32_t)(c.Dg + c.g0) + (uint32_t)(w * 32);
        const uint32_t D = (uint32_t)c.Dg;  // stream layout
        // kApplyIlp genes per iteration: independent draws interleave
        while (need) {
            int bit[kApplyIlp];
            bool have[kApplyIlp];
#pragma unroll
            for (int h = 0; h < kApplyIlp; ++h) {
                have[h] = need != 0u;
                bit[h] = have[h] ? __ffs(need) - 1 : 0;
                need &= need - 1;
            }
            uint64_t x3[kApplyIlp];
            uint32_t h3[kApplyIlp];
            bool state[kApplyIlp];
#pragma unroll
            for (int h = 0; h < kApplyIlp; ++h) {
                state[h] = !early || ((f2 >> bit[h]) & 1u);
                x3[h] = mix_pre2(key, base + (uint32_t)bit[h] + (state[h] ? 3 * D : 4 * D), c);
                h3[h] = mix_hi2(x3[h]);
            }
#pragma unroll
            for (int h = 0; h < kApplyIlp; ++h) {
                if (!have[h]) continue;
                if (state[h]) {
                    pl[2] |= ((h3[h] >> 31) == 0u ? 1u : 0u) << bit[h];  // u < 0.5
                } else {
                    uint32_t L = 0;
                    if (K == 4 && c.plus_dyadic) {
                        L = 1u + (h3[h] >> 30);  // thresholds c/4: L = 1 + floor(4u)
                    } else {
#pragma unroll
                        for (int cc = 0; cc <= K; ++cc) L += passes_hi(c.thr_plus[cc], x3[h], h3[h]) ? 0u : 1u;
                    }
                    pl[2] |= (L & 1u) << bit[h];
                    pl[3] |= ((L >> 1) & 1u) << bit[h];
                    pl[4] |= ((L >> 2) & 1u) << bit[h];
                }
            }
        }
    }
    const uint32_t word = wolf_word<K>(ld, pl, early) & valid;
    a.bits[(int64_t)a.spare_of[i] * c.W + w] = word;  // scored from the spare slot
    a.cbits[i * c.W + w] = word;                       // scored from here; multi-GPU: all-gathered
}

// ---------------------------------------------------------------- run_gwo
// gwo_reference_update (optimizer.py:302-332) with the three ranked leaders
__global__ void __launch_bounds__(kRowThreads) k_gwo_continuous(RunConsts c, const EngineState *st,
                                                                const double *__restrict__ sched, int64_t row_lo,
                                                                const int32_t *slot_of, const int32_t *spare_of,
                                                                uint8_t *__restrict__ slot_bin,
                                                                double *__restrict__ genome,
                                                                uint32_t *__restrict__ bits) {
    pdl_wait();
    const int64_t i = row_lo + blockIdx.y;
    for (int t = 0; t < 3; ++t)
        if (st->leaders[t] == i) return;
    const int64_t g = st->g;
    const double a = sched[g * QPM_SCHED_COLS + QPM_SCHED_A_NOW];
    const double two_a = 2.0 * a;
    const uint64_t key = fold_key3(c.seed, (uint64_t)g, (uint64_t)i);
    const uint64_t gD = (uint64_t)c.Dg * kGold;  // stream layout (Dg genes; this shard's gene j is g0 + j)
    const RowRef x = row_ref(c, slot_of[i], slot_bin, genome, bits);
    const RowRef L0 = row_ref(c, slot_of[st->leaders[0]], slot_bin, genome, bits);
    const RowRef L1 = row_ref(c, slot_of[st->leaders[1]], slot_bin, genome, bits);
    const RowRef L2 = row_ref(c, slot_of[st->leaders[2]], slot_bin, genome, bits);
    const int64_t out_slot = spare_of[i];
    double *out = genome + out_slot * c.Dp;
    uint32_t *bout = bits + out_slot * c.W;
    for (int64_t jb = 0; jb < c.Dp; jb += kGenesPerBlock)
#pragma unroll
    for (int it = 0; it < kGenesPerThread; ++it) {
        const int64_t j = jb + it * kRowThreads + threadIdx.x;
        bool neg = false;
        if (j < c.D) {
            const uint64_t jj = (uint64_t)(c.g0 + j);
            const double xj = x.at(j);
            const double Lm[3] = {L0.at(j), L1.at(j), L2.at(j)};
            double moved[3];
            // counter states: position p sits at key + (p + 1) GOLD, so the six
            // draws of gene jj are one product plus constant offsets k D GOLD
            const uint64_t zj = key + (jj + 1) * kGold;
#pragma unroll
            for (int m = 0; m < 3; ++m) {
                const double r1 = (double)(mix64(zj + (uint64_t)(2 * m) * gD) >> 11) * kTwoM53;
                const double r2 = (double)(mix64(zj + (uint64_t)(2 * m + 1) * gD) >> 11) * kTwoM53;
                const double av = two_a * r1 - a;
                const double cv = 2.0 * r2;
                const double dist = fabs(cv * Lm[m] - xj);
                moved[m] = Lm[m] - av * dist;
            }
            const double denom = (fabs(moved[0]) + fabs(moved[1])) + fabs(moved[2]);
            double acc = 0.0;
#pragma unroll
            for (int m = 0; m < 3; ++m) {
                const double w = denom > 0.0 ? fabs(moved[m]) / denom : 1.0 / 3.0;
                const double p = w * moved[m];
                acc = m == 0 ? p : acc + p;
            }
            if (c.divide) acc /= 3.0;
            out[j] = acc;
            neg = !(acc >= 0.0);
        }
        const uint32_t word = __ballot_sync(0xffffffffu, neg);
        if ((threadIdx.x & 31) == 0 && j < c.Dp) bout[j >> 5] = word;
    }
    if (threadIdx.x == 0) slot_bin[out_slot] = 0;
}

// ---------------------------------------------------------------- block helpers
struct Cand {
    double v;
    int32_t i;
};
// (-value, index) order; index -1 marks an empty slot (worse than anything).
// Bitwise, not short-circuit: straight-line code for the merge networks.
__device__ __forceinline__ bool better(const Cand &a, const Cand &b) {
    const bool gt = a.v > b.v, eq = a.v == b.v, lo = a.i < b.i;
    return (a.i >= 0) & ((b.i < 0) | gt | (eq & lo));
}

// top-K by (-value, index) (parexec.reduce_best), whole CTA.  (-value,
// index) is a strict total order on the elements, so the top-K set and its
// order are unique: any merge structure gives the same, exact answer.  Each
// thread keeps a sorted 4-slot list (unused slots are sentinels, index -1)
// by insertion; each warp takes the top-k of its lanes' lists by k argmax
// rounds over the list heads, and warp 0 does the same over the warps' lists.
constexpr int kTopSlots = 4;

__device__ __forceinline__ void cswap(Cand &a, Cand &b) {  // a := better of the two
    const bool sw = better(b, a);
    const Cand x = a, y = b;
    a.v = sw ? y.v : x.v;
    a.i = sw ? y.i : x.i;
    b.v = sw ? x.v : y.v;
    b.i = sw ? x.i : y.i;
}

__device__ __forceinline__ void topk_insert(Cand (&L)[kTopSlots], Cand e) {
#pragma unroll
    for (int t = 0; t < kTopSlots; ++t) cswap(L[t], e);
}

// top-k (k <= 4, warp-uniform) of the union of the lanes' sorted lists: k
// rounds of a warp argmax over the list heads (xor butterfly, so every lane
// sees the winner); the lane whose head won pops it.  About half the
// instructions of merging whole 4-lists at every butterfly level, which
// dominated the single-CTA selection kernels (ncu: ~700 warp instructions
// per warp, issue-bound on one SM).
__device__ __forceinline__ void topk_warp_rounds(Cand (&L)[kTopSlots], int k, Cand (&R)[kTopSlots]) {
#pragma unroll
    for (int t = 0; t < kTopSlots; ++t) {
        R[t] = Cand{0.0, -1};
        if (t >= k) continue;
        Cand b = L[0];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            Cand o;
            o.v = __shfl_xor_sync(0xffffffffu, b.v, off);
            o.i = __shfl_xor_sync(0xffffffffu, b.i, off);
            const bool tk = better(o, b);
            b.v = tk ? o.v : b.v;
            b.i = tk ? o.i : b.i;
        }
        R[t] = b;
        if (L[0].i == b.i) {  // indices are unique: this lane's head won (or both are sentinels)
            L[0] = L[1];
            L[1] = L[2];
            L[2] = L[3];
            L[3] = Cand{0.0, -1};
        }
    }
}

// the CTA's top-k (k <= 4) of the per-thread lists into out[0..k); every
// thread must call it
__device__ void block_topk_lists(Cand (&L)[kTopSlots], int k, int32_t *out) {
    __shared__ double s_v[32][kTopSlots];
    __shared__ int32_t s_i[32][kTopSlots];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nwarps = (int)(blockDim.x >> 5);
    Cand R[kTopSlots];
    topk_warp_rounds(L, k, R);
    if (lane == 0) {
#pragma unroll
        for (int t = 0; t < kTopSlots; ++t) {
            s_v[warp][t] = R[t].v;
            s_i[warp][t] = R[t].i;
        }
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int t = 0; t < kTopSlots; ++t) L[t] = lane < nwarps ? Cand{s_v[lane][t], s_i[lane][t]} : Cand{0.0, -1};
        topk_warp_rounds(L, k, R);
        if (lane == 0) {
#pragma unroll
            for (int t = 0; t < kTopSlots; ++t)
                if (t < k) out[t] = R[t].i;
        }
    }
    __syncthreads();
}

__device__ void block_topk_k(const double *vals, int64_t n, int k, int32_t *out) {
    Cand L[kTopSlots];
#pragma unroll
    for (int t = 0; t < kTopSlots; ++t) L[t] = {0.0, -1};
    // the loads of kBatch strides first, then the inserts: one L2 round trip
    // per batch instead of one per element (C2: 4 elements per thread)
    constexpr int kBatch = 4;
    for (int64_t i0 = threadIdx.x; i0 < n; i0 += (int64_t)kBatch * blockDim.x) {
        double v[kBatch];
#pragma unroll
        for (int u = 0; u < kBatch; ++u) {
            const int64_t i = i0 + (int64_t)u * blockDim.x;
            v[u] = i < n ? __ldcg(vals + i) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kBatch; ++u) {
            const int64_t i = i0 + (int64_t)u * blockDim.x;
            if (i < n) topk_insert(L, Cand{v[u], (int32_t)i});
        }
    }
    block_topk_lists(L, k, out);
}

// numpy pairwise sum (np.add.reduce, pairwise.c) of v[0..n) over the
// host-built split tree.  Tree structure and node values live in shared
// memory (ts).  A leaf (<= 128 elements) is summed by 8 lanes: lane k owns
// numpy's accumulator r_k (elements k, k+8, ... in order), the eight are
// combined as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) by xor shuffles, and the
// tail (n % 8 elements) is added in order; internal nodes follow by height.
struct TreeSmem {
    int32_t *leaf_off, *kid, *lvl;
    double *val;
};

// SQDEV: the sum of (v_i - m)^2 instead, each term formed as numpy's
// `x = arr - mean; x = x * x` forms it (no separate squared-deviation pass)
template <bool SQDEV = false>
__device__ double block_pairwise(const double *v, const RunConsts &c, const TreeSmem &ts, double m = 0.0) {
    const int lane = threadIdx.x & 31, sub = lane & 7;
    const int groups = (int)(blockDim.x >> 3);
    for (int base = (int)(threadIdx.x >> 3) - (lane >> 3); base < c.n_leaf; base += groups) {
        const int l = base + (lane >> 3);  // warp-uniform trip count: shuffles see all lanes
        const bool ok = l < c.n_leaf;
        const int off = ok ? ts.leaf_off[l] : 0;
        const int len = ok ? ts.leaf_off[l + 1] - off : 0;
        const double *a = v + off;
        const int mlen = len - len % 8;
        double r = 0.0;
        if (len >= 8) {
            // a leaf has <= 128 elements, so <= 16 per accumulator: every
            // shared-memory load is issued first, then the adds run in numpy's
            // order (a dependent chain of adds instead of load-add round trips)
            double x[16];
#pragma unroll
            for (int t = 0; t < 16; ++t) {
                x[t] = sub + 8 * t < mlen ? a[sub + 8 * t] : 0.0;
                if (SQDEV) {
                    const double d = x[t] - m;
                    x[t] = d * d;
                }
            }
            r = x[0];
#pragma unroll
            for (int t = 1; t < 16; ++t)
                if (sub + 8 * t < mlen) r += x[t];
        }
        r += __shfl_xor_sync(0xffffffffu, r, 1);
        r += __shfl_xor_sync(0xffffffffu, r, 2);
        r += __shfl_xor_sync(0xffffffffu, r, 4);
        if (ok && sub == 0) {
            double res = len >= 8 ? r : 0.0;
            for (int i = mlen; i < len; ++i) {
                double t = a[i];
                if (SQDEV) {
                    const double d = t - m;
                    t = d * d;
                }
                res += t;
            }
            ts.val[l] = res;
        }
    }
    __syncthreads();
    if (c.n_leaf <= 64) {  // few internal nodes: one warp, warp-level barriers
        if (threadIdx.x < 32) {
            for (int h = 0; h < c.n_levels; ++h) {
                for (int t = ts.lvl[h] + (int)threadIdx.x; t < ts.lvl[h + 1]; t += 32)
                    ts.val[c.n_leaf + t] = ts.val[ts.kid[2 * t]] + ts.val[ts.kid[2 * t + 1]];
                __syncwarp();
            }
        }
    } else {
        for (int h = 0; h < c.n_levels; ++h) {
            for (int t = ts.lvl[h] + (int)threadIdx.x; t < ts.lvl[h + 1]; t += blockDim.x)
                ts.val[c.n_leaf + t] = ts.val[ts.kid[2 * t]] + ts.val[ts.kid[2 * t + 1]];
            __syncthreads();
        }
    }
    __syncthreads();
    const double r = ts.val[c.n_leaf > 1 ? 2 * c.n_leaf - 2 : 0];
    __syncthreads();
    return r;
}

// ---------------------------------------------------------------- select + top-k
// de_select over all individuals (strict >, ties keep the target), then
// rank_leaders (optimizer.py:437-444).  One CTA.
// Large populations use several CTAs (kTopkMaxCtas at most): each selects a
// contiguous slice and publishes its top-k indices; the last CTA to finish
// (arrival counter, reset by it for the next launch) merges the lists by
// argmax rounds over the lists' heads, values re-read from fit.  (-value,
// index) is a strict total order, so the leaders are the same for any split.
constexpr int kTopkMaxCtas = 32;
struct TopkScratch {
    int32_t *idx;   // [kTopkMaxCtas][kTopSlots]
    unsigned *cnt;  // arrival counter, zero between launches
};

__global__ void __launch_bounds__(kCtaThreads) k_select_topk(RunConsts c, EngineState *__restrict__ st,
                                                             const double *cand,
                                                             double *__restrict__ fit, int32_t *__restrict__ slot_of,
                                                             int32_t *__restrict__ spare_of, TopkScratch ts,
                                                             uint32_t *__restrict__ slot_tag) {
    QTRACE(3);
    pdl_wait();
    QTRACE_STARTED();
    Cand L[kTopSlots];
#pragma unroll
    for (int t = 0; t < kTopSlots; ++t) L[t] = {0.0, -1};
    const int64_t per = (c.NP + gridDim.x - 1) / gridDim.x;
    const int64_t lo = blockIdx.x * per, hi = min(c.NP, lo + per);
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        // the slot ids are loaded with the fitness values (one L2 round trip,
        // not two) and written back only on acceptance
        const double f = cand[i];
        double v = fit[i];
        const int32_t a = slot_of[i], b = spare_of[i];
        if (f > v) {
            slot_of[i] = b;
            spare_of[i] = a;
            if (slot_tag) slot_tag[i] = (uint32_t)b;  // a DE trial: an f64 row
            fit[i] = f;
            v = f;
        }
        topk_insert(L, Cand{v, (int32_t)i});  // the selected value, straight from registers
    }
    if (gridDim.x == 1) {
        block_topk_lists(L, c.k, st->leaders);
        return;
    }
    block_topk_lists(L, c.k, ts.idx + blockIdx.x * kTopSlots);
    __shared__ unsigned s_last;
    __threadfence();  // this CTA's selection writes and list, before its arrival
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(ts.cnt, 1u) + 1u == gridDim.x;
    __syncthreads();
    if (!s_last || threadIdx.x >= 32) return;
    __threadfence();
    const int lane = threadIdx.x;
#pragma unroll
    for (int t = 0; t < kTopSlots; ++t) {
        const int32_t id = lane < (int)gridDim.x && t < c.k ? __ldcg(ts.idx + lane * kTopSlots + t) : -1;
        L[t] = Cand{id >= 0 ? __ldcg(fit + id) : 0.0, id};
    }
    Cand R[kTopSlots];
    topk_warp_rounds(L, c.k, R);
    if (lane == 0) {
#pragma unroll
        for (int t = 0; t < kTopSlots; ++t)
            if (t < c.k) st->leaders[t] = R[t].i;
        *ts.cnt = 0u;
    }
}

__global__ void __launch_bounds__(kCtaThreads) k_topk_leaders(RunConsts c, EngineState *__restrict__ st,
                                                              const double *fit, int k) {
    pdl_wait();
    block_topk_k(fit, c.NP, k, st->leaders);
}

// ---------------------------------------------------------------- select + stats
// mode 0: DE selection of everyone (run_de); 1: wolf selection of the
// non-leaders, accepted slots become +/-1 rows (run_hybrid); 2: unconditional
// replacement of the non-leaders (run_gwo); 3: none (init).  Then np.max /
// np.mean / np.std, the convergence window and adaptive_f_update
// (optimizer.py:277-299, 469-485), or run_gwo's a-row and best-ever tracking
// (optimizer.py:586-589), and the trace row.  One CTA.
// the statistics' dynamic shared memory: [fit (n), squared deviations (n)]
// when n fits, then the pairwise-sum tree (values, leaf offsets, children, levels)
__device__ __forceinline__ TreeSmem stats_tree_smem(const RunConsts &c, double *s_dyn) {
    const bool on_chip = c.NP <= kStatsSmemMaxNP;
    TreeSmem ts;
    ts.val = s_dyn + (on_chip ? 2 * c.NP : 0);
    ts.leaf_off = reinterpret_cast<int32_t *>(ts.val + 2 * c.n_leaf);
    ts.kid = ts.leaf_off + c.n_leaf + 1;
    ts.lvl = ts.kid + 2 * c.n_leaf;
    return ts;
}
// the tree is the engine's constant: staged before waiting on the predecessor
__device__ __forceinline__ void stats_tree_stage(const RunConsts &c, const SumTree &tr, const SumTreeInline &tri,
                                                 const TreeSmem &ts) {
    if (tri.n) {
        const int nl = c.n_leaf + 1, nk = 2 * (c.n_leaf - 1);
        for (int t = threadIdx.x; t < tri.n; t += blockDim.x) {
            const int32_t v = tri.v[t];
            if (t < nl)
                ts.leaf_off[t] = v;
            else if (t < nl + nk)
                ts.kid[t - nl] = v;
            else
                ts.lvl[t - nl - nk] = v;
        }
    } else {
        for (int t = threadIdx.x; t <= c.n_leaf; t += blockDim.x) ts.leaf_off[t] = tr.leaf_off[t];
        for (int t = threadIdx.x; t < 2 * (c.n_leaf - 1); t += blockDim.x) ts.kid[t] = tr.kid[t];
        for (int t = threadIdx.x; t <= c.n_levels; t += blockDim.x) ts.lvl[t] = tr.lvl[t];
    }
}

__device__ __forceinline__ void select_stats_body(const RunConsts &c, int mode, EngineState *__restrict__ st,
                                                  const double *__restrict__ sched, const double *cand,
                                                  double *__restrict__ fit, int32_t *__restrict__ slot_of,
                                                  int32_t *__restrict__ spare_of, uint8_t *__restrict__ slot_bin,
                                                  double *__restrict__ scratch, const SumTree &tr,
                                                  double *__restrict__ trace, const SumTreeInline &tri, bool wait,
                                                  uint32_t *__restrict__ slot_tag, bool staged = false) {
    const int64_t n = c.NP;
    // dynamic shared memory: [fit (n), squared deviations (n)] when n fits,
    // then the pairwise-sum tree (values, leaf offsets, children, levels)
    extern __shared__ double s_dyn[];
    const bool on_chip = n <= kStatsSmemMaxNP;
    double *fv = on_chip ? s_dyn : fit;
    const TreeSmem ts = stats_tree_smem(c, s_dyn);
    if (!staged) stats_tree_stage(c, tr, tri, ts);  // (the fused caller stages it at its entry)
    if (wait) pdl_wait();
    // the state is copied to shared memory for the serial tail: its words are
    // loaded here and stored after the fitness loads below are in flight
    __shared__ EngineState s_state;
    constexpr int kStateWords = (int)(sizeof(EngineState) / 4);
    const uint32_t *st_src = reinterpret_cast<const uint32_t *>(st);
    uint32_t st_w0 = (int)threadIdx.x < kStateWords ? st_src[threadIdx.x] : 0u;
    if (mode == 3 && threadIdx.x == 0) QSTAMP_ID(5, 4);
    int32_t lead[kMaxLeaders];
#pragma unroll
    for (int t = 0; t < kMaxLeaders; ++t) lead[t] = (mode == 1 || mode == 2) && t < c.k ? st->leaders[t] : -1;
    // selection; every thread keeps its elements' final values for the max/min
    double mx = -INFINITY, mn = INFINITY;
    int64_t amx = n;
    constexpr int kBatch = 4;  // loads of kBatch strides issued together (one L2 round trip per batch)
    for (int64_t i0 = threadIdx.x; i0 < n; i0 += (int64_t)kBatch * blockDim.x) {
        double vb[kBatch];
#pragma unroll
        for (int u = 0; u < kBatch; ++u) {
            const int64_t i = i0 + (int64_t)u * blockDim.x;
            vb[u] = i < n ? __ldcg(fit + i) : 0.0;  // (coherent: a fused caller's other CTAs wrote it)
        }
        if (i0 == (int64_t)threadIdx.x) {  // first batch: the state words, now that the loads are issued
            uint32_t *dst = reinterpret_cast<uint32_t *>(&s_state);
            if ((int)threadIdx.x < kStateWords) dst[threadIdx.x] = st_w0;
            for (int t = (int)threadIdx.x + (int)blockDim.x; t < kStateWords; t += blockDim.x) dst[t] = st_src[t];
        }
#pragma unroll
        for (int u = 0; u < kBatch; ++u) {
            const int64_t i = i0 + (int64_t)u * blockDim.x;
            if (i >= n) break;
            double v = vb[u];
            if (mode != 3) {
                bool is_leader = false;
#pragma unroll
                for (int t = 0; t < kMaxLeaders; ++t) is_leader |= lead[t] == i;
                const double f = cand[i];
                const int32_t a = slot_of[i], b = spare_of[i];
                if (!is_leader && (mode == 2 || f > v)) {
                    slot_of[i] = b;
                    spare_of[i] = a;
                    fit[i] = f;
                    if (mode == 1) slot_bin[b] = 1;
                    if (slot_tag) slot_tag[i] = (uint32_t)b | (mode == 1 ? kBinTag : 0u);
                    v = f;
                }
            }
            if (on_chip) fv[i] = v;
            if (v > mx || (v == mx && i < amx)) {  // max, lowest index on ties
                mx = v;
                amx = i;
            }
            mn = v < mn ? v : mn;
        }
    }
    if ((int64_t)threadIdx.x >= n) {  // (no batch ran in this thread)
        uint32_t *dst = reinterpret_cast<uint32_t *>(&s_state);
        if ((int)threadIdx.x < kStateWords) dst[threadIdx.x] = st_w0;
        for (int t = (int)threadIdx.x + (int)blockDim.x; t < kStateWords; t += blockDim.x) dst[t] = st_src[t];
    }
    for (int off = 16; off > 0; off >>= 1) {
        const double omx = __shfl_down_sync(0xffffffffu, mx, off);
        const int64_t oam = __shfl_down_sync(0xffffffffu, amx, off);
        const double omn = __shfl_down_sync(0xffffffffu, mn, off);
        if (omx > mx || (omx == mx && oam < amx)) {
            mx = omx;
            amx = oam;
        }
        mn = omn < mn ? omn : mn;
    }
    __shared__ double s_mx[kCtaThreads / 32], s_mn[kCtaThreads / 32];
    __shared__ int64_t s_am[kCtaThreads / 32];
    const int lane = threadIdx.x & 31, nw = (int)(blockDim.x >> 5);
    if (lane == 0) {
        s_mx[threadIdx.x >> 5] = mx;
        s_mn[threadIdx.x >> 5] = mn;
        s_am[threadIdx.x >> 5] = amx;
    }
    __syncthreads();  // also publishes fv (and, without on-chip staging, fit)
    mx = lane < nw ? s_mx[lane] : -INFINITY;
    mn = lane < nw ? s_mn[lane] : INFINITY;
    amx = lane < nw ? s_am[lane] : n;
    for (int off = 16; off > 0; off >>= 1) {  // every warp reduces the 32 partials itself
        const double omx = __shfl_down_sync(0xffffffffu, mx, off);
        const int64_t oam = __shfl_down_sync(0xffffffffu, amx, off);
        const double omn = __shfl_down_sync(0xffffffffu, mn, off);
        if (omx > mx || (omx == mx && oam < amx)) {
            mx = omx;
            amx = oam;
        }
        mn = omn < mn ? omn : mn;
    }
    mx = __shfl_sync(0xffffffffu, mx, 0);
    mn = __shfl_sync(0xffffffffu, mn, 0);
    amx = __shfl_sync(0xffffffffu, amx, 0);
    if (mode == 3 && threadIdx.x == 0) QSTAMP_ID(5, 5);
    // x / n: by an exact reciprocal multiply when n is a power of two (the
    // same correctly rounded value, without the division sequence)
    const bool n_pow2 = (n & (n - 1)) == 0;
    const double inv_n = 1.0 / (double)n;
    const double sum = block_pairwise(fv, c, ts);
    const double mean = n_pow2 ? sum * inv_n : sum / (double)n;
    if (mode == 3 && threadIdx.x == 0) QSTAMP_ID(5, 6);
    const double ssq = block_pairwise<true>(fv, c, ts, mean);  // (fv is published: block_pairwise ends in a barrier)
    const double var = n_pow2 ? ssq * inv_n : ssq / (double)n;
    if (threadIdx.x != 0) return;
    if (mode == 3) QSTAMP_ID(5, 7);
    // serial tail on the shared-memory copy of the state (fetched at entry);
    // only the fields this kernel owns are written back (g_plan belongs to
    // the planner stream)
    const EngineState &ss = s_state;
    const double sd = sqrt(var);
    const int64_t g = ss.g;
    double *row = trace + g * 5;
    row[0] = (double)g;
    row[1] = mx;
    row[2] = mean;
    row[4] = sd;
    if (c.algorithm == QPM_ALGO_GWO) {
        row[3] = g == 0 ? c.gwo_a0 : sched[g * QPM_SCHED_COLS + QPM_SCHED_A_NOW];
        if (g == 0 || mx > ss.best_fit) {
            st->best_fit = mx;
            st->best_idx = (int32_t)amx;
            st->best_flag = 1;
        } else {
            st->best_flag = 0;
        }
    } else if (g == 0) {
        st->baseline_std = sd;
        st->F = c.f_max;
        st->best_prev = mx;
        st->win_len = 0;
        row[3] = c.f_max;
    } else {
        // convergence window: deque(maxlen=conv_window) of best_now > best_prev
        const int cap = c.conv_window;
        int len = ss.win_len;
        const uint8_t improved = mx > ss.best_prev ? 1 : 0;
        int cnt = 0;
        if (len < cap) {
            for (int t = 0; t < len; ++t) cnt += ss.win[t];
            st->win[len] = improved;
            ++len;
        } else {
            for (int t = 1; t < cap; ++t) {
                st->win[t - 1] = ss.win[t];
                cnt += ss.win[t];
            }
            st->win[cap - 1] = improved;
        }
        cnt += improved;
        st->win_len = len;
        st->best_prev = mx;
        const double conv = len ? (double)cnt / (double)len : 1.0;
        const double *sg = sched + g * QPM_SCHED_COLS;
        const double base = ss.baseline_std;
        double f = sg[QPM_SCHED_F_ENV];
        if (c.adaptive) {
            const double tl = c.theta_low_frac * base;
            const double th = c.theta_high_frac * base;
            const double rt = c.range_trigger_frac * base;
            if (sd < tl || conv < c.conv_threshold) f *= c.explore_boost;
            if (sd > th || (mx - mn) < rt) f *= c.exploit_factor;
        }
        f *= sg[QPM_SCHED_DECAY];
        const double lo = c.f_min > f ? c.f_min : f;  // max(f, f_min)
        f = c.f_max < lo ? c.f_max : lo;              // min(., f_max)
        st->F = f;
        row[3] = f;
    }
    st->g = g + 1;
}

__global__ void __launch_bounds__(kCtaThreads) k_select_stats(RunConsts c, int mode, EngineState *__restrict__ st,
                                                              const double *__restrict__ sched,
                                                              const double *cand,
                                                              double *__restrict__ fit, int32_t *__restrict__ slot_of,
                                                              int32_t *__restrict__ spare_of,
                                                              uint8_t *__restrict__ slot_bin,
                                                              double *__restrict__ scratch, SumTree tr,
                                                              double *__restrict__ trace, SumTreeInline tri,
                                                              uint32_t *__restrict__ slot_tag) {
    QTRACE(5);
    select_stats_body(c, mode, st, sched, cand, fit, slot_of, spare_of, slot_bin, scratch, tr, trace, tri, true,
                      slot_tag);
}

// Fused fitness finish + selection (run_hybrid): one warp per row stitches its
// segment partials (finish_row, the k_fit_finish arithmetic), lane 0 selects
// the row (strict >, ties keep the target; MODE 1: leaders stay), and the
// last CTA to finish (arrival counter, reset by it) runs the whole-population
// part: MODE 0 the top-k leaders, MODE 1 np.max/mean/std, window, F and the
// trace row (select_stats_body with the selection already done).  Saves the
// separate finish launch and moves the selection onto every SM.
#ifndef QPM_FS_THREADS
#define QPM_FS_THREADS 256
#endif
#ifndef QPM_FS_THREADS1
#define QPM_FS_THREADS1 QPM_FS_THREADS
#endif
#ifndef QPM_FS_WIDE
#define QPM_FS_WIDE 1  // fused finish/selection for NP > 2048 too (1024-thread CTAs)
#endif
// fused finish + selection CTA: <0> (leaders) and <1> (statistics)
template <int MODE>
__host__ __device__ constexpr int fs_threads() { return MODE == 0 ? QPM_FS_THREADS : QPM_FS_THREADS1; }
// THREADS: fs_threads<MODE>() (NP <= 2048), or kCtaThreads for large
// populations, whose last CTA then has the single-CTA kernels' width
template <int MODE, int THREADS = fs_threads<MODE>()>
__global__ void __launch_bounds__(THREADS) k_finish_select(RunConsts c, FinishArgs f, EngineState *__restrict__ st,
                                                               const double *__restrict__ sched, double *cand,
                                                               double *__restrict__ fit, int32_t *__restrict__ slot_of,
                                                               int32_t *__restrict__ spare_of,
                                                               uint8_t *__restrict__ slot_bin,
                                                               double *__restrict__ scratch, SumTree tr,
                                                               double *__restrict__ trace, SumTreeInline tri,
                                                               unsigned *cnt, uint32_t *__restrict__ slot_tag) {
    QTRACE(MODE == 0 ? 3 : 5);
    extern __shared__ double s_dyn[];
    if (MODE == 1) stats_tree_stage(c, tr, tri, stats_tree_smem(c, s_dyn));  // every CTA: any may be the last
    pdl_wait();
    pdl_trigger<4>();
    QTRACE_STARTED();
    QSTAMP(0);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t r = (int64_t)blockIdx.x * (THREADS / 32) + warp;
    if (r < c.NP) {  // warp-uniform
        const double g = finish_row(f, r, lane);
        if (lane == 0) {
            cand[r] = g;
            bool take = g > __ldcg(fit + r);
            if (MODE == 1) {
#pragma unroll
                for (int t = 0; t < kMaxLeaders; ++t) take &= !(t < c.k && st->leaders[t] == r);
            }
            if (take) {
                const int32_t a = slot_of[r], b = spare_of[r];
                slot_of[r] = b;
                spare_of[r] = a;
                fit[r] = g;
                if (MODE == 1) slot_bin[b] = 1;
                if (slot_tag) slot_tag[r] = (uint32_t)b | (MODE == 1 ? kBinTag : 0u);
            }
        }
    }
    // arrival: the barrier orders this CTA's selections before thread 0's
    // acquire-release add (cumulative at gpu scope); the last CTA's thread 0
    // acquires every other CTA's, and its barrier passes that on to the CTA
    // (the grid-synchronisation pattern, one fence-free atomic per CTA)
    __shared__ unsigned s_last;
    __syncthreads();
    QSTAMP(1);
    if (threadIdx.x == 0) {
        unsigned prev;
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(cnt) : "memory");
        s_last = prev + 1u == gridDim.x;
    }
    __syncthreads();
    if (!s_last) return;
    if (threadIdx.x == 0) QSTAMP_ANY(2);
    if (MODE == 0)
        block_topk_k(fit, c.NP, c.k, st->leaders);
    else
        select_stats_body(c, 3, st, sched, cand, fit, slot_of, spare_of, slot_bin, scratch, tr, trace, tri, false,
                          nullptr, true);
    if (threadIdx.x == 0) QSTAMP_ANY(3);
    if (threadIdx.x == 0) *cnt = 0u;  // ready for the next launch (stream-ordered)
}

// best row -> result buffer (when flagged), expanding +/-1 slots from bits
__global__ void k_copy_best(RunConsts c, const EngineState *__restrict__ st, const int32_t *__restrict__ slot_of,
                            const uint8_t *__restrict__ slot_bin, const double *__restrict__ genome,
                            const uint32_t *__restrict__ bits, double *__restrict__ best_genome,
                            uint32_t *__restrict__ best_bits) {
    if (!st->best_flag) return;
    const int64_t slot = slot_of[st->best_idx];
    const RowRef r = row_ref(c, slot, slot_bin, genome, bits);
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < c.Dp; j += (int64_t)gridDim.x * blockDim.x) {
        best_genome[j] = j < c.D ? r.at(j) : 0.0;
        if (j < c.W) best_bits[j] = bits[slot * c.W + j];
    }
}

__global__ void k_finalize_best(RunConsts c, EngineState *st, const double *fit) {
    // rank_leaders(pop, 1): highest fitness, lowest index on ties
    __shared__ int32_t top[kMaxLeaders];
    block_topk_k(fit, c.NP, 1, top);
    if (threadIdx.x == 0) {
        st->best_idx = top[0];
        st->best_fit = __ldcg(fit + top[0]);  // read back with the state (one copy)
        st->best_flag = 1;
    }
}

__global__ void k_reset_flag(EngineState *st) { st->best_flag = 0; }

// ---------------------------------------------------------------- checkpoint
// Checkpoint / resume (a checkpoint is (g, F, window,
// baseline_std, genome, fitness, best_prev); the counter RNG has no state).
// The current individuals are gathered in individual order (±1 rows expanded
// to f64, with their flags) and scattered back into slots 0..NP-1 on restore:
// slot numbers carry no meaning, so the resumed run is bit-identical.
__global__ void k_gather_rows(RunConsts c, const int32_t *slot_of, const uint8_t *slot_bin, const double *genome,
                              const uint32_t *bits, double *out_g, uint32_t *out_b, uint8_t *out_bin) {
    const int64_t i = blockIdx.y;
    const int64_t slot = slot_of[i];
    const RowRef r = row_ref(c, slot, slot_bin, genome, bits);
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < c.Dp; j += (int64_t)gridDim.x * blockDim.x) {
        out_g[i * c.Dp + j] = j < c.D ? r.at((int)j) : 0.0;
        if (j < c.W) out_b[i * c.W + j] = bits[slot * c.W + j];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) out_bin[i] = slot_bin[slot];
}

__global__ void k_scatter_rows(RunConsts c, const double *in_g, const uint32_t *in_b, const uint8_t *in_bin,
                               int32_t *slot_of, int32_t *spare_of, uint32_t *slot_tag, uint8_t *slot_bin,
                               double *genome, uint32_t *bits) {
    const int64_t i = blockIdx.y;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < c.Dp; j += (int64_t)gridDim.x * blockDim.x) {
        genome[i * c.Dp + j] = in_g[i * c.Dp + j];
        if (j < c.W) bits[i * c.W + j] = in_b[i * c.W + j];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        const uint8_t bin = in_bin[i];
        slot_of[i] = (int32_t)i;
        spare_of[i] = (int32_t)(c.NP + i);
        slot_bin[i] = bin;
        slot_bin[c.NP + i] = 0;
        if (slot_tag) slot_tag[i] = (uint32_t)i | (bin ? kBinTag : 0u);
    }
}

struct CkptHeader {
    char magic[8];  // "QPMCKPT1"
    int32_t version, algorithm, fitness_mode, rank;
    int32_t world, pad;
    int64_t NP, D, W, G, seed, g0, g_done;
};

// ---------------------------------------------------------------- state checks
// QPM_CHECKS builds (libqpm_b200_checks.so, tests/test_gpu_checks.py): after
// every generation one CTA verifies the engine's invariants and records the
// first violation in a device word pair (the pool runs no compute-sanitizer;
// these are the bounds checks and asserts the engine carries instead):
//   1 slot ids in [0, 2 NP) and {slot_of} u {spare_of} a permutation of them
//   2 the next generation's DE picks r1, r2, r3 distinct, != i, in [0, NP);
//     m >= 3; j_rand in [0, Dg)
//   4 leaders distinct and in [0, NP) (hybrid, gwo)
//   8 every fitness finite (NaN / inf would break the strict-> selection)
//  16 the trace row just written finite and its generation number right
//  32 the generation counter g_plan of the planner equals g + 1 (hybrid, de)
#ifndef QPM_CHECKS
#define QPM_CHECKS 0
#endif
struct CheckArgs {
    const EngineState *st;
    const int32_t *slot_of, *spare_of;
    const int4 *picks;
    const int32_t *jrand;
    const double *fit, *trace;
    unsigned *err;  // [0] violation bits, [1] first detail: code << 24 | index
};
__device__ __forceinline__ void check_fail(unsigned *err, unsigned code, unsigned idx) {
    atomicOr(err, code);
    atomicCAS(err + 1, 0u, (code << 24) | (idx & 0xFFFFFFu));
}
//  64 a candidate's fitness differs from a recomputation of the same
//     candidate rows after the fact (the scan / finish saw inconsistent data)
__global__ void k_check_fitness(const double *cand, const double *again, int64_t n, unsigned *err) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n && !(__double_as_longlong(cand[i]) == __double_as_longlong(again[i]))) check_fail(err, 64u, (unsigned)i);
}
__global__ void __launch_bounds__(kCtaThreads) k_check_state(RunConsts c, CheckArgs a) {
    extern __shared__ uint32_t s_seen[];  // 2 NP bits
    const int64_t NP = c.NP, nw = (2 * NP + 31) / 32;
    for (int64_t w = threadIdx.x; w < nw; w += blockDim.x) s_seen[w] = 0u;
    __syncthreads();
    const int64_t g = a.st->g;  // the generation computed next
    for (int64_t i = threadIdx.x; i < NP; i += blockDim.x) {
        const int32_t sl[2] = {a.slot_of[i], a.spare_of[i]};
        for (int t = 0; t < 2; ++t) {
            if (sl[t] < 0 || sl[t] >= 2 * NP) {
                check_fail(a.err, 1u, (unsigned)i);
                continue;
            }
            const uint32_t bit = 1u << (sl[t] & 31);
            if (atomicOr(&s_seen[sl[t] >> 5], bit) & bit) check_fail(a.err, 1u, (unsigned)i);
        }
        if (!isfinite(a.fit[i])) check_fail(a.err, 8u, (unsigned)i);
        if (c.algorithm != QPM_ALGO_GWO && g <= c.G) {
            const int4 pk = a.picks[(g & 1) * NP + i];
            const int32_t jr = a.jrand[(g & 1) * NP + i];
            const bool ok = pk.x >= 0 && pk.x < NP && pk.y >= 0 && pk.y < NP && pk.z >= 0 && pk.z < NP &&
                            pk.x != i && pk.y != i && pk.z != i && pk.x != pk.y && pk.x != pk.z && pk.y != pk.z &&
                            pk.w >= 3 && jr >= 0 && jr < c.Dg;
            if (!ok) check_fail(a.err, 2u, (unsigned)i);
        }
    }
    __syncthreads();
    for (int64_t w = threadIdx.x; w < nw; w += blockDim.x) {
        const int64_t lo = w * 32, n = 2 * NP - lo < 32 ? 2 * NP - lo : 32;
        const uint32_t want = n == 32 ? 0xffffffffu : ((1u << n) - 1u);
        if (s_seen[w] != want) check_fail(a.err, 1u, (unsigned)lo);
    }
    if (threadIdx.x == 0) {
        if (c.algorithm != QPM_ALGO_DE) {
            const int k = c.algorithm == QPM_ALGO_GWO ? 3 : c.k;
            for (int t = 0; t < k; ++t) {
                const int32_t l = a.st->leaders[t];
                bool ok = l >= 0 && l < NP;
                for (int u = 0; u < t; ++u) ok &= a.st->leaders[u] != l;
                if (!ok && g > 1) check_fail(a.err, 4u, (unsigned)t);
            }
        }
        const double *row = a.trace + (g - 1) * 5;
        bool ok = g >= 1 && row[0] == (double)(g - 1);
        for (int t = 1; t < 5; ++t) ok &= isfinite(row[t]);
        if (!ok) check_fail(a.err, 16u, (unsigned)g);
        if (c.algorithm != QPM_ALGO_GWO && g <= c.G && a.st->g_plan != g + 1) check_fail(a.err, 32u, (unsigned)g);
    }
}

// ---------------------------------------------------------------- engine
struct Engine {
    Problem *prob = nullptr;
    FitScratch fs;  // this engine's fitness scratch (engines may share a problem)
    qpm_run_params P{};
    RunConsts c{};
    cudaStream_t stream = nullptr;
    double *genome = nullptr;
    uint32_t *bits = nullptr;
    uint8_t *slot_bin = nullptr;
    uint32_t *planes = nullptr;  // [2][NP][W][kPlanes] by generation parity (kPlanes = 4)
    uint32_t *cbits = nullptr;   // [NP][W] wolf candidates staged for exchange
    GenThr *gthr = nullptr;
    cudaStream_t side = nullptr;  // low-priority planner stream
    // column shard of this engine (multi-GPU): genes [c.g0, c.g0 + c.D) of
    // every individual = the fitness segments [seg_lo, seg_lo + seg_n) of the
    // problem = its stitch super-blocks owned by this rank (qpm_finish.cuh);
    // one GPU: rank 0 of 1, all of it
    int rank = 0, world = 1;
    int seg_lo = 0, seg_n = 0;
    qpm_problem *lprob = nullptr;  // the shard's columns of the problem (world > 1, owned)
    int SB_slot = 1;               // super-block partials per rank slot in gpart
    double *gpart = nullptr;       // [world][n_wl][NP][SB_slot][6] all-gathered super-block partials (sharded)
    double *ggains = nullptr;      // [NP][n_wl] finish scratch (world > 1)
    void *comm = nullptr;          // ncclComm_t
    // the sharded flow (scan, all-gather, finish): several ranks, or one rank
    // with a communicator (exercises the collective path on one GPU)
    bool sharded() const { return world > 1 || comm != nullptr; }
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    int32_t *slot_of = nullptr, *spare_of = nullptr, *jrand = nullptr;
    double *fit = nullptr, *cand = nullptr, *scratch = nullptr;
    int32_t *tree_i = nullptr;
    double *tree_v = nullptr;
    SumTree tree{};
    SumTreeInline tree_inline{};
    uint64_t *keys = nullptr;
    int4 *picks = nullptr;
    double *sched = nullptr, *trace = nullptr;
    EngineState *st = nullptr;
    double *best_genome = nullptr;
    uint32_t *best_bits = nullptr;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    // QPM_GRAPH_GENS > 1: also a graph of that many generations back to back,
    // whose later generations start with a programmatic launch of the trial
    int graph_gens = 10;  // measured: 118.5 -> 117.3 us per C2 generation, alternating A/B
    cudaGraph_t graph_k = nullptr;
    cudaGraphExec_t exec_k = nullptr;
    bool pdl_trial = false;  // set while capturing generations 2.. of such a graph
    int launches = 0;
    int plan_grid = 148;       // k_plan_wolf CTAs (QPM_PLAN_CTAS)
    bool plan_after_trial = false;  // fork the planner after k_de_trial (QPM_PLAN_FORK=trial)
    bool wolf_in_planner = false;   // wolf planes on the side stream (QPM_WOLF=planner)
    bool wolf_mixed = false;        // wolf planes in separate CTAs of the trial kernel (QPM_WOLF=mixed)
    bool wolf_side = false;         // this generation's planes on the side stream during the DE fitness (QPM_WOLF=side)
    cudaEvent_t ev_wfork = nullptr, ev_wjoin = nullptr;
    int topk_threads = kCtaThreads;   // k_select_topk block (QPM_TOPK_THREADS)
    int topk_ctas = 1;                 // k_select_topk CTAs (NP / 2048, at most kTopkMaxCtas; QPM_TOPK_CTAS)
    bool fused_select = true;          // run_hybrid, NP <= 2048: fused finish + selection kernels (QPM_FUSED_SELECT)
    unsigned *fs_cnt = nullptr;        // their arrival counters [2]
    uint32_t *slot_tag = nullptr;      // [NP] slot | +/-1 flag per individual (trial setup in one load; QPM_SLOT_TAG)
    int S_cur = 1;                     // segments of the last one-GPU scan
    int32_t *topk_idx = nullptr;       // [kTopkMaxCtas][kTopSlots] per-CTA lists
    unsigned *topk_cnt = nullptr;      // arrival counter
    int64_t de_rows_max_dp = kDeRowsDefaultDp;  // warp-item trial kernel up to this row length (QPM_DE_ROWS)
    bool de_tma = QPM_DE_TMA != 0;          // TMA-staged trial rows (QPM_DE_TMA=0: global loads)
    bool fs_wide = false;                   // fused finish/selection with 1024-thread CTAs (large NP)
    int de_item = 1024;                      // genes per warp item on longer rows (QPM_DE_ITEM, multiple of 128)
    int stats_threads = kCtaThreads;  // k_select_stats block (QPM_STATS_THREADS)
    bool pdl = true;                // programmatic dependent launch on the main chain (QPM_PDL=0 disables)
    int64_t g_done = 0;
    bool initialized = false;
    bool init_pending = false;  // emulated shard: fitness scan of generation 0 done, exchange pending
    bool owns_stream = false;
    bool failed = false;  // a collective failed or timed out: the communicator was aborted
    unsigned *check_err = nullptr;  // QPM_CHECKS builds: [2] first invariant violation
    FitScratch check_fs;            // QPM_CHECKS builds: the candidates' fitness recomputed
    double *check_fit = nullptr;
    int64_t device_bytes = 0;
    std::vector<std::pair<void *, size_t>> allocs;
};

template <typename T>
static int dalloc(Engine *e, T **p, size_t count) {
    const size_t bytes = std::max<size_t>(count * sizeof(T), 16);
    *p = (T *)dev_cache_alloc(bytes);
    if (!*p) {
        set_error("out of device memory (%zu bytes)", bytes);
        return QPM_ERR_CUDA;
    }
    e->allocs.emplace_back((void *)*p, bytes);
    e->device_bytes += (int64_t)bytes;
    return QPM_OK;
}

// numpy's pairwise split tree of an n-vector: leaves in order (ids
// 0..L-1), internal nodes grouped by height so children precede parents
struct HostTree {
    std::vector<int32_t> leaf_off, kid, lvl;
};

struct TmpNode {
    int height, left, right;
    int64_t off;
};

static int tree_rec(int64_t off, int64_t n, std::vector<TmpNode> &nodes) {
    if (n <= 128) {
        nodes.push_back({0, -1, -1, off});
        return (int)nodes.size() - 1;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    const int a = tree_rec(off, n2, nodes);
    const int b = tree_rec(off + n2, n - n2, nodes);
    nodes.push_back({1 + std::max(nodes[a].height, nodes[b].height), a, b, off});
    return (int)nodes.size() - 1;
}

static HostTree build_tree(int64_t n) {
    std::vector<TmpNode> nodes;
    tree_rec(0, n, nodes);
    HostTree t;
    int max_h = 0;
    for (const TmpNode &v : nodes) max_h = std::max(max_h, v.height);
    std::vector<int> final_id(nodes.size(), -1);
    int next = 0;
    for (size_t v = 0; v < nodes.size(); ++v)
        if (nodes[v].height == 0) {
            final_id[v] = next++;
            t.leaf_off.push_back((int32_t)nodes[v].off);
        }
    const int nleaf = next;
    t.lvl.push_back(0);
    std::vector<int> order;
    for (int h = 1; h <= max_h; ++h) {
        for (size_t v = 0; v < nodes.size(); ++v)
            if (nodes[v].height == h) {
                final_id[v] = next++;
                order.push_back((int)v);
            }
        t.lvl.push_back(next - nleaf);
    }
    for (int v : order) {
        t.kid.push_back(final_id[nodes[v].left]);
        t.kid.push_back(final_id[nodes[v].right]);
    }
    t.leaf_off.push_back((int32_t)n);  // sentinel
    return t;
}

// one CTA per row; the CTA strides over the row's genes, so per-row setup
// (key folding, index draws, slot lookups) is paid once per row
static dim3 row_grid(const Engine *e, int64_t rows) {
    (void)e;
    return dim3(1u, (unsigned)rows);
}

// optional per-stage event marks (qpm_engine_profile)
constexpr int kMaxStages = 16;
struct StageMarks {
    cudaEvent_t ev[kMaxStages + 1];
    const char *name[kMaxStages];
    int n = 0;
    void mark(cudaStream_t s, const char *next_name) {
        cudaEventRecord(ev[n], s);
        if (next_name) name[n] = next_name;
        ++n;
    }
};

static size_t stats_smem_bytes(const RunConsts &c) {
    const size_t fitv = c.NP <= kStatsSmemMaxNP ? (size_t)2 * c.NP * sizeof(double) : 0;
    const size_t tree = (size_t)2 * c.n_leaf * sizeof(double) +
                        (size_t)((c.n_leaf + 1) + 2 * c.n_leaf + (c.n_levels + 1)) * sizeof(int32_t);
    return fitv + ((tree + 15) & ~(size_t)15);
}

static int launch_select_stats(Engine *e, int mode, cudaStream_t s) {
    QPM_CUDA_TRY(launch_k(e->pdl, k_select_stats, dim3(1), dim3(e->stats_threads), stats_smem_bytes(e->c), s, e->c, mode,
                          e->st, (const double *)e->sched, (const double *)e->cand, e->fit, e->slot_of, e->spare_of,
                          e->slot_bin, e->scratch, e->tree, e->trace, e->tree_inline, e->slot_tag));
    return QPM_OK;
}

static TrialArgs trial_args(const Engine *e, int64_t row_lo, int64_t n_rows) {
    TrialArgs a;
    a.st = e->st;
    a.gthr = e->gthr;
    a.row_lo = row_lo;
    a.n_rows = n_rows;
    a.picks = e->picks;
    a.keys = e->keys;
    a.jrand = e->jrand;
    a.planes = e->planes;
    a.cbits = e->cbits;
    a.slot_of = e->slot_of;
    a.slot_tag = e->slot_tag;
    a.spare_of = e->spare_of;
    a.slot_bin = e->slot_bin;
    a.genome = e->genome;
    a.bits = e->bits;
    return a;
}

static PlanArgs plan_args(const Engine *e) {
    PlanArgs a;
    a.st = e->st;
    a.gthr = e->gthr;
    a.row_lo = 0;
    a.n_rows = e->c.NP;
    a.keys = e->keys;
    a.picks = e->picks;
    a.jrand = e->jrand;
    a.planes = e->planes;
    return a;
}

// the planner for generation st->g_plan on stream s (then g_plan += 1)
static int enqueue_planner(Engine *e, cudaStream_t s) {
    const RunConsts &c = e->c;
    const PlanArgs pa = plan_args(e);
    k_plan_rows<<<(unsigned)((c.NP + 127) / 128), 128, 0, s>>>(c, pa);
    if (c.algorithm == QPM_ALGO_HYBRID && e->wolf_in_planner) {
        if (c.k == 4)
            k_plan_wolf<4><<<e->plan_grid, kRowThreads, 0, s>>>(c, pa);
        else
            k_plan_wolf<3><<<e->plan_grid, kRowThreads, 0, s>>>(c, pa);
    }
    k_plan_bump<<<1, 1, 0, s>>>(e->st);
    QPM_LAUNCH_CHECK();
    return QPM_OK;
}

// ---------------------------------------------------------------- NCCL
// Loaded at run time from the process's libnccl.so.2 (the one torch already
// mapped), so the library has no link-time NCCL dependency.
typedef int (*nccl_get_id_fn)(void *);
typedef int (*nccl_init_rank_fn)(void **, int, ncclUniqueIdPod, int);
typedef int (*nccl_allgather_fn)(const void *, void *, size_t, int, void *, cudaStream_t);
typedef int (*nccl_destroy_fn)(void *);
typedef const char *(*nccl_err_fn)(int);
typedef int (*nccl_async_err_fn)(void *, int *);
typedef int (*nccl_abort_fn)(void *);
struct NcclApi {
    bool loaded = false;
    nccl_get_id_fn get_id = nullptr;
    nccl_init_rank_fn init_rank = nullptr;
    nccl_allgather_fn allgather = nullptr;
    nccl_destroy_fn destroy = nullptr;
    nccl_err_fn err = nullptr;
    nccl_async_err_fn async_err = nullptr;  // ncclCommGetAsyncError
    nccl_abort_fn abort = nullptr;          // ncclCommAbort
};
constexpr int kNcclSuccess = 0, kNcclInProgress = 7;  // ncclResult_t (nccl.h)
static NcclApi g_nccl;
constexpr int kNcclFloat64 = 8;  // ncclFloat64 in nccl.h
constexpr int kNcclUint8 = 1;    // ncclUint8

static int nccl_load() {
    if (g_nccl.loaded) return QPM_OK;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        set_error("dlopen(libnccl.so.2) failed: %s", dlerror());
        return QPM_ERR_NCCL;
    }
    g_nccl.get_id = (nccl_get_id_fn)dlsym(h, "ncclGetUniqueId");
    g_nccl.init_rank = (nccl_init_rank_fn)dlsym(h, "ncclCommInitRank");
    g_nccl.allgather = (nccl_allgather_fn)dlsym(h, "ncclAllGather");
    g_nccl.destroy = (nccl_destroy_fn)dlsym(h, "ncclCommDestroy");
    g_nccl.err = (nccl_err_fn)dlsym(h, "ncclGetErrorString");
    g_nccl.async_err = (nccl_async_err_fn)dlsym(h, "ncclCommGetAsyncError");
    g_nccl.abort = (nccl_abort_fn)dlsym(h, "ncclCommAbort");
    if (!g_nccl.get_id || !g_nccl.init_rank || !g_nccl.allgather || !g_nccl.destroy || !g_nccl.err ||
        !g_nccl.async_err || !g_nccl.abort) {
        set_error("libnccl.so.2 lacks a required symbol");
        return QPM_ERR_NCCL;
    }
    g_nccl.loaded = true;
    return QPM_OK;
}

// exchange before phase `phase`: every rank's segment partials of the
// candidates' fitness (its columns of every row), all-gathered into gpart
static size_t gpart_slot(const Engine *e) { return (size_t)e->prob->n_wl * e->c.NP * e->SB_slot * kPartDoubles; }
static int enqueue_exchange(Engine *e, int phase) {
    (void)phase;
    if (!e->comm) return QPM_OK;  // one GPU, or emulated ranks (qpm_engine_exchange_from)
    const size_t n = gpart_slot(e);
    const int r = g_nccl.allgather(e->gpart + e->rank * n, e->gpart, n, kNcclFloat64, e->comm, e->stream);
    if (r != 0) {
        set_error("ncclAllGather: %s", g_nccl.err(r));
        return QPM_ERR_NCCL;
    }
    return QPM_OK;
}

// Failure detection for the collective path (the reference's failure
// contract is an exception, parexec.py:27-33; a hung or failed collective
// inside a replayed graph would otherwise block every later synchronize).
// An asynchronous NCCL error aborts the communicator and surfaces as
// QPM_ERR_NCCL; the engine is unusable afterwards.
static int nccl_poll(Engine *e) {
    if (!e->comm) return QPM_OK;
    int aerr = kNcclSuccess;
    const int r = g_nccl.async_err(e->comm, &aerr);
    if (r != kNcclSuccess || (aerr != kNcclSuccess && aerr != kNcclInProgress)) {
        const int code = r != kNcclSuccess ? r : aerr;
        set_error("NCCL asynchronous error on rank %d of %d: %s (communicator aborted)", e->rank, e->world,
                  g_nccl.err(code));
        g_nccl.abort(e->comm);
        e->comm = nullptr;
        e->failed = true;
        return QPM_ERR_NCCL;
    }
    return QPM_OK;
}

// the candidates' fitness into out[NP]: one GPU scores them now; a column
// shard scans its segments into its gpart slot and fit_finish scores them
// after the exchange
// run_hybrid on one GPU with the fused finish + selection kernels: the scans
// only write partials (QPM_FUSED_SELECT=0 restores finish + select kernels)
static bool fused_select(const Engine *e) { return e->c.algorithm == QPM_ALGO_HYBRID && e->fused_select; }
static int fit_scan(Engine *e, const uint32_t *bits, const int32_t *row_index, double *out, cudaStream_t s, int *n) {
    const RunConsts &c = e->c;
    if (!e->sharded() && fused_select(e))
        return launch_fitness_partials(e->prob, &e->fs, bits, c.W, row_index, c.NP, e->P.fitness_mode, s, n, e->pdl,
                                       &e->S_cur);
    if (!e->sharded())
        return launch_fitness(e->prob, &e->fs, bits, c.W, row_index, c.NP, out, e->P.fitness_mode, s, n, e->pdl);
    // a column shard: scan its segments, then pre-stitch its super-blocks
    // into its slot of the all-gather buffer
    const Problem *lp = e->lprob ? &e->lprob->p : e->prob;
    int rc = launch_fitness_scan(lp, bits, c.W, row_index, c.NP, e->fs.part, lp->S, s, n, e->pdl);
    if (rc) return rc;
    return launch_prestitch(e->prob, e->fs.part, lp->S, e->seg_lo, e->rank, e->world, e->SB_slot, c.NP,
                            e->gpart + e->rank * gpart_slot(e), s, n, e->pdl);
}
static FinishArgs fused_finish_args(const Engine *e) {
    if (e->sharded()) return finish_args_pre(e->prob, e->gpart, e->world, e->SB_slot, e->c.NP, e->ggains);
    return finish_args(e->prob, e->fs.part, e->S_cur, e->c.NP, e->fs.gains);
}
static int launch_finish_select(Engine *e, int mode, cudaStream_t s) {
    const RunConsts &c = e->c;
    if (e->fs_wide) {  // large populations: 32 rows per CTA, a 1024-thread last CTA
        constexpr int rw = kCtaThreads / 32;
        const dim3 grid((unsigned)((c.NP + rw - 1) / rw));
        if (mode == 0)
            QPM_CUDA_TRY(launch_k(e->pdl, k_finish_select<0, kCtaThreads>, grid, dim3(kCtaThreads), 0, s, c,
                                  fused_finish_args(e), e->st, (const double *)e->sched, e->cand, e->fit, e->slot_of,
                                  e->spare_of, e->slot_bin, e->scratch, e->tree, e->trace, e->tree_inline, e->fs_cnt,
                                  e->slot_tag));
        else
            QPM_CUDA_TRY(launch_k(e->pdl, k_finish_select<1, kCtaThreads>, grid, dim3(kCtaThreads), stats_smem_bytes(c),
                                  s, c, fused_finish_args(e), e->st, (const double *)e->sched, e->cand, e->fit,
                                  e->slot_of, e->spare_of, e->slot_bin, e->scratch, e->tree, e->trace, e->tree_inline,
                                  e->fs_cnt + 1, e->slot_tag));
        return QPM_OK;
    }
    constexpr int r0 = fs_threads<0>() / 32, r1 = fs_threads<1>() / 32;
    if (mode == 0)
        QPM_CUDA_TRY(launch_k(e->pdl, k_finish_select<0>, dim3((unsigned)((c.NP + r0 - 1) / r0)), dim3(fs_threads<0>()), 0,
                              s, c, fused_finish_args(e),
                              e->st, (const double *)e->sched, e->cand, e->fit, e->slot_of, e->spare_of, e->slot_bin,
                              e->scratch, e->tree, e->trace, e->tree_inline, e->fs_cnt, e->slot_tag));
    else
        QPM_CUDA_TRY(launch_k(e->pdl, k_finish_select<1>, dim3((unsigned)((c.NP + r1 - 1) / r1)), dim3(fs_threads<1>()),
                              stats_smem_bytes(c), s, c,
                              fused_finish_args(e), e->st, (const double *)e->sched, e->cand, e->fit, e->slot_of,
                              e->spare_of, e->slot_bin, e->scratch, e->tree, e->trace, e->tree_inline, e->fs_cnt + 1,
                              e->slot_tag));
    return QPM_OK;
}
static int fit_finish(Engine *e, double *out, cudaStream_t s, int *n) {
    if (!e->sharded()) return QPM_OK;
    return launch_fitness_finish(finish_args_pre(e->prob, e->gpart, e->world, e->SB_slot, e->c.NP, e->ggains), out, s,
                                 n, e->pdl);
}

// QPM_CHECKS builds: the candidates' fitness (cand, from cbits) recomputed by a
// separate scan + finish and compared bit for bit (one GPU)
static int enqueue_fit_check(Engine *e, cudaStream_t s, int *n) {
    if (!QPM_CHECKS || !e->check_err || e->sharded()) return QPM_OK;
    int rc = launch_fitness(e->prob, &e->check_fs, e->cbits, e->c.W, nullptr, e->c.NP, e->check_fit,
                            e->P.fitness_mode, s, n, false);
    if (rc) return rc;
    k_check_fitness<<<(unsigned)((e->c.NP + 255) / 256), 256, 0, s>>>(e->cand, e->check_fit, e->c.NP, e->check_err);
    QPM_LAUNCH_CHECK();
    *n += 1;
    return QPM_OK;
}

// QPM_CHECKS builds: the invariant check at the end of a generation (after the planner join)
static int enqueue_check(Engine *e, cudaStream_t s, int *n) {
    if (!QPM_CHECKS || !e->check_err) return QPM_OK;
    CheckArgs a{e->st, e->slot_of, e->spare_of, e->picks, e->jrand, e->fit, e->trace, e->check_err};
    const size_t smem = (size_t)((2 * e->c.NP + 31) / 32) * sizeof(uint32_t);
    k_check_state<<<1, kCtaThreads, smem, s>>>(e->c, a);
    QPM_LAUNCH_CHECK();
    *n += 1;
    return QPM_OK;
}

static int phase_count(const Engine *e) { return e->c.algorithm == QPM_ALGO_HYBRID ? 3 : 2; }

// One generation = phases separated by exchanges of the candidates' fitness
// partials (column shards; with one GPU the exchange is empty and each
// fitness is scored at once):
//   hybrid  P0 trial, scan | X | P1 finish, select+top-k, wolf, scan | X | P2 finish, select+stats
//   de      P0 trial, scan | X | P1 finish, select+stats
//   gwo     P0 top-k, wolf move, scan | X | P1 finish, replace+stats
// Every rank runs the per-gene kernels on its columns of all NP rows and the
// per-row kernels (finish, selection, statistics) on all rows, replicated.
static int enqueue_phase(Engine *e, int phase, int *n, StageMarks *pm) {
    const RunConsts &c = e->c;
    cudaStream_t s = e->stream;
    int rc;
    auto mark = [&](const char *next) {
        if (pm) pm->mark(s, next);
    };
    const int64_t NP = c.NP;
    const bool sharded = e->sharded();
    const int64_t de_chunks = (c.Dp + kDeChunk - 1) / kDeChunk;
    if (phase > 0 && sharded && !fused_select(e)) {
        mark("fitness_finish");
        if ((rc = fit_finish(e, e->cand, s, n))) return rc;
    }
    if (c.algorithm == QPM_ALGO_GWO) {
        if (phase == 0) {
            mark("topk");
            QPM_CUDA_TRY(launch_k(false, k_topk_leaders, dim3(1), dim3(kCtaThreads), 0, s, c, e->st,
                                  (const double *)e->fit, 3));  // rank_leaders(pop, 3); first kernel: no PDL
            mark("gwo_continuous");
            QPM_CUDA_TRY(launch_k(e->pdl, k_gwo_continuous, row_grid(e, NP), dim3(kRowThreads), 0, s, c,
                                  (const EngineState *)e->st, (const double *)e->sched, (int64_t)0,
                                  (const int32_t *)e->slot_of, (const int32_t *)e->spare_of, e->slot_bin, e->genome,
                                  e->bits));
            QPM_LAUNCH_CHECK();
            *n += 2;
            mark("fitness");
            if ((rc = fit_scan(e, e->bits, e->spare_of, e->cand, s, n))) return rc;
        } else {
            mark("replace_stats");
            if ((rc = launch_select_stats(e, 2, s))) return rc;
            k_copy_best<<<64, 256, 0, s>>>(c, e->st, e->slot_of, e->slot_bin, e->genome, e->bits, e->best_genome,
                                           e->best_bits);
            QPM_LAUNCH_CHECK();
            *n += 2;
            return enqueue_check(e, s, n);
        }
        return QPM_OK;
    }
    const bool hybrid = c.algorithm == QPM_ALGO_HYBRID;
    TrialArgs all = trial_args(e, 0, NP);
    if (phase == 0) {
        // fork: the planner draws generation g+1 on the side stream
        auto fork = [&]() -> int {
            QPM_CUDA_TRY(cudaEventRecord(e->ev_fork, s));
            QPM_CUDA_TRY(cudaStreamWaitEvent(e->side, e->ev_fork, 0));
            int r = enqueue_planner(e, e->side);
            if (r) return r;
            QPM_CUDA_TRY(cudaEventRecord(e->ev_join, e->side));
            *n += (hybrid && e->wolf_in_planner) ? 3 : 2;
            return QPM_OK;
        };
        if (!e->plan_after_trial && (rc = fork())) return rc;
        mark("de_trial");
        // the generation's first kernel is launched programmatically only
        // inside a multi-generation graph (after the previous generation's
        // select_stats); a graph's root node would otherwise overlap the
        // previous replay's tail, including its planner branch
        const bool pdl_trial = e->pdl && e->pdl_trial;
        const unsigned items = (unsigned)(NP * de_chunks);
        const bool wolf_side = hybrid && e->wolf_side;
        const bool rows_mode = c.Dp <= e->de_rows_max_dp && !e->wolf_mixed;
        const int ch = c.Dp <= kDeRowsMaxDp ? (int)c.Dp : e->de_item;  // genes per warp item
        const int64_t n_items = NP * ((c.Dp + ch - 1) / ch);
        const unsigned row_ctas = (unsigned)((n_items + kRowThreads / 32 - 1) / (kRowThreads / 32));
        if (rows_mode) {
            const bool k0 = !hybrid || e->wolf_in_planner || wolf_side;
            QPM_CUDA_TRY(launch_k(pdl_trial, k0 ? k_de_trial_rows<0> : (c.k == 4 ? k_de_trial_rows<4> : k_de_trial_rows<3>),
                                  dim3(row_ctas), dim3(kRowThreads), 0, s, c, all, ch));
        } else if (e->de_tma && ((!hybrid || e->wolf_in_planner || wolf_side) || !e->wolf_mixed)) {
            const bool long_rows = c.Dp >= kTmaLongRows;
            const int kw = (!hybrid || e->wolf_in_planner || wolf_side) ? 0 : c.k;
            const unsigned ti = (unsigned)(NP * ((c.Dp + (long_rows ? 8192 : kDeChunk) - 1) /
                                                 (long_rows ? 8192 : kDeChunk)));
            auto kern = long_rows ? (kw == 0 ? k_de_trial_tma<0, 8192> : kw == 4 ? k_de_trial_tma<4, 8192>
                                                                                  : k_de_trial_tma<3, 8192>)
                                  : (kw == 0 ? k_de_trial_tma<0> : kw == 4 ? k_de_trial_tma<4> : k_de_trial_tma<3>);
            QPM_CUDA_TRY(launch_k(pdl_trial, kern, dim3(ti), dim3(kRowThreads), kTmaSmem, s, c, all));
        }
        else if (!hybrid || e->wolf_in_planner || wolf_side)
            QPM_CUDA_TRY(launch_k(pdl_trial, k_de_trial<0>, dim3(items), dim3(kRowThreads), 0, s, c, all));
        else if (e->wolf_mixed)
            QPM_CUDA_TRY(launch_k(pdl_trial, c.k == 4 ? k_de_trial_mixed<4> : k_de_trial_mixed<3>, dim3(2 * items),
                                  dim3(kRowThreads), 0, s, c, all));
        else
            QPM_CUDA_TRY(launch_k(pdl_trial, c.k == 4 ? k_de_trial<4> : k_de_trial<3>, dim3(items), dim3(kRowThreads), 0,
                                  s, c, all));
        QPM_LAUNCH_CHECK();
        *n += 1;
        if (wolf_side) {  // the planes of this generation, concurrent with the DE fitness and selection
            QPM_CUDA_TRY(cudaEventRecord(e->ev_wfork, s));
            QPM_CUDA_TRY(cudaStreamWaitEvent(e->side, e->ev_wfork, 0));
            const PlanArgs pa = plan_args(e);
            if (c.k == 4)
                k_plan_wolf<4, true><<<e->plan_grid, kRowThreads, 0, e->side>>>(c, pa);
            else
                k_plan_wolf<3, true><<<e->plan_grid, kRowThreads, 0, e->side>>>(c, pa);
            QPM_LAUNCH_CHECK();
            QPM_CUDA_TRY(cudaEventRecord(e->ev_wjoin, e->side));
            *n += 1;
        }
        if (e->plan_after_trial && (rc = fork())) return rc;
        mark("fitness_de");
        return fit_scan(e, e->cbits, nullptr, e->cand, s, n);
    }
    if (phase == 1) {
        if (!hybrid) {
            if ((rc = enqueue_fit_check(e, s, n))) return rc;  // the DE candidates (QPM_CHECKS)
            mark("select_stats");
            if ((rc = launch_select_stats(e, 0, s))) return rc;
            *n += 1;
            QPM_CUDA_TRY(cudaStreamWaitEvent(s, e->ev_join, 0));  // join the planner
            return enqueue_check(e, s, n);
        }
        if (fused_select(e)) {
            mark("finish_select_topk");
            if ((rc = launch_finish_select(e, 0, s))) return rc;
        } else {
            mark("select_topk");
            QPM_CUDA_TRY(launch_k(e->pdl, k_select_topk, dim3((unsigned)e->topk_ctas), dim3(e->topk_threads), 0, s, c,
                                  e->st, (const double *)e->cand, e->fit, e->slot_of, e->spare_of,
                                  TopkScratch{e->topk_idx, e->topk_cnt}, e->slot_tag));
        }
        if ((rc = enqueue_fit_check(e, s, n))) return rc;  // the DE candidates (QPM_CHECKS)
        if (e->wolf_side) QPM_CUDA_TRY(cudaStreamWaitEvent(s, e->ev_wjoin, 0));  // this generation's planes
        mark("gwo_apply");
        QPM_CUDA_TRY(launch_k(e->pdl, c.k == 4 ? k_gwo_apply<4> : k_gwo_apply<3>,
                              dim3((unsigned)((NP * c.W + kApplyThreads - 1) / kApplyThreads)), dim3(kApplyThreads),
                              0, s, c, all));
        QPM_LAUNCH_CHECK();
        *n += 2;
        mark("fitness_gwo");
        return fit_scan(e, e->cbits, nullptr, e->cand, s, n);
    }
    // phase 2 (hybrid)
    if (fused_select(e)) {
        mark("finish_select_stats");
        if ((rc = launch_finish_select(e, 1, s))) return rc;
    } else {
        mark("select_stats");
        if ((rc = launch_select_stats(e, 1, s))) return rc;
    }
    *n += 1;
    if ((rc = enqueue_fit_check(e, s, n))) return rc;  // the wolf candidates (QPM_CHECKS)
    QPM_CUDA_TRY(cudaStreamWaitEvent(s, e->ev_join, 0));  // join the planner
    return enqueue_check(e, s, n);
}

// one generation's launch sequence
static int enqueue_generation(Engine *e, int *launches, StageMarks *pm = nullptr) {
    int n = 0, rc;
    const int np = phase_count(e);
    for (int ph = 0; ph < np; ++ph) {
        if (ph > 0 && (rc = enqueue_exchange(e, ph))) return rc;
        if ((rc = enqueue_phase(e, ph, &n, pm))) return rc;
    }
    if (pm) pm->mark(e->stream, nullptr);
    if (launches) *launches = n;
    return QPM_OK;
}

// Process-wide pool of the planner's side streams and fork/join events:
// engines created and destroyed back to back (run_hybrid in a loop, trials)
// reuse them instead of creating a stream and four events per run.
struct SideSet {
    int device;
    cudaStream_t side;
    cudaEvent_t ev[4];
};
static std::mutex g_side_mu;
static std::vector<SideSet> g_side_pool;

static int side_acquire(Engine *e) {
    int dev = 0;
    cudaGetDevice(&dev);
    {
        std::lock_guard<std::mutex> lk(g_side_mu);
        for (size_t k = 0; k < g_side_pool.size(); ++k)
            if (g_side_pool[k].device == dev) {
                const SideSet ss = g_side_pool[k];
                g_side_pool[k] = g_side_pool.back();
                g_side_pool.pop_back();
                e->side = ss.side;
                e->ev_fork = ss.ev[0], e->ev_join = ss.ev[1], e->ev_wfork = ss.ev[2], e->ev_wjoin = ss.ev[3];
                return QPM_OK;
            }
    }
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);  // lo = least urgent
    if (cudaStreamCreateWithPriority(&e->side, cudaStreamNonBlocking, lo) != cudaSuccess ||
        cudaEventCreateWithFlags(&e->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&e->ev_join, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&e->ev_wfork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&e->ev_wjoin, cudaEventDisableTiming) != cudaSuccess) {
        set_error("planner stream/event creation failed");
        return QPM_ERR_CUDA;
    }
    return QPM_OK;
}

// (the side stream is idle: engine_free synchronised it)
static void side_release(Engine *e) {
    if (!e->side) return;
    int dev = 0;
    cudaGetDevice(&dev);
    if (e->ev_fork && e->ev_join && e->ev_wfork && e->ev_wjoin) {
        std::lock_guard<std::mutex> lk(g_side_mu);
        if (g_side_pool.size() < 64) {
            g_side_pool.push_back({dev, e->side, {e->ev_fork, e->ev_join, e->ev_wfork, e->ev_wjoin}});
            e->side = nullptr;
            e->ev_fork = e->ev_join = e->ev_wfork = e->ev_wjoin = nullptr;
            return;
        }
    }
    cudaStreamDestroy(e->side);
    e->side = nullptr;
}

static void engine_free(Engine *e) {
    // the buffers go back to the block cache: nothing queued may still use them
    if (e->stream) cudaStreamSynchronize(e->stream);
    if (e->owns_stream && e->stream) cudaStreamDestroy(e->stream);
    if (e->side) {
        cudaStreamSynchronize(e->side);
        side_release(e);  // back to the pool (with its events), or destroyed
    }
    if (e->comm && g_nccl.destroy) g_nccl.destroy(e->comm);
    if (e->ev_fork) cudaEventDestroy(e->ev_fork);
    if (e->ev_join) cudaEventDestroy(e->ev_join);
    if (e->ev_wfork) cudaEventDestroy(e->ev_wfork);
    if (e->ev_wjoin) cudaEventDestroy(e->ev_wjoin);
    if (e->exec) cudaGraphExecDestroy(e->exec);
    if (e->graph) cudaGraphDestroy(e->graph);
    if (e->exec_k) cudaGraphExecDestroy(e->exec_k);
    if (e->graph_k) cudaGraphDestroy(e->graph_k);
    for (auto &pb : e->allocs) dev_cache_release(pb.first, pb.second);
    scratch_free(&e->fs);
    scratch_free(&e->check_fs);
    if (e->lprob) qpm_problem_destroy(e->lprob);
    delete e;
}

}  // namespace qpm

struct qpm_engine {
    qpm::Engine *e;
};

using namespace qpm;

extern "C" {

// A per-thread pinned host buffer of at least `bytes` (nullptr when pinned
// memory is unavailable: callers then copy through pageable memory).  Used
// between an enqueue and the stream synchronisation that ends its use.
// Copies out of the buffer may still be in flight from the previous user
// (engine creation does not wait for its uploads): pinned_staging_busy(s)
// records that, and the next pinned_staging call waits for it first.
static thread_local cudaEvent_t t_staging_ev = nullptr;
static thread_local bool t_staging_pending = false;
static void pinned_staging_busy(cudaStream_t s) {
    if (!t_staging_ev && cudaEventCreateWithFlags(&t_staging_ev, cudaEventDisableTiming) != cudaSuccess) {
        t_staging_ev = nullptr;
        cudaStreamSynchronize(s);  // (no event: wait here instead)
        return;
    }
    if (cudaEventRecord(t_staging_ev, s) == cudaSuccess)
        t_staging_pending = true;
    else
        cudaStreamSynchronize(s);
}
static char *pinned_staging(size_t bytes) {
    static thread_local char *pinned = nullptr;
    static thread_local size_t pinned_bytes = 0;
    if (t_staging_pending) {
        cudaEventSynchronize(t_staging_ev);
        t_staging_pending = false;
    }
    if (pinned_bytes < bytes) {
        if (pinned) cudaFreeHost(pinned);
        pinned = nullptr;
        pinned_bytes = 0;
        const size_t want = std::max<size_t>(bytes, (size_t)1 << 20);
        if (cudaMallocHost(&pinned, want) == cudaSuccess) pinned_bytes = want;
    }
    return pinned;
}

int qpm_engine_create(qpm_engine **out, qpm_problem *prob, const qpm_run_params *P, const double *sched,
                      void *stream) {
    QPM_ARG_CHECK(out && prob && P && sched, "out, problem, params, sched");
    QPM_ARG_CHECK(P->NP >= 4, "population size must be >= 4");
    QPM_ARG_CHECK(P->G >= 0, "generations >= 0");
    QPM_ARG_CHECK(P->algorithm >= QPM_ALGO_HYBRID && P->algorithm <= QPM_ALGO_GWO, "algorithm");
    QPM_ARG_CHECK(P->fitness_mode == QPM_MODE_FAST || P->fitness_mode == QPM_MODE_EXACT, "fitness_mode");
    QPM_ARG_CHECK(P->algorithm == QPM_ALGO_GWO || P->leader_count == 3 || P->leader_count == 4,
                  "leader_count must be 3 or 4");
    QPM_ARG_CHECK(P->conv_window >= 1 && P->conv_window <= kMaxWindow, "conv_window in [1, 256]");
    QPM_ARG_CHECK(P->shard_world >= 1 && P->shard_rank >= 0 && P->shard_rank < P->shard_world,
                  "shard_rank in [0, shard_world)");
    QPM_ARG_CHECK(P->NP < (1LL << 30), "NP < 2^30");
    const Problem &gp = prob->p;
    if (P->shard_world > 1) {
        QPM_ARG_CHECK(P->fitness_mode == QPM_MODE_FAST,
                      "multi-GPU runs score in fast mode (exact mode is the single-GPU parity tool)");
        QPM_ARG_CHECK(gp.nsb >= P->shard_world,
                      "fewer fitness super-blocks than ranks: D is too small for this many GPUs "
                      "(a shorter seg_chunks at qpm_problem_create gives more segments)");
    }
    Engine *e = new Engine();
    e->prob = &prob->p;
    e->P = *P;
    e->rank = P->shard_rank;
    e->world = P->shard_world;
    e->stream = (cudaStream_t)stream;
    if (!e->stream) {
        // graphs cannot be captured on the legacy default stream: own a stream
        int lo_p = 0, hi_p = 0;
        cudaDeviceGetStreamPriorityRange(&lo_p, &hi_p);
        if (cudaStreamCreateWithPriority(&e->stream, cudaStreamNonBlocking, hi_p) != cudaSuccess) {
            set_error("cudaStreamCreateWithFlags failed");
            delete e;
            return QPM_ERR_CUDA;
        }
        e->owns_stream = true;
    }
    if (side_acquire(e) != QPM_OK) {
        engine_free(e);
        return QPM_ERR_CUDA;
    }
    RunConsts &c = e->c;
    c.algorithm = P->algorithm;
    c.NP = P->NP;
    c.Dg = gp.D;
    if (e->world > 1) {
        // rank k owns the stitch super-blocks [floor(k nsb / W), floor((k+1)
        // nsb / W)), i.e. a contiguous run of fitness segments, and the genes
        // under them (segment boundaries are 128-domain aligned)
        const int sb0 = sb_first(e->rank, gp.nsb, e->world), sb1 = sb_first(e->rank + 1, gp.nsb, e->world);
        e->seg_lo = sb_lo(sb0, gp.S, gp.nsb);
        const int seg_hi = sb_lo(sb1, gp.S, gp.nsb);
        e->seg_n = seg_hi - e->seg_lo;
        e->SB_slot = (gp.nsb + e->world - 1) / e->world;
        const int64_t seg_len = (int64_t)gp.seg_chunks * 128;
        c.g0 = e->seg_lo * seg_len;
        const int64_t g1 = std::min<int64_t>(gp.D, seg_hi * seg_len);
        const int rc = problem_slice(&gp, c.g0, g1 - c.g0, &e->lprob);
        if (rc) {
            engine_free(e);
            return rc;
        }
        c.D = e->lprob->p.D;
        c.W = e->lprob->p.W;
    } else {
        e->seg_n = gp.S;
        e->SB_slot = gp.nsb;  // (used when a 1-rank communicator makes the engine take the sharded flow)
        c.g0 = 0;
        c.D = gp.D;
        c.W = gp.W;
    }
    c.Dp = c.W * 32;
    c.G = P->G;
    c.seed = (uint64_t)P->seed;
    c.f_max = P->f_max;
    c.f_min = P->f_min;
    c.cr_thr = le_threshold(P->cr);
    c.thr_cr = make_thr(c.cr_thr);
    if (P->algorithm == QPM_ALGO_GWO) {
        c.x_lo = P->gwo_lo;
        c.x_span = P->gwo_hi - P->gwo_lo;
        c.k = 3;
    } else {
        c.x_lo = P->x_min;
        c.x_span = P->x_max - P->x_min;
        c.k = P->leader_count;
    }
    c.divide = P->divide_by_leader_count;
    c.theta_low_frac = P->theta_low_frac;
    c.theta_high_frac = P->theta_high_frac;
    c.range_trigger_frac = P->range_trigger_frac;
    c.explore_boost = P->explore_boost;
    c.exploit_factor = P->exploit_factor;
    c.conv_threshold = P->conv_threshold;
    c.conv_window = P->conv_window;
    c.adaptive = P->adaptive_branches;
    c.gwo_a0 = P->gwo_a0;
    {
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        e->plan_grid = sms * 2;
        // scheduling knobs for A/B measurement and the schedule tests: read
        // only when QPM_DEV_KNOBS=1 (none changes a result: every combination
        // reproduces the default trace bit for bit, tests/test_gpu_schedules.py)
        const bool dev_knobs = getenv("QPM_DEV_KNOBS") && atoi(getenv("QPM_DEV_KNOBS")) != 0;
        auto knob = [dev_knobs](const char *name) -> const char * { return dev_knobs ? getenv(name) : nullptr; };
        if (const char *v = knob("QPM_PLAN_CTAS")) e->plan_grid = std::max(1, atoi(v));
        const char *fork = knob("QPM_PLAN_FORK");
        if (fork) e->plan_after_trial = strcmp(fork, "trial") == 0;
        if (const char *v = knob("QPM_WOLF")) {
            e->wolf_in_planner = strcmp(v, "planner") == 0;
            e->wolf_mixed = strcmp(v, "mixed") == 0;
            e->wolf_side = strcmp(v, "side") == 0;
        }
        // wolf planes on the side stream are drawn after the trial (round 1:
        // forked at the start of the generation, C2 traces differed from run
        // to run); QPM_PLAN_FORK=start keeps the start fork for the
        // race probe (tools/sanitize.sh)
        if (e->wolf_in_planner && !(fork && strcmp(fork, "start") == 0)) e->plan_after_trial = true;
        if (const char *v = knob("QPM_PDL")) e->pdl = atoi(v) != 0;
        if (const char *v = knob("QPM_GRAPH_GENS")) e->graph_gens = std::min(64, std::max(1, atoi(v)));
        if (const char *v = knob("QPM_DE_ROWS")) e->de_rows_max_dp = atoll(v);
        if (const char *v = knob("QPM_DE_TMA")) e->de_tma = atoi(v) != 0;
        e->topk_ctas = (int)std::min<int64_t>(kTopkMaxCtas, std::max<int64_t>(1, c.NP / 2048));
        if (const char *v = knob("QPM_TOPK_CTAS")) e->topk_ctas = std::min(kTopkMaxCtas, std::max(1, atoi(v)));
        // fused finish + selection: its last CTA runs the whole-population part
        // alone, which pays up to ~2k rows (C2: 116.0 -> 113.8 us per
        // generation; NP 8192: 133 -> 149 us, alternating A/B)
        // ... and with 1024-thread CTAs up to 4,096 rows (C4 391.1 -> 388.2
        // us/gen; emulated NP 4096 shards 193 -> 187 us); at 8,192 the
        // multi-CTA top-k kernel is faster than one wide last CTA
        e->fused_select = c.NP <= 2048 || (QPM_FS_WIDE && c.NP <= 4096);
        e->fs_wide = c.NP > 2048;
        if (const char *v = knob("QPM_FUSED_SELECT")) e->fused_select = atoi(v) != 0;
        if (const char *v = knob("QPM_DE_ITEM")) e->de_item = std::max(128, atoi(v) / 128 * 128);
        auto cta_knob = [&knob](const char *name, int &dst) {  // multiple of 32 in [32, kCtaThreads]
            if (const char *v = knob(name)) dst = std::min(kCtaThreads, std::max(32, atoi(v) / 32 * 32));
        };
        cta_knob("QPM_TOPK_THREADS", e->topk_threads);
        cta_knob("QPM_STATS_THREADS", e->stats_threads);
    }
    HostTree ht = build_tree(c.NP);
    c.n_leaf = (int32_t)ht.leaf_off.size() - 1;
    c.n_levels = (int32_t)ht.lvl.size() - 1;
    {
        // the attributes are per function: raised to the device's opt-in
        // maximum once per process (one device per process), whatever the
        // engine's size; each engine then only checks its own need
        struct SmemAttrs {
            int max_optin = 0;
            size_t st_static = 0, fs_static = 0, fw_static = 0;
            bool st_ok = false, fs_ok = false, fw_ok = false, tma_ok = false;
        };
        static SmemAttrs sa;
        static std::once_flag attrs_once;
        std::call_once(attrs_once, [] {
            int dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sa.max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
            cudaFuncAttributes fa{}, fb{}, fw{};
            cudaFuncGetAttributes(&fa, k_select_stats);
            cudaFuncGetAttributes(&fb, k_finish_select<1>);
            cudaFuncGetAttributes(&fw, k_finish_select<1, kCtaThreads>);
            sa.st_static = fa.sharedSizeBytes;
            sa.fs_static = fb.sharedSizeBytes;
            sa.fw_static = fw.sharedSizeBytes;
            sa.st_ok = cudaFuncSetAttribute(k_select_stats, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            sa.max_optin - (int)fa.sharedSizeBytes) == cudaSuccess;
            sa.fs_ok = cudaFuncSetAttribute(k_finish_select<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            sa.max_optin - (int)fb.sharedSizeBytes) == cudaSuccess;
            sa.fw_ok = cudaFuncSetAttribute(k_finish_select<1, kCtaThreads>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            sa.max_optin - (int)fw.sharedSizeBytes) == cudaSuccess;
            // the TMA-staged trial's stage ring (static shared memory on top)
            const void *ks[6] = {(const void *)k_de_trial_tma<0>, (const void *)k_de_trial_tma<3>,
                                 (const void *)k_de_trial_tma<4>, (const void *)k_de_trial_tma<0, 8192>,
                                 (const void *)k_de_trial_tma<3, 8192>, (const void *)k_de_trial_tma<4, 8192>};
            sa.tma_ok = true;
            for (const void *k : ks)
                if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTmaSmem) != cudaSuccess)
                    sa.tma_ok = false;
            cudaGetLastError();  // (a failed attribute call is reported through the flags)
        });
        const size_t need = stats_smem_bytes(c) + sa.st_static;
        if ((size_t)sa.max_optin < need || !sa.st_ok) {
            set_error("k_select_stats needs %zu bytes of shared memory (device: %d)", need, sa.max_optin);
            engine_free(e);
            return QPM_ERR_CUDA;
        }
        if (!sa.tma_ok) e->de_tma = false;  // (the global-load trial then runs)
        const bool narrow_ok = sa.fs_ok && (size_t)sa.max_optin >= stats_smem_bytes(c) + sa.fs_static;
        const bool wide_ok = sa.fw_ok && (size_t)sa.max_optin >= stats_smem_bytes(c) + sa.fw_static;
        if (!(e->fs_wide ? wide_ok : narrow_ok)) e->fused_select = false;  // (the statistics then run in k_select_stats)
    }

    const int64_t NP = c.NP;
    int rc = QPM_OK;
#define QPM_ALLOC(ptr, count)                     \
    if ((rc = dalloc(e, &(ptr), (count))) != 0) { \
        engine_free(e);                           \
        return rc;                                \
    }
    QPM_ALLOC(e->genome, (size_t)2 * NP * c.Dp);
    QPM_ALLOC(e->bits, (size_t)2 * NP * c.W);
    QPM_ALLOC(e->slot_bin, (size_t)2 * NP);
    QPM_ALLOC(e->planes, P->algorithm == QPM_ALGO_HYBRID ? (size_t)2 * NP * c.W * kPlanes : 16);
    QPM_ALLOC(e->cbits, P->algorithm != QPM_ALGO_GWO ? (size_t)NP * c.W : 16);
    QPM_ALLOC(e->gthr, (size_t)(P->G + 1));
    QPM_ALLOC(e->slot_of, NP);
    QPM_ALLOC(e->spare_of, NP);
    QPM_ALLOC(e->jrand, 2 * NP);
    QPM_ALLOC(e->fit, NP);
    QPM_ALLOC(e->cand, NP);
    QPM_ALLOC(e->scratch, NP);
    QPM_ALLOC(e->tree_i, ht.leaf_off.size() + ht.kid.size() + ht.lvl.size());
    QPM_ALLOC(e->tree_v, 2 * (size_t)c.n_leaf);
    QPM_ALLOC(e->keys, 2 * NP);
    QPM_ALLOC(e->picks, 2 * NP);
    QPM_ALLOC(e->sched, (size_t)(P->G + 1) * QPM_SCHED_COLS);
    QPM_ALLOC(e->trace, (size_t)(P->G + 1) * 5);
    QPM_ALLOC(e->st, 1);
    QPM_ALLOC(e->best_genome, c.Dp);
    QPM_ALLOC(e->best_bits, c.W);
    QPM_ALLOC(e->topk_idx, (size_t)kTopkMaxCtas * kTopSlots);
    QPM_ALLOC(e->topk_cnt, 1);
    QPM_ALLOC(e->fs_cnt, 2);
    if (QPM_CHECKS) {
        QPM_ALLOC(e->check_err, 2);
        QPM_ALLOC(e->check_fit, NP);
    }
    if (QPM_SLOT_TAG) QPM_ALLOC(e->slot_tag, NP);
    if (e->world > 1) {
        QPM_ALLOC(e->gpart, (size_t)e->world * gpart_slot(e));
        QPM_ALLOC(e->ggains, (size_t)NP * gp.n_wl);
    }  // one rank with a communicator: allocated by qpm_engine_set_comm
#undef QPM_ALLOC
    if ((rc = scratch_reserve(e->lprob ? &e->lprob->p : e->prob, &e->fs, NP)) != 0) {
        engine_free(e);
        return rc;
    }
    e->device_bytes += e->fs.bytes;
    if (QPM_CHECKS && (rc = scratch_reserve(e->prob, &e->check_fs, NP)) != 0) {
        engine_free(e);
        return rc;
    }
    std::vector<int32_t> tree_host;
    tree_host.insert(tree_host.end(), ht.leaf_off.begin(), ht.leaf_off.end());
    tree_host.insert(tree_host.end(), ht.kid.begin(), ht.kid.end());
    tree_host.insert(tree_host.end(), ht.lvl.begin(), ht.lvl.end());
    e->tree.leaf_off = e->tree_i;
    e->tree.kid = e->tree_i + ht.leaf_off.size();
    e->tree.lvl = e->tree_i + ht.leaf_off.size() + ht.kid.size();
    e->tree.val = e->tree_v;
    {
        const size_t nt = ht.leaf_off.size() + ht.kid.size() + ht.lvl.size();
        e->tree_inline.n = 0;
        if (QPM_TREE_INLINE && nt <= (size_t)kTreeInline && ht.kid.size() == 2 * (ht.leaf_off.size() - 2)) {
            size_t k = 0;
            for (int32_t v : ht.leaf_off) e->tree_inline.v[k++] = v;
            for (int32_t v : ht.kid) e->tree_inline.v[k++] = v;
            for (int32_t v : ht.lvl) e->tree_inline.v[k++] = v;
            e->tree_inline.n = (int32_t)nt;
        }
    }
    // host-side constants of the state: p_plus thresholds (optimizer.py:362-365)
    EngineState hs;
    memset(&hs, 0, sizeof(hs));
    for (int cnt = 0; cnt <= c.k && cnt <= kMaxLeaders; ++cnt) {
        double pp = (double)cnt / (double)c.k;
        if (P->discreteness_factor != 1.0) pp = 0.5 + P->discreteness_factor * (pp - 0.5);
        hs.thr_plus[cnt] = lt_threshold(pp);
        if (cnt < 5) c.thr_plus[cnt] = make_thr(hs.thr_plus[cnt]);
    }
    c.plus_dyadic = (c.k == 4 && P->discreteness_factor == 1.0) ? 1 : 0;
    // p_plus(0) = 0 and p_plus(K) = 1: the plus level L lies in [1, K], so
    // unanimous leaders decide "plus" without the draw
    c.plus_ends = (c.k <= kMaxLeaders && hs.thr_plus[0] == 0 && hs.thr_plus[c.k] > kTwo53) ? 1 : 0;
    c.m4 = 4;
    c.m32 = 32;
    c.m2 = 2;
    hs.g = 0;
    hs.g_plan = 1;
    hs.F = P->f_max;
    // per-generation wolf thresholds from the schedule table (optimizer.py:447-453)
    std::vector<GenThr> gth((size_t)P->G + 1);
    for (int64_t g = 0; g <= P->G; ++g) {
        const double *sg = sched + g * QPM_SCHED_COLS;
        gth[g].sl = make_thr(lt_threshold(sg[QPM_SCHED_P_SL]));
        gth[g].dist = make_thr(lt_threshold(sg[QPM_SCHED_P_DIST]));
        gth[g].flip = make_thr(lt_threshold(sg[QPM_SCHED_P_FLIP]));
        gth[g].early = sg[QPM_SCHED_EARLY] != 0.0 ? 1u : 0u;
        gth[g].pad = 0;
    }
    // the uploads go through a pinned per-thread staging buffer: asynchronous
    // copies (a pageable source makes every cudaMemcpyAsync a staged,
    // synchronous copy); the stream synchronisation below ends its use
    const size_t b_st = sizeof(hs), b_gth = sizeof(GenThr) * gth.size(),
                 b_sched = sizeof(double) * (P->G + 1) * QPM_SCHED_COLS, b_tree = sizeof(int32_t) * tree_host.size();
    const size_t o_gth = round_up((int64_t)b_st, 256), o_sched = o_gth + round_up((int64_t)b_gth, 256),
                 o_tree = o_sched + round_up((int64_t)b_sched, 256), b_all = o_tree + b_tree;
    char *pinned = pinned_staging(b_all);
    const char *src_st = reinterpret_cast<const char *>(&hs), *src_gth = reinterpret_cast<const char *>(gth.data()),
               *src_sched = reinterpret_cast<const char *>(sched),
               *src_tree = reinterpret_cast<const char *>(tree_host.data());
    if (pinned) {
        memcpy(pinned, &hs, b_st);
        memcpy(pinned + o_gth, gth.data(), b_gth);
        memcpy(pinned + o_sched, sched, b_sched);
        memcpy(pinned + o_tree, tree_host.data(), b_tree);
        src_st = pinned, src_gth = pinned + o_gth, src_sched = pinned + o_sched, src_tree = pinned + o_tree;
    }
    cudaError_t err = cudaMemcpyAsync(e->st, src_st, b_st, cudaMemcpyHostToDevice, e->stream);
    if (err == cudaSuccess) err = cudaMemcpyAsync(e->gthr, src_gth, b_gth, cudaMemcpyHostToDevice, e->stream);
    if (err == cudaSuccess) err = cudaMemcpyAsync(e->sched, src_sched, b_sched, cudaMemcpyHostToDevice, e->stream);
    if (err == cudaSuccess) err = cudaMemcpyAsync(e->tree_i, src_tree, b_tree, cudaMemcpyHostToDevice, e->stream);
    if (err == cudaSuccess) err = cudaMemsetAsync(e->trace, 0, sizeof(double) * (P->G + 1) * 5, e->stream);
    // (the genome pool is not cleared: init_population writes every gene of the
    // current slots, a spare slot is written whole -- padding included -- by the
    // trial or the continuous move before it becomes current, and ±1 slots are
    // read from their bits; clearing cost 30 us at C2, ~4 ms at C3)
    if (err == cudaSuccess) err = cudaMemsetAsync(e->bits, 0, sizeof(uint32_t) * 2 * NP * c.W, e->stream);
    if (err == cudaSuccess) err = cudaMemsetAsync(e->slot_bin, 0, 2 * NP, e->stream);
    if (err == cudaSuccess) err = cudaMemsetAsync(e->topk_cnt, 0, sizeof(unsigned), e->stream);
    if (err == cudaSuccess) err = cudaMemsetAsync(e->fs_cnt, 0, 2 * sizeof(unsigned), e->stream);
    if (err == cudaSuccess && e->check_err) err = cudaMemsetAsync(e->check_err, 0, 2 * sizeof(unsigned), e->stream);
    if (err == cudaSuccess && e->check_err)
        err = cudaFuncSetAttribute(k_check_state, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)(((2 * NP + 31) / 32) * sizeof(uint32_t)));
    if (err != cudaSuccess) {
        set_error("engine upload: %s", cudaGetErrorString(err));
        cudaStreamSynchronize(e->stream);
        engine_free(e);
        return QPM_ERR_CUDA;
    }
    // no synchronisation: the uploads are stream-ordered before the engine's
    // work; the staging buffer's next user waits for them (pinned_staging)
    if (pinned) pinned_staging_busy(e->stream);
    auto *h = new qpm_engine();
    h->e = e;
    *out = h;
    return QPM_OK;
}

int qpm_engine_destroy(qpm_engine *h) {
    if (!h) return QPM_OK;
    if (h->e->stream && !h->e->owns_stream) cudaStreamSynchronize(h->e->stream);
    engine_free(h->e);
    delete h;
    return QPM_OK;
}

int64_t qpm_engine_device_bytes(const qpm_engine *h) { return h ? h->e->device_bytes : -1; }

// generation 0: init_population, its fitness, statistics and trace row, and
// the planner's draws for generation 1.  An emulated column shard (world > 1,
// no communicator) stops after its fitness scan: the caller exchanges the
// partials (qpm_engine_exchange_from) and calls qpm_engine_init_finish.
static int init_tail(Engine *e) {
    const RunConsts &c = e->c;
    cudaStream_t s = e->stream;
    int rc = fit_finish(e, e->fit, s, nullptr);
    if (rc) return rc;
    if ((rc = launch_select_stats(e, 3, s))) return rc;
    k_copy_best<<<64, 256, 0, s>>>(c, e->st, e->slot_of, e->slot_bin, e->genome, e->bits, e->best_genome,
                                   e->best_bits);
    QPM_LAUNCH_CHECK();
    if (c.algorithm != QPM_ALGO_GWO && (rc = enqueue_planner(e, s))) return rc;  // generation 1's draws
    e->initialized = true;
    e->init_pending = false;
    e->g_done = 0;
    return QPM_OK;
}

int qpm_engine_init(qpm_engine *h) {
    QPM_ARG_CHECK(h, "engine");
    Engine *e = h->e;
    if (e->initialized || e->init_pending) {
        // a second init would rerun init_population with st->g past 0, and the
        // statistics kernel would then write trace row g instead of row 0
        set_error("qpm_engine_init called twice: create a new engine for a new run");
        return QPM_ERR_STATE;
    }
    const RunConsts &c = e->c;
    cudaStream_t s = e->stream;
    k_init_population<<<row_grid(e, c.NP), kRowThreads, 0, s>>>(c, e->genome, e->bits, e->slot_of, e->spare_of,
                                                                 e->slot_tag);
    QPM_LAUNCH_CHECK();
    int rc;
    if (e->sharded()) {
        if ((rc = fit_scan(e, e->bits, e->slot_of, e->fit, s, nullptr))) return rc;
        if (!e->comm) {
            e->init_pending = true;
            return QPM_OK;
        }
        if ((rc = enqueue_exchange(e, 0))) return rc;
    } else if ((rc = launch_fitness(e->prob, &e->fs, e->bits, c.W, e->slot_of, c.NP, e->fit, e->P.fitness_mode, s,
                                    nullptr))) {
        return rc;
    }
    return init_tail(e);
}

int qpm_engine_init_finish(qpm_engine *h) {
    QPM_ARG_CHECK(h, "engine");
    if (!h->e->init_pending) {
        set_error("qpm_engine_init_finish without a pending emulated-shard init");
        return QPM_ERR_STATE;
    }
    return init_tail(h->e);
}

constexpr int64_t kGraphMinGens = 256;  // fresh engines capture graphs from this run length on

// capture `gens` generations into one executable graph (uploaded to the
// device, so its first launch costs no more than a replay)
static int capture_graph(Engine *e, int gens, cudaGraph_t *graph, cudaGraphExec_t *exec) {
    QPM_CUDA_TRY(cudaStreamBeginCapture(e->stream, cudaStreamCaptureModeThreadLocal));
    int launches = 0, rc = QPM_OK;
    for (int t = 0; t < gens && rc == QPM_OK; ++t) {
        e->pdl_trial = t > 0;
        int l = 0;
        rc = enqueue_generation(e, &l);
        launches += l;
    }
    e->pdl_trial = false;
    cudaGraph_t g = nullptr;
    cudaError_t err = cudaStreamEndCapture(e->stream, &g);
    if (rc) {
        if (g) cudaGraphDestroy(g);
        return rc;
    }
    if (err != cudaSuccess) {
        set_error("graph capture: %s", cudaGetErrorString(err));
        return QPM_ERR_CUDA;
    }
    *graph = g;
    QPM_CUDA_TRY(cudaGraphInstantiateWithFlags(exec, g, cudaGraphInstantiateFlagUseNodePriority));
    QPM_CUDA_TRY(cudaGraphUpload(*exec, e->stream));
    e->launches = launches / gens;
    return QPM_OK;
}

// every graph a graph-mode step of n generations replays: the one-generation
// graph, and the graph_gens-generation graph when n reaches it
static int ensure_graphs(Engine *e, int64_t n) {
    int rc;
    const bool use_k = e->graph_gens > 1 && n >= e->graph_gens;
    const bool need_1 = !use_k || n % e->graph_gens != 0;
    if (need_1 && !e->exec && (rc = capture_graph(e, 1, &e->graph, &e->exec))) return rc;
    if (use_k && !e->exec_k && (rc = capture_graph(e, e->graph_gens, &e->graph_k, &e->exec_k))) return rc;
    return QPM_OK;
}

static int step_ready(Engine *e, const char *what) {
    if (e->failed) {
        set_error("%s: the engine's collective failed earlier (communicator aborted); create a new engine", what);
        return QPM_ERR_NCCL;
    }
    if (!e->initialized) {
        set_error("%s before qpm_engine_init", what);
        return QPM_ERR_STATE;
    }
    if (e->world > 1 && !e->comm) {
        set_error("sharded engine without a communicator: drive it with qpm_engine_run_phase");
        return QPM_ERR_STATE;
    }
    return QPM_OK;
}

int qpm_engine_prepare(qpm_engine *h, int64_t n) {
    QPM_ARG_CHECK(h, "engine");
    Engine *e = h->e;
    int rc;
    if ((rc = step_ready(e, "qpm_engine_prepare"))) return rc;
    QPM_ARG_CHECK(n >= 0, "n >= 0");
    if (n == 0) return QPM_OK;
    if ((rc = ensure_graphs(e, n))) return rc;
    QPM_CUDA_TRY(cudaStreamSynchronize(e->stream));
    return QPM_OK;
}

int qpm_engine_step(qpm_engine *h, int64_t n, int use_graph) {
    QPM_ARG_CHECK(h, "engine");
    Engine *e = h->e;
    int rc0;
    if ((rc0 = step_ready(e, "qpm_engine_step"))) return rc0;
    QPM_ARG_CHECK(n >= 0 && e->g_done + n <= e->c.G, "generation count exceeds G");
    if (n == 0) return QPM_OK;
    // A short run on an engine without graphs launches eagerly: PDL already
    // overlaps the launches, so a replayed generation saves only ~3 us
    // against ~0.9 ms of capture, instantiation and teardown (C2, B200,
    // tools/e2e_probe.py: 20 generations 3.0 ms eager vs 3.9 ms with graphs).
    // Both paths run the same kernels in the same order (bit-identical).
    const bool have = e->exec || e->exec_k;
    if (use_graph && !have && n < kGraphMinGens) use_graph = 0;
    if (use_graph) {
        if ((rc0 = ensure_graphs(e, n))) return rc0;
        int64_t t = 0;
        if (e->graph_gens > 1 && n >= e->graph_gens)
            for (; t + e->graph_gens <= n; t += e->graph_gens) {
                QPM_CUDA_TRY(cudaGraphLaunch(e->exec_k, e->stream));
                if ((rc0 = nccl_poll(e))) return rc0;
            }
        for (; t < n; ++t) {
            QPM_CUDA_TRY(cudaGraphLaunch(e->exec, e->stream));
            if ((rc0 = nccl_poll(e))) return rc0;
        }
    } else {
        for (int64_t t = 0; t < n; ++t) {
            int launches = 0;
            int rc = enqueue_generation(e, &launches);
            if (rc) return rc;
            e->launches = launches;
            if ((rc = nccl_poll(e))) return rc;
        }
    }
    e->g_done += n;
    return QPM_OK;
}

int qpm_engine_finalize(qpm_engine *h) {
    QPM_ARG_CHECK(h, "engine");
    Engine *e = h->e;
    if (!e->initialized) {
        set_error("qpm_engine_finalize before qpm_engine_init");
        return QPM_ERR_STATE;
    }
    const RunConsts &c = e->c;
    if (c.algorithm == QPM_ALGO_GWO) return QPM_OK;  // best-ever is already in the result buffer
    k_finalize_best<<<1, kCtaThreads, 0, e->stream>>>(c, e->st, e->fit);
    k_copy_best<<<64, 256, 0, e->stream>>>(c, e->st, e->slot_of, e->slot_bin, e->genome, e->bits, e->best_genome,
                                           e->best_bits);
    k_reset_flag<<<1, 1, 0, e->stream>>>(e->st);
    QPM_LAUNCH_CHECK();
    return QPM_OK;
}

int qpm_engine_generation(const qpm_engine *h, int64_t *g_done) {
    QPM_ARG_CHECK(h && g_done, "engine, g_done");
    *g_done = h->e->g_done;
    return QPM_OK;
}

int qpm_engine_read_trace(qpm_engine *h, int64_t first_row, int64_t n_rows, double *host_rows) {
    QPM_ARG_CHECK(h && host_rows, "engine, out");
    Engine *e = h->e;
    QPM_ARG_CHECK(first_row >= 0 && n_rows >= 0 && first_row + n_rows <= e->c.G + 1, "trace rows");
    QPM_CUDA_TRY(cudaMemcpyAsync(host_rows, e->trace + first_row * 5, sizeof(double) * 5 * n_rows,
                                 cudaMemcpyDeviceToHost, e->stream));
    QPM_CUDA_TRY(cudaStreamSynchronize(e->stream));
    return QPM_OK;
}

// the best individual (and optionally trace rows) through one pinned buffer
// and one synchronisation
static int read_result(Engine *e, int64_t first_row, int64_t n_rows, double *host_rows, double *genome, int8_t *proj,
                       double *fitness) {
    const RunConsts &c = e->c;
    const size_t bg = sizeof(double) * c.Dp, bb = sizeof(uint32_t) * c.W, bt = sizeof(double) * 5 * n_rows;
    const size_t total = bg + bb + sizeof(double) + bt;
    char *pin = pinned_staging(total);
    std::vector<char> pageable;
    if (!pin) {
        pageable.resize(total);
        pin = pageable.data();
    }
    QPM_CUDA_TRY(cudaMemcpyAsync(pin, e->best_genome, bg, cudaMemcpyDeviceToHost, e->stream));
    QPM_CUDA_TRY(cudaMemcpyAsync(pin + bg, e->best_bits, bb, cudaMemcpyDeviceToHost, e->stream));
    QPM_CUDA_TRY(cudaMemcpyAsync(pin + bg + bb, reinterpret_cast<const char *>(e->st) + offsetof(EngineState, best_fit),
                                 sizeof(double), cudaMemcpyDeviceToHost, e->stream));
    if (n_rows)
        QPM_CUDA_TRY(cudaMemcpyAsync(pin + bg + bb + sizeof(double), e->trace + first_row * 5, bt,
                                     cudaMemcpyDeviceToHost, e->stream));
    QPM_CUDA_TRY(cudaStreamSynchronize(e->stream));
    const uint32_t *b = reinterpret_cast<const uint32_t *>(pin + bg);
    if (genome) memcpy(genome, pin, sizeof(double) * c.D);
    if (proj)
        for (int64_t j = 0; j < c.D; ++j) proj[j] = ((b[j >> 5] >> (j & 31)) & 1u) ? -1 : 1;
    if (fitness) memcpy(fitness, pin + bg + bb, sizeof(double));  // run_gwo: best-ever; else the finalize's top-1
    if (n_rows) memcpy(host_rows, pin + bg + bb + sizeof(double), bt);
    return QPM_OK;
}

int qpm_engine_read_best(qpm_engine *h, double *genome, int8_t *proj, double *fitness) {
    QPM_ARG_CHECK(h, "engine");
    return read_result(h->e, 0, 0, nullptr, genome, proj, fitness);
}

int qpm_engine_read_result(qpm_engine *h, int64_t first_row, int64_t n_rows, double *host_rows, double *genome,
                           int8_t *proj, double *fitness) {
    QPM_ARG_CHECK(h, "engine");
    Engine *e = h->e;
    QPM_ARG_CHECK(first_row >= 0 && n_rows >= 0 && first_row + n_rows <= e->c.G + 1 && (n_rows == 0 || host_rows),
                  "trace rows");
    return read_result(e, first_row, n_rows, host_rows, genome, proj, fitness);
}

int qpm_engine_read_population(qpm_engine *h, double *genome, double *fitness) {
    QPM_ARG_CHECK(h, "engine");
    Engine *e = h->e;
    const RunConsts &c = e->c;
    std::vector<int32_t> slots(c.NP);
    std::vector<uint8_t> bin(2 * c.NP);
    QPM_CUDA_TRY(cudaMemcpyAsync(slots.data(), e->slot_of, sizeof(int32_t) * c.NP, cudaMemcpyDeviceToHost, e->stream));
    QPM_CUDA_TRY(cudaMemcpyAsync(bin.data(), e->slot_bin, 2 * c.NP, cudaMemcpyDeviceToHost, e->stream));
    if (fitness)
        QPM_CUDA_TRY(cudaMemcpyAsync(fitness, e->fit, sizeof(double) * c.NP, cudaMemcpyDeviceToHost, e->stream));
    QPM_CUDA_TRY(cudaStreamSynchronize(e->stream));
    if (genome) {
        std::vector<uint32_t> b(c.W);
        for (int64_t i = 0; i < c.NP; ++i) {
            const int64_t slot = slots[i];
            if (bin[slot]) {
                QPM_CUDA_TRY(cudaMemcpy(b.data(), e->bits + slot * c.W, sizeof(uint32_t) * c.W, cudaMemcpyDeviceToHost));
                for (int64_t j = 0; j < c.D; ++j) genome[i * c.D + j] = ((b[j >> 5] >> (j & 31)) & 1u) ? -1.0 : 1.0;
            } else {
                QPM_CUDA_TRY(cudaMemcpyAsync(genome + i * c.D, e->genome + slot * c.Dp, sizeof(double) * c.D,
                                             cudaMemcpyDeviceToHost, e->stream));
            }
        }
        QPM_CUDA_TRY(cudaStreamSynchronize(e->stream));
    }
    return QPM_OK;
}

int qpm_engine_profile(qpm_engine *h, int64_t n, double *stage_ms, int *n_stages, char *names, int name_len) {
    QPM_ARG_CHECK(h && stage_ms && n_stages, "engine, outputs");
    Engine *e = h->e;
    if (!e->initialized) {
        set_error("qpm_engine_profile before qpm_engine_init");
        return QPM_ERR_STATE;
    }
    QPM_ARG_CHECK(n >= 1 && e->g_done + n <= e->c.G, "generation count exceeds G");
    StageMarks pm;
    for (int t = 0; t <= kMaxStages; ++t) QPM_CUDA_TRY(cudaEventCreate(&pm.ev[t]));
    double acc[kMaxStages] = {0};
    int stages = 0;
    int rc = QPM_OK;
    for (int64_t t = 0; t < n && rc == QPM_OK; ++t) {
        pm.n = 0;
        int launches = 0;
        rc = enqueue_generation(e, &launches, &pm);
        if (rc) break;
        cudaError_t err = cudaEventSynchronize(pm.ev[pm.n - 1]);
        if (err != cudaSuccess) {
            set_error("profile sync: %s", cudaGetErrorString(err));
            rc = QPM_ERR_CUDA;
            break;
        }
        stages = pm.n - 1;
        for (int k = 0; k < stages; ++k) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, pm.ev[k], pm.ev[k + 1]);
            acc[k] += ms;
        }
        e->g_done += 1;
    }
    for (int t = 0; t <= kMaxStages; ++t) cudaEventDestroy(pm.ev[t]);
    if (rc) return rc;
    *n_stages = stages;
    for (int k = 0; k < stages; ++k) {
        stage_ms[k] = acc[k] / (double)n;
        if (names && name_len > 0) {
            strncpy(names + k * name_len, pm.name[k], name_len - 1);
            names[k * name_len + name_len - 1] = 0;
        }
    }
    return QPM_OK;
}

int qpm_nccl_unique_id(uint8_t *id_out) {
    QPM_ARG_CHECK(id_out, "id_out");
    int rc = nccl_load();
    if (rc) return rc;
    ncclUniqueIdPod id;
    const int r = g_nccl.get_id(&id);
    if (r != 0) {
        set_error("ncclGetUniqueId: %s", g_nccl.err(r));
        return QPM_ERR_NCCL;
    }
    memcpy(id_out, id.internal, sizeof(id.internal));
    return QPM_OK;
}

int qpm_engine_set_comm(qpm_engine *h, int rank, int world, const uint8_t *id) {
    QPM_ARG_CHECK(h && id, "engine, id");
    Engine *e = h->e;
    QPM_ARG_CHECK(rank == e->rank && world == e->world, "rank / world must match the engine's shard_rank / shard_world");
    QPM_ARG_CHECK(!e->exec && !e->initialized, "the communicator must be set before qpm_engine_init");
    int rc;
    if ((rc = nccl_load())) return rc;
    ncclUniqueIdPod uid;
    memcpy(uid.internal, id, sizeof(uid.internal));
    if (!e->gpart) {  // one rank: the sharded flow needs its partial buffers too
        QPM_ARG_CHECK(e->P.fitness_mode == QPM_MODE_FAST, "the collective path scores in fast mode");
        if ((rc = dalloc(e, &e->gpart, (size_t)e->world * gpart_slot(e))) ||
            (rc = dalloc(e, &e->ggains, (size_t)e->c.NP * e->prob->n_wl)))
            return rc;
    }
    const int r = g_nccl.init_rank(&e->comm, world, uid, rank);
    if (r != 0) {
        e->comm = nullptr;
        set_error("ncclCommInitRank: %s", g_nccl.err(r));
        return QPM_ERR_NCCL;
    }
    return QPM_OK;
}

int qpm_engine_columns(const qpm_engine *h, int64_t *g0, int64_t *d) {
    QPM_ARG_CHECK(h && g0 && d, "engine, out");
    *g0 = h->e->c.g0;
    *d = h->e->c.D;
    return QPM_OK;
}

int qpm_engine_phases(const qpm_engine *h) { return h ? phase_count(h->e) : -1; }

int qpm_engine_run_phase(qpm_engine *h, int phase) {
    QPM_ARG_CHECK(h, "engine");
    Engine *e = h->e;
    if (!e->initialized) {
        set_error("qpm_engine_run_phase before qpm_engine_init");
        return QPM_ERR_STATE;
    }
    const int np = phase_count(e);
    QPM_ARG_CHECK(phase >= 0 && phase < np, "phase index");
    QPM_ARG_CHECK(e->g_done < e->c.G, "generation count exceeds G");
    int n = 0;
    int rc = enqueue_phase(e, phase, &n, nullptr);
    if (rc) return rc;
    if (phase == np - 1) e->g_done += 1;
    return QPM_OK;
}

int qpm_engine_exchange_from(qpm_engine *dst, qpm_engine *src, int phase) {
    QPM_ARG_CHECK(dst && src, "engines");
    (void)phase;  // every exchange moves the same buffer: the scanning rank's partial slot
    Engine *d = dst->e, *s = src->e;
    QPM_ARG_CHECK(d->world > 1 && d->world == s->world && d->c.NP == s->c.NP && d->SB_slot == s->SB_slot &&
                      d->rank != s->rank,
                  "engines of one sharded run");
    const size_t n = gpart_slot(s);
    QPM_CUDA_TRY(cudaStreamSynchronize(s->stream));
    QPM_CUDA_TRY(cudaMemcpyAsync(d->gpart + s->rank * n, s->gpart + s->rank * n, sizeof(double) * n,
                                 cudaMemcpyDeviceToDevice, d->stream));
    QPM_CUDA_TRY(cudaStreamSynchronize(d->stream));
    return QPM_OK;
}

int qpm_engine_wait(qpm_engine *h, int64_t timeout_ms) {
    QPM_ARG_CHECK(h, "engine");
    Engine *e = h->e;
    if (e->failed) {
        set_error("qpm_engine_wait: the engine's collective failed earlier (communicator aborted)");
        return QPM_ERR_NCCL;
    }
    // poll the stream and, on the collective path, NCCL's asynchronous error
    // state; on timeout abort the communicator so the stuck kernels exit
    // instead of hanging every later synchronize
    const auto t0 = std::chrono::steady_clock::now();
    for (int spin = 0;; ++spin) {
        const cudaError_t q = cudaStreamQuery(e->stream);
        if (q == cudaSuccess) return nccl_poll(e);
        if (q != cudaErrorNotReady) {
            set_error("qpm_engine_wait: %s", cudaGetErrorString(q));
            return QPM_ERR_CUDA;
        }
        int rc;
        if ((rc = nccl_poll(e))) return rc;
        const auto ms =
            std::chrono::duration_cast<std::chrono::milliseconds>(std::chrono::steady_clock::now() - t0).count();
        if (timeout_ms >= 0 && ms > timeout_ms) {
            if (e->comm) {
                g_nccl.abort(e->comm);
                e->comm = nullptr;
                e->failed = true;
                set_error("qpm_engine_wait: rank %d of %d timed out after %lld ms waiting for the generation "
                          "(a peer stopped participating in the collective); communicator aborted",
                          e->rank, e->world, (long long)ms);
                return QPM_ERR_NCCL;
            }
            set_error("qpm_engine_wait: timed out after %lld ms", (long long)ms);
            return QPM_ERR_STATE;
        }
        if (spin > 64) std::this_thread::sleep_for(std::chrono::microseconds(200));
    }
}

int qpm_engine_partials_info(const qpm_engine *h, int64_t *slot_doubles, int *world, int *rank) {
    QPM_ARG_CHECK(h, "engine");
    const Engine *e = h->e;
    if (slot_doubles) *slot_doubles = e->gpart ? (int64_t)gpart_slot(e) : 0;
    if (world) *world = e->world;
    if (rank) *rank = e->rank;
    return QPM_OK;
}

int qpm_engine_partials_read(qpm_engine *h, double *host_out) {
    QPM_ARG_CHECK(h && host_out, "engine, out");
    Engine *e = h->e;
    QPM_ARG_CHECK(e->gpart != nullptr, "not a sharded engine");
    const size_t n = gpart_slot(e);
    QPM_CUDA_TRY(cudaMemcpyAsync(host_out, e->gpart + e->rank * n, sizeof(double) * n, cudaMemcpyDeviceToHost,
                                 e->stream));
    QPM_CUDA_TRY(cudaStreamSynchronize(e->stream));
    return QPM_OK;
}

int qpm_engine_partials_write(qpm_engine *h, int rank, const double *host_in) {
    QPM_ARG_CHECK(h && host_in, "engine, in");
    Engine *e = h->e;
    QPM_ARG_CHECK(e->gpart != nullptr, "not a sharded engine");
    QPM_ARG_CHECK(rank >= 0 && rank < e->world && rank != e->rank, "a peer rank of this engine's run");
    const size_t n = gpart_slot(e);
    QPM_CUDA_TRY(cudaMemcpyAsync(e->gpart + rank * n, host_in, sizeof(double) * n, cudaMemcpyHostToDevice,
                                 e->stream));
    QPM_CUDA_TRY(cudaStreamSynchronize(e->stream));
    return QPM_OK;
}

static int64_t ckpt_bytes(const Engine *e) {
    const RunConsts &c = e->c;
    return (int64_t)sizeof(CkptHeader) + (int64_t)sizeof(EngineState) + c.NP * 8 /* fit */ +
           (e->g_done + 1) * 5 * 8 /* trace */ + c.NP /* bin flags */ + c.NP * c.W * 4 + c.NP * c.Dp * 8 +
           c.Dp * 8 + c.W * 4 /* best row */;
}

int64_t qpm_engine_checkpoint_bytes(const qpm_engine *h) { return h ? ckpt_bytes(h->e) : -1; }

int qpm_engine_checkpoint(qpm_engine *h, void *host_buf, int64_t bytes) {
    QPM_ARG_CHECK(h && host_buf, "engine, buffer");
    Engine *e = h->e;
    const RunConsts &c = e->c;
    if (!e->initialized) {
        set_error("qpm_engine_checkpoint before qpm_engine_init");
        return QPM_ERR_STATE;
    }
    QPM_ARG_CHECK(bytes >= ckpt_bytes(e), "buffer smaller than qpm_engine_checkpoint_bytes()");
    QPM_CUDA_TRY(cudaStreamSynchronize(e->stream));
    if (e->side) QPM_CUDA_TRY(cudaStreamSynchronize(e->side));
    char *p = static_cast<char *>(host_buf);
    CkptHeader hd{};
    memcpy(hd.magic, "QPMCKPT1", 8);
    hd.version = 1;
    hd.algorithm = c.algorithm;
    hd.fitness_mode = e->P.fitness_mode;
    hd.rank = e->rank;
    hd.world = e->world;
    hd.NP = c.NP, hd.D = c.D, hd.W = c.W, hd.G = c.G, hd.seed = (int64_t)c.seed, hd.g0 = c.g0, hd.g_done = e->g_done;
    memcpy(p, &hd, sizeof(hd));
    p += sizeof(hd);
    QPM_CUDA_TRY(cudaMemcpy(p, e->st, sizeof(EngineState), cudaMemcpyDeviceToHost));
    p += sizeof(EngineState);
    QPM_CUDA_TRY(cudaMemcpy(p, e->fit, c.NP * 8, cudaMemcpyDeviceToHost));
    p += c.NP * 8;
    QPM_CUDA_TRY(cudaMemcpy(p, e->trace, (e->g_done + 1) * 5 * 8, cudaMemcpyDeviceToHost));
    p += (e->g_done + 1) * 5 * 8;
    const size_t gb = (size_t)c.NP * c.Dp * 8, bb = (size_t)c.NP * c.W * 4;
    double *tg = (double *)dev_cache_alloc(gb);
    uint32_t *tb = (uint32_t *)dev_cache_alloc(bb);
    uint8_t *tf = (uint8_t *)dev_cache_alloc((size_t)c.NP);
    int rc = QPM_OK;
    if (!tg || !tb || !tf) {
        set_error("out of device memory for the checkpoint staging");
        rc = QPM_ERR_CUDA;
    } else {
        k_gather_rows<<<dim3(4, (unsigned)c.NP), 256, 0, e->stream>>>(c, e->slot_of, e->slot_bin, e->genome, e->bits, tg,
                                                                     tb, tf);
        if (cudaGetLastError() != cudaSuccess || cudaMemcpyAsync(p, tf, c.NP, cudaMemcpyDeviceToHost, e->stream) ||
            cudaMemcpyAsync(p + c.NP, tb, bb, cudaMemcpyDeviceToHost, e->stream) ||
            cudaMemcpyAsync(p + c.NP + bb, tg, gb, cudaMemcpyDeviceToHost, e->stream) ||
            cudaMemcpyAsync(p + c.NP + bb + gb, e->best_genome, c.Dp * 8, cudaMemcpyDeviceToHost, e->stream) ||
            cudaMemcpyAsync(p + c.NP + bb + gb + c.Dp * 8, e->best_bits, c.W * 4, cudaMemcpyDeviceToHost, e->stream) ||
            cudaStreamSynchronize(e->stream) != cudaSuccess) {
            set_error("checkpoint copy failed");
            rc = QPM_ERR_CUDA;
        }
    }
    cudaStreamSynchronize(e->stream);
    dev_cache_release(tg, gb);
    dev_cache_release(tb, bb);
    dev_cache_release(tf, (size_t)c.NP);
    return rc;
}

int qpm_engine_restore(qpm_engine *h, const void *host_buf, int64_t bytes) {
    QPM_ARG_CHECK(h && host_buf, "engine, buffer");
    Engine *e = h->e;
    const RunConsts &c = e->c;
    if (e->initialized || e->init_pending) {
        set_error("qpm_engine_restore needs a freshly created engine (not initialised)");
        return QPM_ERR_STATE;
    }
    const char *p = static_cast<const char *>(host_buf);
    QPM_ARG_CHECK(bytes >= (int64_t)sizeof(CkptHeader), "buffer too small for a checkpoint");
    CkptHeader hd;
    memcpy(&hd, p, sizeof(hd));
    QPM_ARG_CHECK(memcmp(hd.magic, "QPMCKPT1", 8) == 0 && hd.version == 1, "not a qpm engine checkpoint");
    QPM_ARG_CHECK(hd.algorithm == c.algorithm && hd.fitness_mode == e->P.fitness_mode && hd.NP == c.NP &&
                      hd.D == c.D && hd.W == c.W && hd.G == c.G && hd.seed == (int64_t)c.seed && hd.g0 == c.g0 &&
                      hd.rank == e->rank && hd.world == e->world,
                  "checkpoint of a different run (algorithm, mode, NP, D, G, seed or shard)");
    QPM_ARG_CHECK(hd.g_done >= 0 && hd.g_done <= c.G, "checkpoint generation outside [0, G]");
    e->g_done = hd.g_done;
    QPM_ARG_CHECK(bytes >= ckpt_bytes(e), "truncated checkpoint");
    p += sizeof(hd);
    EngineState hs;
    memcpy(&hs, p, sizeof(hs));
    p += sizeof(hs);
    hs.g_plan = hs.g;  // the planner re-draws the next generation below
    QPM_CUDA_TRY(cudaMemcpyAsync(e->st, &hs, sizeof(hs), cudaMemcpyHostToDevice, e->stream));
    QPM_CUDA_TRY(cudaMemcpyAsync(e->fit, p, c.NP * 8, cudaMemcpyHostToDevice, e->stream));
    p += c.NP * 8;
    QPM_CUDA_TRY(cudaMemcpyAsync(e->trace, p, (hd.g_done + 1) * 5 * 8, cudaMemcpyHostToDevice, e->stream));
    p += (hd.g_done + 1) * 5 * 8;
    const size_t gb = (size_t)c.NP * c.Dp * 8, bb = (size_t)c.NP * c.W * 4;
    double *tg = (double *)dev_cache_alloc(gb);
    uint32_t *tb = (uint32_t *)dev_cache_alloc(bb);
    uint8_t *tf = (uint8_t *)dev_cache_alloc((size_t)c.NP);
    int rc = QPM_OK;
    if (!tg || !tb || !tf) {
        set_error("out of device memory for the checkpoint staging");
        rc = QPM_ERR_CUDA;
    } else if (cudaMemcpyAsync(tf, p, c.NP, cudaMemcpyHostToDevice, e->stream) ||
               cudaMemcpyAsync(tb, p + c.NP, bb, cudaMemcpyHostToDevice, e->stream) ||
               cudaMemcpyAsync(tg, p + c.NP + bb, gb, cudaMemcpyHostToDevice, e->stream) ||
               cudaMemcpyAsync(e->best_genome, p + c.NP + bb + gb, c.Dp * 8, cudaMemcpyHostToDevice, e->stream) ||
               cudaMemcpyAsync(e->best_bits, p + c.NP + bb + gb + c.Dp * 8, c.W * 4, cudaMemcpyHostToDevice,
                               e->stream)) {
        set_error("restore copy failed");
        rc = QPM_ERR_CUDA;
    } else {
        k_scatter_rows<<<dim3(4, (unsigned)c.NP), 256, 0, e->stream>>>(c, tg, tb, tf, e->slot_of, e->spare_of,
                                                                      e->slot_tag, e->slot_bin, e->genome, e->bits);
        if (cudaGetLastError() != cudaSuccess) {
            set_error("restore scatter launch failed");
            rc = QPM_ERR_CUDA;
        }
    }
    if (rc == QPM_OK && c.algorithm != QPM_ALGO_GWO) rc = enqueue_planner(e, e->stream);  // the next generation's draws
    if (cudaStreamSynchronize(e->stream) != cudaSuccess && rc == QPM_OK) {
        set_error("restore failed on the device");
        rc = QPM_ERR_CUDA;
    }
    dev_cache_release(tg, gb);
    dev_cache_release(tb, bb);
    dev_cache_release(tf, (size_t)c.NP);
    if (rc) return rc;
    e->initialized = true;
    e->init_pending = false;
    return QPM_OK;
}

int qpm_engine_check_status(qpm_engine *h, uint32_t *flags, uint32_t *detail) {
    QPM_ARG_CHECK(h && flags, "engine, flags");
    Engine *e = h->e;
    if (!e->check_err) {
        set_error("qpm_engine_check_status: library built without QPM_CHECKS");
        return QPM_ERR_STATE;
    }
    uint32_t w[2];
    QPM_CUDA_TRY(cudaMemcpyAsync(w, e->check_err, sizeof(w), cudaMemcpyDeviceToHost, e->stream));
    QPM_CUDA_TRY(cudaStreamSynchronize(e->stream));
    *flags = w[0];
    if (detail) *detail = w[1];
    return QPM_OK;
}

int qpm_engine_cand_ptr(qpm_engine *h, double **cand_dev) {
    QPM_ARG_CHECK(h && cand_dev, "engine, out");
    *cand_dev = h->e->cand;
    return QPM_OK;
}

int qpm_engine_stream(qpm_engine *h, void **stream) {
    QPM_ARG_CHECK(h && stream, "engine, out");
    *stream = (void *)h->e->stream;
    return QPM_OK;
}

int qpm_engine_launches_per_generation(const qpm_engine *h) {
    if (!h) return -1;
    if (h->e->launches) return h->e->launches;
    const int a = h->e->c.algorithm;
    return a == QPM_ALGO_HYBRID ? 10 : 6;  // single-rank counts (enqueue_phase)
}

int qpm_engine_fitness_ptr(qpm_engine *h, double **fit_dev) {
    QPM_ARG_CHECK(h && fit_dev, "engine, out");
    *fit_dev = h->e->fit;
    return QPM_OK;
}

// development timeline (-DQPM_TRACE builds; -2 otherwise): reset, or copy
// this translation unit's log [kTraceIds][kTraceLen][3] (globaltimer ns) and
// per-id launch counts.  Not part of include/qpm_b200.h.
int qpm_dev_trace_engine(int reset, unsigned long long *log, unsigned int *launches) {
#ifdef QPM_TRACE
    if (reset == 2) return qpm::trace_stamps_tu(log);  // intra-kernel stamps [kTraceIds][64][8]
    if (reset) return qpm::trace_reset_tu();
    return qpm::trace_read_tu(log, launches);
#else
    (void)reset;
    (void)log;
    (void)launches;
    return -2;
#endif
}

}  // extern "C"
