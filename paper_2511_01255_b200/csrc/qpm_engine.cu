// qpm_engine.cu -- device-resident HWSDA generation loop (run_hybrid /
// run_de / run_gwo, optimizer.py:400-592) for one B200.
//
// HBM layout (one engine):
//   genome  f64 [2 NP][Dp]   slot pool; individual i lives in slot_of[i],
//                            its trial / candidate is written to spare_of[i]
//                            and acceptance swaps the two ids (no row copies)
//   bits    u32 [2 NP][W]    sign bits of each slot (bit 1 <=> gene < 0)
//   fit     f64 [NP]         fitness of individual i;  cand f64 [NP]
//   keys    u64 [NP]         fold_key(seed, g, i) of the current generation
//   picks   int4 [NP]        r1, r2, r3 and the index-draw count m (DE)
//   sched   f64 [G+1][8]     per-generation scalars, host-computed
//   trace   f64 [G+1][5]     (g, best, mean, F|a, pop_std) rows
//   state   EngineState      g, F, window, leaders, best-ever bookkeeping
// Dp = W * 32 with W a multiple of 4, so rows start on 512-byte boundaries.
//
// Every generation is a fixed launch sequence that reads g and F from
// device memory, so one CUDA graph replays it for all generations with no
// host round trip.  Decisions reproduce the reference bit-for-bit given the
// same fitness values:
//   - stream positions follow Appendix A of SURVEY.md (de_mutate rejection
//     draws 0..m-1, j_rand at m, mask m+1..m+D, wolf block from m+1+D);
//   - DE arithmetic x_r1 + F (x_r2 - x_r3) is unfused (-fmad=false);
//   - u < p comparisons are exact integer compares on the 53-bit mantissa;
//   - np.mean / np.std use a replica of numpy's pairwise summation.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "qpm_common.cuh"
#include "qpm_internal.cuh"

namespace qpm {

constexpr int kMaxLeaders = 8;
constexpr int kMaxWindow = 256;
constexpr int kRowThreads = 256;   // threads per row-block in the elementwise kernels
constexpr int kGenesPerThread = 4; // genes per thread (strided by kRowThreads)
constexpr int kGenesPerBlock = kRowThreads * kGenesPerThread;
constexpr int kStatsThreads = 512;

struct EngineState {
    int64_t g;  // generation computed next (0 before init)
    double F;
    double best_prev;
    double baseline_std;
    double best_fit;  // run_gwo best-ever fitness
    int32_t best_idx;
    int32_t best_flag;
    int32_t win_len;
    int32_t pad0;
    int32_t leaders[kMaxLeaders];
    uint64_t thr_plus[kMaxLeaders + 1];  // u_plus < p_plus(count) thresholds
    uint8_t win[kMaxWindow];
};

struct RunConsts {
    int algorithm;
    int64_t NP, D, Dp, W, G;
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
    int64_t n_leaf;  // pairwise-sum leaves of an NP-vector
};

// ---------------------------------------------------------------- init
__global__ void __launch_bounds__(kRowThreads) k_init_population(RunConsts c, double *__restrict__ genome,
                                                                 uint32_t *__restrict__ bits,
                                                                 int32_t *__restrict__ slot_of,
                                                                 int32_t *__restrict__ spare_of) {
    const int64_t i = blockIdx.y;
    const uint64_t key = fold_key3(c.seed, 0, (uint64_t)i);  // stream (seed, 0, i), optimizer.py:223
    double *row = genome + i * c.Dp;
    uint32_t *brow = bits + i * c.W;
#pragma unroll
    for (int it = 0; it < kGenesPerThread; ++it) {
        const int64_t j = (int64_t)blockIdx.x * kGenesPerBlock + it * kRowThreads + threadIdx.x;
        bool neg = false;
        if (j < c.D) {
            const double x = c.x_lo + draw_u(key, (uint64_t)j) * c.x_span;
            row[j] = x;
            neg = !(x >= 0.0);
        }
        const uint32_t word = __ballot_sync(0xffffffffu, neg);
        if ((threadIdx.x & 31) == 0 && j < c.Dp) brow[j >> 5] = word;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        slot_of[i] = (int32_t)i;
        spare_of[i] = (int32_t)(c.NP + i);
    }
}

// ---------------------------------------------------------------- DE
// de_mutate index draws (optimizer.py:229-247) + j_rand (optimizer.py:258)
__global__ void k_de_draws(RunConsts c, const EngineState *__restrict__ st, uint64_t *__restrict__ keys,
                           int4 *__restrict__ picks, int32_t *__restrict__ jrand) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= c.NP) return;
    const uint64_t key = fold_key3(c.seed, (uint64_t)st->g, (uint64_t)i);
    keys[i] = key;
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
    picks[i] = make_int4((int)r[0], (int)r[1], (int)r[2], (int)m);
    jrand[i] = (int32_t)randint(key, m, c.D);
}

// de_crossover (optimizer.py:250-262): trial_j = (u_j <= CR or j == j_rand)
// ? x_r1 + F (x_r2 - x_r3) : x_i, written to the spare slot with its bits.
__global__ void __launch_bounds__(kRowThreads) k_de_trial(RunConsts c, const EngineState *__restrict__ st,
                                                          const uint64_t *__restrict__ keys,
                                                          const int4 *__restrict__ picks,
                                                          const int32_t *__restrict__ jrand,
                                                          const int32_t *__restrict__ slot_of,
                                                          const int32_t *__restrict__ spare_of,
                                                          double *__restrict__ genome, uint32_t *__restrict__ bits) {
    const int64_t i = blockIdx.y;
    const int4 pk = picks[i];
    const uint64_t key = keys[i];
    const int64_t jr = jrand[i];
    const double F = st->F;
    const double *xi = genome + (int64_t)slot_of[i] * c.Dp;
    const double *x1 = genome + (int64_t)slot_of[pk.x] * c.Dp;
    const double *x2 = genome + (int64_t)slot_of[pk.y] * c.Dp;
    const double *x3 = genome + (int64_t)slot_of[pk.z] * c.Dp;
    const int64_t out_slot = spare_of[i];
    double *out = genome + out_slot * c.Dp;
    uint32_t *bout = bits + out_slot * c.W;
    const uint64_t base = (uint64_t)pk.w + 1;
#pragma unroll
    for (int it = 0; it < kGenesPerThread; ++it) {
        const int64_t j = (int64_t)blockIdx.x * kGenesPerBlock + it * kRowThreads + threadIdx.x;
        bool neg = false;
        if (j < c.D) {
            const bool take = draw53(key, base + (uint64_t)j) < c.cr_thr || j == jr;
            double v;
            if (take) {
                const double d = x2[j] - x3[j];
                v = x1[j] + F * d;
            } else {
                v = xi[j];
            }
            out[j] = v;
            neg = !(v >= 0.0);
        }
        const uint32_t word = __ballot_sync(0xffffffffu, neg);
        if ((threadIdx.x & 31) == 0 && j < c.Dp) bout[j >> 5] = word;
    }
}

// ---------------------------------------------------------------- selection
// de_select (optimizer.py:265-269): strict >, ties keep the target.  With
// skip_leaders the k current leaders are not movers (optimizer.py:454).
__global__ void k_select(RunConsts c, const EngineState *__restrict__ st, int skip_leaders, int unconditional,
                         const double *__restrict__ cand, double *__restrict__ fit, int32_t *__restrict__ slot_of,
                         int32_t *__restrict__ spare_of, uint8_t *__restrict__ accepted) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= c.NP) return;
    if (skip_leaders) {
        for (int t = 0; t < c.k; ++t)
            if (st->leaders[t] == i) {
                accepted[i] = 0;
                return;
            }
    }
    const double f = cand[i];
    if (unconditional || f > fit[i]) {
        const int32_t a = slot_of[i];
        slot_of[i] = spare_of[i];
        spare_of[i] = a;
        fit[i] = f;
        accepted[i] = 1;
    } else {
        accepted[i] = 0;
    }
}

// ---------------------------------------------------------------- GWO (hybrid)
// gwo_discrete_update (optimizer.py:335-376), draws taken lazily: only the
// rows of the 6 x D block a gene's branch reads (positions are unchanged).
__global__ void __launch_bounds__(kRowThreads) k_gwo_discrete(RunConsts c, const EngineState *__restrict__ st,
                                                              const double *__restrict__ sched,
                                                              const uint64_t *__restrict__ keys,
                                                              const int4 *__restrict__ picks,
                                                              const int32_t *__restrict__ slot_of,
                                                              const int32_t *__restrict__ spare_of,
                                                              uint32_t *__restrict__ bits) {
    const int64_t i = blockIdx.y;
    const int k = c.k;
    for (int t = 0; t < k; ++t)
        if (st->leaders[t] == i) return;  // leaders do not move
    const int64_t g = st->g;
    const double *sg = sched + g * QPM_SCHED_COLS;
    const uint64_t thr_sl = lt_threshold(sg[QPM_SCHED_P_SL]);
    const uint64_t thr_dist = lt_threshold(sg[QPM_SCHED_P_DIST]);
    const uint64_t thr_flip = lt_threshold(sg[QPM_SCHED_P_FLIP]);
    const bool early = sg[QPM_SCHED_EARLY] != 0.0;
    const uint64_t key = keys[i];
    const uint64_t base = (uint64_t)picks[i].w + 1 + (uint64_t)c.D;
    const uint64_t D = (uint64_t)c.D;
    const uint32_t *lrow[kMaxLeaders];
    for (int t = 0; t < k; ++t) lrow[t] = bits + (int64_t)slot_of[st->leaders[t]] * c.W;
    uint32_t *bout = bits + (int64_t)spare_of[i] * c.W;
    const uint64_t half = 1ULL << 52;  // u_state < 0.5
#pragma unroll
    for (int it = 0; it < kGenesPerThread; ++it) {
        const int64_t j = (int64_t)blockIdx.x * kGenesPerBlock + it * kRowThreads + threadIdx.x;
        bool neg = false;
        if (j < c.D) {
            const int64_t wi = j >> 5;
            const uint32_t bit = (uint32_t)(j & 31);
            int cnt_plus = 0;
            for (int t = 0; t < k; ++t) cnt_plus += ((lrow[t][wi] >> bit) & 1u) ^ 1u;
            const uint64_t jj = (uint64_t)j;
            int state;
            if (draw53(key, base + jj) < thr_sl) {
                // social learning: copy leader min(int(u_pick k), k - 1)
                const double up = draw_u(key, base + D + jj);
                int pick = (int)(up * (double)k);
                pick = pick < k - 1 ? pick : k - 1;
                state = ((lrow[pick][wi] >> bit) & 1u) ? -1 : 1;
            } else if (early) {
                if (draw53(key, base + 2 * D + jj) < thr_dist)
                    state = draw53(key, base + 3 * D + jj) < half ? 1 : -1;
                else
                    state = draw53(key, base + 4 * D + jj) < st->thr_plus[cnt_plus] ? 1 : -1;
            } else {
                int maj;
                if (2 * cnt_plus > k)
                    maj = 1;
                else if (2 * cnt_plus < k)
                    maj = -1;
                else
                    maj = draw53(key, base + 3 * D + jj) < half ? 1 : -1;
                state = draw53(key, base + 5 * D + jj) < thr_flip ? -maj : maj;
            }
            neg = state < 0;
        }
        const uint32_t word = __ballot_sync(0xffffffffu, neg);
        if ((threadIdx.x & 31) == 0 && j < c.Dp) bout[j >> 5] = word;
    }
}

// accepted wolves: genome = +/-1.0 from their bits (optimizer.py:376)
__global__ void __launch_bounds__(kRowThreads) k_materialize(RunConsts c, const uint8_t *__restrict__ accepted,
                                                             const int32_t *__restrict__ slot_of,
                                                             const uint32_t *__restrict__ bits,
                                                             double *__restrict__ genome) {
    const int64_t i = blockIdx.y;
    if (!accepted[i]) return;
    const int64_t slot = slot_of[i];
    const uint32_t *br = bits + slot * c.W;
    double *row = genome + slot * c.Dp;
#pragma unroll
    for (int it = 0; it < kGenesPerThread; ++it) {
        const int64_t j = (int64_t)blockIdx.x * kGenesPerBlock + it * kRowThreads + threadIdx.x;
        if (j < c.D) row[j] = ((br[j >> 5] >> (j & 31)) & 1u) ? -1.0 : 1.0;
    }
}

// ---------------------------------------------------------------- GWO (run_gwo)
__global__ void k_keys(RunConsts c, const EngineState *__restrict__ st, uint64_t *__restrict__ keys) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < c.NP) keys[i] = fold_key3(c.seed, (uint64_t)st->g, (uint64_t)i);
}

// gwo_reference_update (optimizer.py:302-332) with the three ranked leaders
__global__ void __launch_bounds__(kRowThreads) k_gwo_continuous(RunConsts c, const EngineState *__restrict__ st,
                                                                const double *__restrict__ sched,
                                                                const uint64_t *__restrict__ keys,
                                                                const int32_t *__restrict__ slot_of,
                                                                const int32_t *__restrict__ spare_of,
                                                                double *__restrict__ genome,
                                                                uint32_t *__restrict__ bits) {
    const int64_t i = blockIdx.y;
    for (int t = 0; t < 3; ++t)
        if (st->leaders[t] == i) return;
    const double a = sched[st->g * QPM_SCHED_COLS + QPM_SCHED_A_NOW];
    const double two_a = 2.0 * a;
    const uint64_t key = keys[i];
    const uint64_t D = (uint64_t)c.D;
    const double *x = genome + (int64_t)slot_of[i] * c.Dp;
    const double *L0 = genome + (int64_t)slot_of[st->leaders[0]] * c.Dp;
    const double *L1 = genome + (int64_t)slot_of[st->leaders[1]] * c.Dp;
    const double *L2 = genome + (int64_t)slot_of[st->leaders[2]] * c.Dp;
    const int64_t out_slot = spare_of[i];
    double *out = genome + out_slot * c.Dp;
    uint32_t *bout = bits + out_slot * c.W;
#pragma unroll
    for (int it = 0; it < kGenesPerThread; ++it) {
        const int64_t j = (int64_t)blockIdx.x * kGenesPerBlock + it * kRowThreads + threadIdx.x;
        bool neg = false;
        if (j < c.D) {
            const uint64_t jj = (uint64_t)j;
            const double xj = x[j];
            const double Lm[3] = {L0[j], L1[j], L2[j]};
            double moved[3];
#pragma unroll
            for (int m = 0; m < 3; ++m) {
                const double r1 = draw_u(key, 2 * m * D + jj);
                const double r2 = draw_u(key, 2 * m * D + D + jj);
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
}

// ---------------------------------------------------------------- stats
// numpy pairwise sum of v[0..n): leaves (precomputed on the host, in order)
// summed in parallel, then the split tree combined by one thread.
__device__ double block_pairwise(const double *v, int64_t n, const int64_t *leaf_off, int64_t n_leaf,
                                 double *leafsum) {
    for (int64_t l = threadIdx.x; l < n_leaf; l += blockDim.x) {
        const int64_t off = leaf_off[l];
        const int64_t len = (l + 1 < n_leaf ? leaf_off[l + 1] : n) - off;
        leafsum[l] = pairwise_leaf(v + off, len);
    }
    __syncthreads();
    __shared__ double result;
    if (threadIdx.x == 0) {
        struct Frame {
            int64_t n;
            int state;
            double left;
        };
        Frame stk[48];
        int top = 0;
        stk[0] = {n, 0, 0.0};
        double ret = 0.0;
        int64_t next = 0;
        while (top >= 0) {
            Frame &f = stk[top];
            if (f.n <= 128) {
                ret = leafsum[next++];
                --top;
                continue;
            }
            int64_t n2 = f.n / 2;
            n2 -= n2 % 8;
            if (f.state == 0) {
                f.state = 1;
                stk[top + 1] = {n2, 0, 0.0};
                ++top;
            } else if (f.state == 1) {
                f.left = ret;
                f.state = 2;
                stk[top + 1] = {f.n - n2, 0, 0.0};
                ++top;
            } else {
                ret = f.left + ret;
                --top;
            }
        }
        result = ret;
    }
    __syncthreads();
    return result;
}

// np.max / np.mean / np.std of the fitness vector, the convergence window,
// adaptive_f_update (optimizer.py:277-299, 469-485) and the trace row; or,
// for run_gwo, the a-coefficient row and best-ever tracking (optimizer.py:586-589).
__global__ void __launch_bounds__(kStatsThreads) k_stats(RunConsts c, EngineState *__restrict__ st,
                                                         const double *__restrict__ sched,
                                                         const double *__restrict__ fit,
                                                         double *__restrict__ scratch,
                                                         const int64_t *__restrict__ leaf_off,
                                                         double *__restrict__ leafsum, double *__restrict__ trace) {
    const int64_t n = c.NP;
    // max with its lowest index, and min
    double mx = -INFINITY, mn = INFINITY;
    int64_t amx = n;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const double v = fit[i];
        if (v > mx || (v == mx && i < amx)) {
            mx = v;
            amx = i;
        }
        mn = v < mn ? v : mn;
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
    __shared__ double s_mx[kStatsThreads / 32], s_mn[kStatsThreads / 32];
    __shared__ int64_t s_am[kStatsThreads / 32];
    if ((threadIdx.x & 31) == 0) {
        s_mx[threadIdx.x >> 5] = mx;
        s_mn[threadIdx.x >> 5] = mn;
        s_am[threadIdx.x >> 5] = amx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
            if (s_mx[w] > mx || (s_mx[w] == mx && s_am[w] < amx)) {
                mx = s_mx[w];
                amx = s_am[w];
            }
            mn = s_mn[w] < mn ? s_mn[w] : mn;
        }
        s_mx[0] = mx;
        s_mn[0] = mn;
        s_am[0] = amx;
    }
    __syncthreads();
    mx = s_mx[0];
    mn = s_mn[0];
    amx = s_am[0];
    const double mean = block_pairwise(fit, n, leaf_off, c.n_leaf, leafsum) / (double)n;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const double d = fit[i] - mean;
        scratch[i] = d * d;
    }
    __syncthreads();
    const double var = block_pairwise(scratch, n, leaf_off, c.n_leaf, leafsum) / (double)n;
    if (threadIdx.x != 0) return;
    const double sd = sqrt(var);
    const int64_t g = st->g;
    double *row = trace + g * 5;
    row[0] = (double)g;
    row[1] = mx;
    row[2] = mean;
    row[4] = sd;
    if (c.algorithm == QPM_ALGO_GWO) {
        row[3] = g == 0 ? c.gwo_a0 : sched[g * QPM_SCHED_COLS + QPM_SCHED_A_NOW];
        if (g == 0 || mx > st->best_fit) {
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
        const uint8_t improved = mx > st->best_prev ? 1 : 0;
        if (st->win_len < cap) {
            st->win[st->win_len++] = improved;
        } else {
            for (int t = 1; t < cap; ++t) st->win[t - 1] = st->win[t];
            st->win[cap - 1] = improved;
        }
        st->best_prev = mx;
        int cnt = 0;
        for (int t = 0; t < st->win_len; ++t) cnt += st->win[t];
        const double conv = st->win_len ? (double)cnt / (double)st->win_len : 1.0;
        const double *sg = sched + g * QPM_SCHED_COLS;
        double f = sg[QPM_SCHED_F_ENV];
        if (c.adaptive) {
            const double tl = c.theta_low_frac * st->baseline_std;
            const double th = c.theta_high_frac * st->baseline_std;
            const double rt = c.range_trigger_frac * st->baseline_std;
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

// best row -> result buffer (when the stats/finalize step flagged it)
__global__ void k_copy_best(RunConsts c, const EngineState *__restrict__ st, const int32_t *__restrict__ slot_of,
                            const double *__restrict__ genome, const uint32_t *__restrict__ bits,
                            double *__restrict__ best_genome, uint32_t *__restrict__ best_bits) {
    if (!st->best_flag) return;
    const int64_t slot = slot_of[st->best_idx];
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < c.Dp; j += (int64_t)gridDim.x * blockDim.x) {
        best_genome[j] = genome[slot * c.Dp + j];
        if (j < c.W) best_bits[j] = bits[slot * c.W + j];
    }
}

__global__ void k_finalize_best(EngineState *st, const int32_t *top1) {
    st->best_idx = top1[0];
    st->best_flag = 1;
}

__global__ void k_reset_flag(EngineState *st) { st->best_flag = 0; }

// ---------------------------------------------------------------- engine
struct Engine {
    Problem *prob = nullptr;
    qpm_run_params P{};
    RunConsts c{};
    cudaStream_t stream = nullptr;
    double *genome = nullptr;
    uint32_t *bits = nullptr;
    int32_t *slot_of = nullptr, *spare_of = nullptr, *jrand = nullptr, *top1 = nullptr;
    double *fit = nullptr, *cand = nullptr, *scratch = nullptr, *leafsum = nullptr;
    int64_t *leaf_off = nullptr;
    uint64_t *keys = nullptr;
    int4 *picks = nullptr;
    uint8_t *accepted = nullptr;
    double *sched = nullptr, *trace = nullptr;
    EngineState *st = nullptr;
    double *best_genome = nullptr;
    uint32_t *best_bits = nullptr;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    int launches = 0;
    int64_t g_done = 0;
    bool initialized = false;
    bool owns_stream = false;
    int64_t device_bytes = 0;
    std::vector<void *> allocs;
};

template <typename T>
static int dalloc(Engine *e, T **p, size_t count) {
    size_t bytes = std::max<size_t>(count * sizeof(T), 16);
    QPM_CUDA_TRY(cudaMalloc((void **)p, bytes));
    e->allocs.push_back((void *)*p);
    e->device_bytes += (int64_t)bytes;
    return QPM_OK;
}

static void pairwise_leaves(int64_t off, int64_t n, std::vector<int64_t> &out) {
    if (n <= 128) {
        out.push_back(off);
        return;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    pairwise_leaves(off, n2, out);
    pairwise_leaves(off + n2, n - n2, out);
}

static dim3 row_grid(const Engine *e) {
    return dim3((unsigned)((e->c.Dp + kGenesPerBlock - 1) / kGenesPerBlock), (unsigned)e->c.NP);
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

// one generation's launch sequence
static int enqueue_generation(Engine *e, int *launches, StageMarks *pm = nullptr) {
    const RunConsts &c = e->c;
    cudaStream_t s = e->stream;
    const unsigned nb = (unsigned)((c.NP + 255) / 256);
    int n = 0;
    int rc;
    auto mark = [&](const char *next) {
        if (pm) pm->mark(s, next);
    };
    if (c.algorithm == QPM_ALGO_GWO) {
        mark("topk");
        rc = launch_reduce_best(e->fit, c.NP, 3, e->st->leaders, s);  // rank_leaders(pop, 3)
        if (rc) return rc;
        mark("gwo_continuous");
        k_keys<<<nb, 256, 0, s>>>(c, e->st, e->keys);
        k_gwo_continuous<<<row_grid(e), kRowThreads, 0, s>>>(c, e->st, e->sched, e->keys, e->slot_of, e->spare_of,
                                                             e->genome, e->bits);
        QPM_LAUNCH_CHECK();
        n += 3;
        mark("fitness");
        rc = launch_fitness(e->prob, e->bits, c.W, e->spare_of, c.NP, e->cand, e->P.fitness_mode, s, &n);
        if (rc) return rc;
        mark("replace");
        k_select<<<nb, 256, 0, s>>>(c, e->st, 1, 1, e->cand, e->fit, e->slot_of, e->spare_of, e->accepted);
        mark("stats");
        k_stats<<<1, kStatsThreads, 0, s>>>(c, e->st, e->sched, e->fit, e->scratch, e->leaf_off, e->leafsum,
                                            e->trace);
        k_copy_best<<<64, 256, 0, s>>>(c, e->st, e->slot_of, e->genome, e->bits, e->best_genome, e->best_bits);
        QPM_LAUNCH_CHECK();
        n += 3;
    } else {
        mark("de_draws");
        k_de_draws<<<nb, 256, 0, s>>>(c, e->st, e->keys, e->picks, e->jrand);
        mark("de_trial");
        k_de_trial<<<row_grid(e), kRowThreads, 0, s>>>(c, e->st, e->keys, e->picks, e->jrand, e->slot_of, e->spare_of,
                                                       e->genome, e->bits);
        QPM_LAUNCH_CHECK();
        n += 2;
        mark("fitness_de");
        rc = launch_fitness(e->prob, e->bits, c.W, e->spare_of, c.NP, e->cand, e->P.fitness_mode, s, &n);
        if (rc) return rc;
        mark("select_de");
        k_select<<<nb, 256, 0, s>>>(c, e->st, 0, 0, e->cand, e->fit, e->slot_of, e->spare_of, e->accepted);
        QPM_LAUNCH_CHECK();
        n += 1;
        if (c.algorithm == QPM_ALGO_HYBRID) {
            mark("topk");
            rc = launch_reduce_best(e->fit, c.NP, c.k, e->st->leaders, s);  // rank_leaders(pop, k)
            if (rc) return rc;
            mark("gwo_discrete");
            k_gwo_discrete<<<row_grid(e), kRowThreads, 0, s>>>(c, e->st, e->sched, e->keys, e->picks, e->slot_of,
                                                               e->spare_of, e->bits);
            QPM_LAUNCH_CHECK();
            n += 2;
            mark("fitness_gwo");
            rc = launch_fitness(e->prob, e->bits, c.W, e->spare_of, c.NP, e->cand, e->P.fitness_mode, s, &n);
            if (rc) return rc;
            mark("select_gwo");
            k_select<<<nb, 256, 0, s>>>(c, e->st, 1, 0, e->cand, e->fit, e->slot_of, e->spare_of, e->accepted);
            k_materialize<<<row_grid(e), kRowThreads, 0, s>>>(c, e->accepted, e->slot_of, e->bits, e->genome);
            QPM_LAUNCH_CHECK();
            n += 2;
        }
        mark("stats");
        k_stats<<<1, kStatsThreads, 0, s>>>(c, e->st, e->sched, e->fit, e->scratch, e->leaf_off, e->leafsum,
                                            e->trace);
        QPM_LAUNCH_CHECK();
        n += 1;
    }
    mark(nullptr);
    if (launches) *launches = n;
    return QPM_OK;
}

static void engine_free(Engine *e) {
    if (e->owns_stream && e->stream) {
        cudaStreamSynchronize(e->stream);
        cudaStreamDestroy(e->stream);
    }
    if (e->exec) cudaGraphExecDestroy(e->exec);
    if (e->graph) cudaGraphDestroy(e->graph);
    for (void *p : e->allocs) cudaFree(p);
    delete e;
}

}  // namespace qpm

struct qpm_engine {
    qpm::Engine *e;
};

using namespace qpm;

extern "C" {

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
    QPM_ARG_CHECK(P->row_lo == 0 && P->row_hi == P->NP, "sharded rows need the multi-GPU engine");
    QPM_ARG_CHECK(P->NP < (1LL << 31), "NP < 2^31");
    Engine *e = new Engine();
    e->prob = &prob->p;
    e->P = *P;
    e->stream = (cudaStream_t)stream;
    if (!e->stream) {
        // graphs cannot be captured on the legacy default stream: own a stream
        if (cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking) != cudaSuccess) {
            set_error("cudaStreamCreateWithFlags failed");
            delete e;
            return QPM_ERR_CUDA;
        }
        e->owns_stream = true;
    }
    RunConsts &c = e->c;
    c.algorithm = P->algorithm;
    c.NP = P->NP;
    c.D = prob->p.D;
    c.W = prob->p.W;
    c.Dp = c.W * 32;
    c.G = P->G;
    c.seed = (uint64_t)P->seed;
    c.f_max = P->f_max;
    c.f_min = P->f_min;
    c.cr_thr = le_threshold(P->cr);
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
    std::vector<int64_t> leaves;
    pairwise_leaves(0, c.NP, leaves);
    c.n_leaf = (int64_t)leaves.size();

    const int64_t NP = c.NP;
    int rc = QPM_OK;
#define QPM_ALLOC(ptr, count)                   \
    if ((rc = dalloc(e, &(ptr), (count))) != 0) { \
        engine_free(e);                         \
        return rc;                              \
    }
    QPM_ALLOC(e->genome, (size_t)2 * NP * c.Dp);
    QPM_ALLOC(e->bits, (size_t)2 * NP * c.W);
    QPM_ALLOC(e->slot_of, NP);
    QPM_ALLOC(e->spare_of, NP);
    QPM_ALLOC(e->jrand, NP);
    QPM_ALLOC(e->top1, 8);
    QPM_ALLOC(e->fit, NP);
    QPM_ALLOC(e->cand, NP);
    QPM_ALLOC(e->scratch, NP);
    QPM_ALLOC(e->leafsum, leaves.size());
    QPM_ALLOC(e->leaf_off, leaves.size());
    QPM_ALLOC(e->keys, NP);
    QPM_ALLOC(e->picks, NP);
    QPM_ALLOC(e->accepted, NP);
    QPM_ALLOC(e->sched, (size_t)(P->G + 1) * QPM_SCHED_COLS);
    QPM_ALLOC(e->trace, (size_t)(P->G + 1) * 5);
    QPM_ALLOC(e->st, 1);
    QPM_ALLOC(e->best_genome, c.Dp);
    QPM_ALLOC(e->best_bits, c.W);
#undef QPM_ALLOC
    if ((rc = problem_reserve(e->prob, NP)) != 0) {
        engine_free(e);
        return rc;
    }
    // host-side constants of the state: p_plus thresholds (optimizer.py:362-365)
    EngineState hs;
    memset(&hs, 0, sizeof(hs));
    for (int cnt = 0; cnt <= c.k && cnt <= kMaxLeaders; ++cnt) {
        double pp = (double)cnt / (double)c.k;
        if (P->discreteness_factor != 1.0) pp = 0.5 + P->discreteness_factor * (pp - 0.5);
        hs.thr_plus[cnt] = lt_threshold(pp);
    }
    hs.g = 0;
    hs.F = P->f_max;
    cudaError_t err = cudaMemcpyAsync(e->st, &hs, sizeof(hs), cudaMemcpyHostToDevice, e->stream);
    if (err == cudaSuccess)
        err = cudaMemcpyAsync(e->sched, sched, sizeof(double) * (P->G + 1) * QPM_SCHED_COLS, cudaMemcpyHostToDevice,
                              e->stream);
    if (err == cudaSuccess)
        err = cudaMemcpyAsync(e->leaf_off, leaves.data(), sizeof(int64_t) * leaves.size(), cudaMemcpyHostToDevice,
                              e->stream);
    if (err == cudaSuccess) err = cudaMemsetAsync(e->trace, 0, sizeof(double) * (P->G + 1) * 5, e->stream);
    if (err == cudaSuccess) err = cudaMemsetAsync(e->genome, 0, sizeof(double) * 2 * NP * c.Dp, e->stream);
    if (err == cudaSuccess) err = cudaMemsetAsync(e->bits, 0, sizeof(uint32_t) * 2 * NP * c.W, e->stream);
    if (err == cudaSuccess) err = cudaStreamSynchronize(e->stream);
    if (err != cudaSuccess) {
        set_error("engine upload: %s", cudaGetErrorString(err));
        engine_free(e);
        return QPM_ERR_CUDA;
    }
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

int qpm_engine_init(qpm_engine *h) {
    QPM_ARG_CHECK(h, "engine");
    Engine *e = h->e;
    const RunConsts &c = e->c;
    cudaStream_t s = e->stream;
    k_init_population<<<row_grid(e), kRowThreads, 0, s>>>(c, e->genome, e->bits, e->slot_of, e->spare_of);
    QPM_LAUNCH_CHECK();
    int rc = launch_fitness(e->prob, e->bits, c.W, e->slot_of, c.NP, e->fit, e->P.fitness_mode, s, nullptr);
    if (rc) return rc;
    k_stats<<<1, kStatsThreads, 0, s>>>(c, e->st, e->sched, e->fit, e->scratch, e->leaf_off, e->leafsum, e->trace);
    k_copy_best<<<64, 256, 0, s>>>(c, e->st, e->slot_of, e->genome, e->bits, e->best_genome, e->best_bits);
    QPM_LAUNCH_CHECK();
    e->initialized = true;
    e->g_done = 0;
    return QPM_OK;
}

int qpm_engine_step(qpm_engine *h, int64_t n, int use_graph) {
    QPM_ARG_CHECK(h, "engine");
    Engine *e = h->e;
    if (!e->initialized) {
        set_error("qpm_engine_step before qpm_engine_init");
        return QPM_ERR_STATE;
    }
    QPM_ARG_CHECK(n >= 0 && e->g_done + n <= e->c.G, "generation count exceeds G");
    if (n == 0) return QPM_OK;
    if (use_graph) {
        if (!e->exec) {
            cudaStreamCaptureMode mode = cudaStreamCaptureModeThreadLocal;
            QPM_CUDA_TRY(cudaStreamBeginCapture(e->stream, mode));
            int launches = 0;
            int rc = enqueue_generation(e, &launches);
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
            e->graph = g;
            QPM_CUDA_TRY(cudaGraphInstantiate(&e->exec, e->graph, 0));
            e->launches = launches;
        }
        for (int64_t t = 0; t < n; ++t) QPM_CUDA_TRY(cudaGraphLaunch(e->exec, e->stream));
    } else {
        for (int64_t t = 0; t < n; ++t) {
            int launches = 0;
            int rc = enqueue_generation(e, &launches);
            if (rc) return rc;
            e->launches = launches;
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
    int rc = launch_reduce_best(e->fit, c.NP, 1, e->top1, e->stream);
    if (rc) return rc;
    k_finalize_best<<<1, 1, 0, e->stream>>>(e->st, e->top1);
    k_copy_best<<<64, 256, 0, e->stream>>>(c, e->st, e->slot_of, e->genome, e->bits, e->best_genome, e->best_bits);
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

int qpm_engine_read_best(qpm_engine *h, double *genome, int8_t *proj, double *fitness) {
    QPM_ARG_CHECK(h, "engine");
    Engine *e = h->e;
    const RunConsts &c = e->c;
    std::vector<double> g(c.Dp);
    std::vector<uint32_t> b(c.W);
    EngineState hs;
    QPM_CUDA_TRY(cudaMemcpyAsync(g.data(), e->best_genome, sizeof(double) * c.Dp, cudaMemcpyDeviceToHost, e->stream));
    QPM_CUDA_TRY(cudaMemcpyAsync(b.data(), e->best_bits, sizeof(uint32_t) * c.W, cudaMemcpyDeviceToHost, e->stream));
    QPM_CUDA_TRY(cudaMemcpyAsync(&hs, e->st, sizeof(hs), cudaMemcpyDeviceToHost, e->stream));
    QPM_CUDA_TRY(cudaStreamSynchronize(e->stream));
    if (genome) memcpy(genome, g.data(), sizeof(double) * c.D);
    if (proj)
        for (int64_t j = 0; j < c.D; ++j) proj[j] = ((b[j >> 5] >> (j & 31)) & 1u) ? -1 : 1;
    if (fitness) {
        if (c.algorithm == QPM_ALGO_GWO) {
            *fitness = hs.best_fit;
        } else {
            QPM_CUDA_TRY(cudaMemcpy(fitness, e->fit + hs.best_idx, sizeof(double), cudaMemcpyDeviceToHost));
        }
    }
    return QPM_OK;
}

int qpm_engine_read_population(qpm_engine *h, double *genome, double *fitness) {
    QPM_ARG_CHECK(h, "engine");
    Engine *e = h->e;
    const RunConsts &c = e->c;
    std::vector<int32_t> slots(c.NP);
    QPM_CUDA_TRY(cudaMemcpyAsync(slots.data(), e->slot_of, sizeof(int32_t) * c.NP, cudaMemcpyDeviceToHost, e->stream));
    if (fitness)
        QPM_CUDA_TRY(cudaMemcpyAsync(fitness, e->fit, sizeof(double) * c.NP, cudaMemcpyDeviceToHost, e->stream));
    QPM_CUDA_TRY(cudaStreamSynchronize(e->stream));
    if (genome) {
        for (int64_t i = 0; i < c.NP; ++i)
            QPM_CUDA_TRY(cudaMemcpyAsync(genome + i * c.D, e->genome + (int64_t)slots[i] * c.Dp, sizeof(double) * c.D,
                                         cudaMemcpyDeviceToHost, e->stream));
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

int qpm_engine_launches_per_generation(const qpm_engine *h) {
    if (!h) return -1;
    if (h->e->launches) return h->e->launches;
    const int a = h->e->c.algorithm;
    return a == QPM_ALGO_HYBRID ? 12 : (a == QPM_ALGO_DE ? 6 : 8);
}

int qpm_engine_fitness_ptr(qpm_engine *h, double **fit_dev) {
    QPM_ARG_CHECK(h && fit_dev, "engine, out");
    *fit_dev = h->e->fit;
    return QPM_OK;
}

}  // extern "C"
