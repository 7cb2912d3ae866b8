/*
 * qpm_oracle.c -- CPU restatement of the qpmdesign HWSDA hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the B200
 * engine in paper_2511_01255_b200/.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.  The product
 * path never links, imports or calls it.
 *
 * Parity status: PINNED.  Every function below is checked against golden
 * vectors produced by running the reference package itself
 * (tests/golden/make_golden.py writes the fixtures tests/golden/NAME.npz), including the
 * reference's own golden_trace_seed7 regression.
 *
 * Arithmetic contract (build with -O2 -ffp-contract=off, no fast-math):
 *   - complex products are written out as (ac - bd, ad + bc) with no FMA, as
 *     numba lowers them (numba complex_mul_impl), and an int8 sign is promoted
 *     to complex(s, 0) before multiplying, exactly as numba types int8*complex;
 *   - |z| is libm hypot (numba lowers abs(complex) to hypot); glibc 2.39's
 *     hypot is the Borges non-FMA kernel, which the CUDA engine replicates;
 *   - float sums over populations use numpy's pairwise summation.
 *
 * Citations are /root/reference/pkg/src/qpmdesign/<file>:<line>.
 */
#include <math.h>
#include <stdint.h>
#include <time.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

#define QPO_GOLD 0x9E3779B97F4A7C15ULL
#define QPO_MIX1 0xBF58476D1CE4E5B9ULL
#define QPO_MIX2 0x94D049BB133111EBULL

/* ------------------------------------------------------------------------ */
/* Tiny pthread parallel-for with dynamic scheduling.  Every loop body below */
/* writes disjoint slots, so results do not depend on the thread count.     */
/* ------------------------------------------------------------------------ */

typedef void (*qpo_body_fn)(void *ctx, int64_t i);
typedef struct {
    qpo_body_fn fn;
    void *ctx;
    int64_t n;
    int64_t next;
    pthread_mutex_t mu;
} qpo_pfor;

static void *qpo_pfor_worker(void *arg) {
    qpo_pfor *pf = (qpo_pfor *)arg;
    for (;;) {
        pthread_mutex_lock(&pf->mu);
        int64_t i = pf->next++;
        pthread_mutex_unlock(&pf->mu);
        if (i >= pf->n) break;
        pf->fn(pf->ctx, i);
    }
    return NULL;
}

int qpo_max_threads(void) {
    long n = sysconf(_SC_NPROCESSORS_ONLN);
    return n > 0 ? (int)n : 1;
}

static void qpo_parallel_for(int64_t n, int threads, qpo_body_fn fn, void *ctx) {
    if (threads < 1) threads = qpo_max_threads();
    if (threads > n) threads = (int)n;
    if (threads <= 1) {
        for (int64_t i = 0; i < n; ++i) fn(ctx, i);
        return;
    }
    qpo_pfor pf = {fn, ctx, n, 0, PTHREAD_MUTEX_INITIALIZER};
    pthread_t tid[256];
    if (threads > 256) threads = 256;
    for (int t = 0; t < threads; ++t) pthread_create(&tid[t], NULL, qpo_pfor_worker, &pf);
    for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
}

/* ------------------------------------------------------------------------ */
/* RNG: rng.py:24-36 (_mix, fold_key), _kernels.py:87-98,144-151            */
/* ------------------------------------------------------------------------ */

static inline uint64_t qpo_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * QPO_MIX1;
    z = (z ^ (z >> 27)) * QPO_MIX2;
    return z ^ (z >> 31);
}

/* rng.fold_key(seed, *path): h = mix(seed); h = mix(h + GOLD + p) per p.
 * Python ints are masked to 64 bits, i.e. two's complement for negatives. */
uint64_t qpo_fold_key(int64_t seed, int npath, const int64_t *path) {
    uint64_t h = qpo_mix((uint64_t)seed);
    for (int k = 0; k < npath; ++k) h = qpo_mix(h + QPO_GOLD + (uint64_t)path[k]);
    return h;
}

static inline uint64_t qpo_key3(int64_t seed, int64_t a, int64_t b) {
    int64_t p[2] = {a, b};
    return qpo_fold_key(seed, 2, p);
}

/* value `pos` of a stream: uniform_fill_numpy (_kernels.py:87-98) */
static inline double qpo_u(uint64_t key, uint64_t pos) {
    uint64_t z = key + (pos + 1ULL) * QPO_GOLD;
    z = qpo_mix(z);
    return (double)(z >> 11) * 0x1p-53;
}

void qpo_uniform_fill(uint64_t key, uint64_t start, int64_t n, double *out) {
    for (int64_t i = 0; i < n; ++i) out[i] = qpo_u(key, start + (uint64_t)i);
}

/* CounterStream.randint (rng.py:61-63): min(int(u * bound), bound - 1) */
static inline int64_t qpo_randint(uint64_t key, uint64_t pos, int64_t bound) {
    double u = qpo_u(key, pos);
    int64_t r = (int64_t)(u * (double)bound);
    return r < bound - 1 ? r : bound - 1;
}

/* ------------------------------------------------------------------------ */
/* numpy pairwise summation (numpy/_core/src/umath/loops_utils.h.src),       */
/* used by np.sum / np.mean / np.std on float64 (optimizer.py:396-397,471). */
/* ------------------------------------------------------------------------ */

double qpo_pairwise_sum(const double *a, int64_t n, int64_t stride) {
    if (n < 8) {
        double res = 0.0;
        for (int64_t i = 0; i < n; ++i) res += a[i * stride];
        return res;
    } else if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; ++j) r[j] = a[j * stride];
        int64_t i;
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; ++j) r[j] += a[(i + j) * stride];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += a[i * stride];
        return res;
    } else {
        int64_t n2 = n / 2;
        n2 -= n2 % 8;
        return qpo_pairwise_sum(a, n2, stride) + qpo_pairwise_sum(a + n2 * stride, n - n2, stride);
    }
}

/* np.mean, np.std (ddof=0) exactly as numpy/_core/_methods.py computes them */
void qpo_mean_std(const double *x, int64_t n, double *mean, double *std, double *scratch) {
    double m = qpo_pairwise_sum(x, n, 1) / (double)n;
    for (int64_t i = 0; i < n; ++i) {
        double d = x[i] - m;
        scratch[i] = d * d;
    }
    double v = qpo_pairwise_sum(scratch, n, 1) / (double)n;
    *mean = m;
    *std = sqrt(v);
}

/* ------------------------------------------------------------------------ */
/* Fitness kernels: _kernels.py:107-142 (numba backend)                     */
/* ------------------------------------------------------------------------ */

/* _thg_sum_nb (_kernels.py:114-122).  Tables interleaved (re, im). */
void qpo_thg_sum(const int8_t *s, int64_t D, const double *e1, const double *b, double *acc_out) {
    double ar = 0.0, ai = 0.0, pr = 0.0, pi = 0.0;
    for (int64_t j = 0; j < D; ++j) {
        double sd = (double)s[j];
        /* s * prefix with s promoted to complex(s, 0) */
        double spr = sd * pr - 0.0 * pi;
        double spi = sd * pi + 0.0 * pr;
        /* (s * prefix) * b[j] */
        double br = b[2 * j], bi = b[2 * j + 1];
        double tr = spr * br - spi * bi;
        double ti = spr * bi + spi * br;
        ar += tr;
        ai += ti;
        /* prefix += s * e1[j] */
        double er = e1[2 * j], ei = e1[2 * j + 1];
        double ser = sd * er - 0.0 * ei;
        double sei = sd * ei + 0.0 * er;
        pr += ser;
        pi += sei;
    }
    acc_out[0] = ar;
    acc_out[1] = ai;
}

/* _shg_sum_nb (_kernels.py:107-112) */
void qpo_shg_sum(const int8_t *s, int64_t D, const double *e1, double *acc_out) {
    double ar = 0.0, ai = 0.0;
    for (int64_t j = 0; j < D; ++j) {
        double sd = (double)s[j];
        double er = e1[2 * j], ei = e1[2 * j + 1];
        ar += sd * er - 0.0 * ei;
        ai += sd * ei + 0.0 * er;
    }
    acc_out[0] = ar;
    acc_out[1] = ai;
}

/* |w * acc + h| with numba's complex mul and libm hypot (_kernels.py:134-142) */
static inline double qpo_cabs_affine(const double *w, const double *acc, const double *h) {
    double zr = w[0] * acc[0] - w[1] * acc[1];
    double zi = w[0] * acc[1] + w[1] * acc[0];
    if (h) {
        zr += h[0];
        zi += h[1];
    }
    return hypot(zr, zi);
}

/*
 * Problem = one PatternObjective (objectives.py:72-123).
 *   process 0 = shg, 1 = thg; multi 0/1; tables per wavelength, (re, im)
 *   interleaved: e1[n_wl][D][2], b[n_wl][D][2], w[n_wl][2] (w1 or w12),
 *   hconst[n_wl][2]; scale = normalization divisor or 1.0 for raw.
 */
typedef struct {
    int process;
    int multi;
    int n_wl;
    int64_t D;
    const double *e1;
    const double *b;
    const double *w;
    const double *hconst;
    double scale;
    double g0;
    double beta;
} qpo_problem;

/* PatternObjective.evaluate_block for one row (objectives.py:110-120) */
static double qpo_eval_row(const qpo_problem *P, const int8_t *s, double *gains) {
    for (int l = 0; l < P->n_wl; ++l) {
        double acc[2];
        const double *e1 = P->e1 + (size_t)l * P->D * 2;
        if (P->process == 1) {
            const double *b = P->b + (size_t)l * P->D * 2;
            qpo_thg_sum(s, P->D, e1, b, acc);
            gains[l] = qpo_cabs_affine(P->w + 2 * l, acc, P->hconst + 2 * l);
        } else {
            qpo_shg_sum(s, P->D, e1, acc);
            gains[l] = qpo_cabs_affine(P->w + 2 * l, acc, NULL);
        }
        if (P->scale != 1.0) gains[l] /= P->scale;
    }
    if (!P->multi) return gains[0];
    /* f = sum |g0 - g| (pairwise over the wavelength axis) + beta (max - min) */
    double gmax = gains[0], gmin = gains[0];
    for (int l = 1; l < P->n_wl; ++l) {
        if (gains[l] > gmax) gmax = gains[l];
        if (gains[l] < gmin) gmin = gains[l];
    }
    double *dev = gains + P->n_wl;
    for (int l = 0; l < P->n_wl; ++l) dev[l] = fabs(P->g0 - gains[l]);
    double f = qpo_pairwise_sum(dev, P->n_wl, 1);
    f += P->beta * (gmax - gmin);
    return -f;
}

typedef struct {
    const qpo_problem *P;
    const int8_t *signs;
    double *out;
} qpo_eval_ctx;

static void qpo_eval_body(void *vctx, int64_t r) {
    qpo_eval_ctx *c = (qpo_eval_ctx *)vctx;
    double gains_stack[2 * 256];
    gains_stack[0] = 0.0; /* (n_wl >= 1: silences gcc's maybe-uninitialized) */
    double *gains = c->P->n_wl <= 256 ? gains_stack : (double *)malloc(sizeof(double) * 2 * c->P->n_wl);
    c->out[r] = qpo_eval_row(c->P, c->signs + (size_t)r * c->P->D, gains);
    if (gains != gains_stack) free(gains);
}

void qpo_evaluate_block(const qpo_problem *P, const int8_t *signs, int64_t rows, double *out,
                        int threads) {
    qpo_eval_ctx c = {P, signs, out};
    qpo_parallel_for(rows, threads, qpo_eval_body, &c);
}

/* the raw complex sums, for parity of the block kernels (_kernels.py:124-132) */
void qpo_sum_block(const qpo_problem *P, int wl, const int8_t *signs, int64_t rows, double *out) {
    const double *e1 = P->e1 + (size_t)wl * P->D * 2;
    const double *b = P->b + (size_t)wl * P->D * 2;
    for (int64_t r = 0; r < rows; ++r) {
        if (P->process == 1)
            qpo_thg_sum(signs + (size_t)r * P->D, P->D, e1, b, out + 2 * r);
        else
            qpo_shg_sum(signs + (size_t)r * P->D, P->D, e1, out + 2 * r);
    }
}

/* ------------------------------------------------------------------------ */
/* Leader ranking: parexec.reduce_best (parexec.py:123-154)                  */
/* top-k by (-f, index): ties go to the lower index.                         */
/* ------------------------------------------------------------------------ */

void qpo_reduce_best(const double *f, int64_t n, int k, int64_t *idx_out) {
    for (int t = 0; t < k; ++t) idx_out[t] = -1;
    for (int64_t i = 0; i < n; ++i) {
        /* insert i if it beats the current t-th entry */
        int pos = k;
        while (pos > 0) {
            int64_t j = idx_out[pos - 1];
            if (j >= 0 && !(f[i] > f[j])) break; /* f[i] <= f[j] and i > j: stays behind */
            --pos;
        }
        if (pos < k) {
            for (int t = k - 1; t > pos; --t) idx_out[t] = idx_out[t - 1];
            idx_out[pos] = i;
        }
    }
}

/* ------------------------------------------------------------------------ */
/* Operators (optimizer.py)                                                 */
/* ------------------------------------------------------------------------ */

/* de_mutate (optimizer.py:229-247): rejection-sampled r1, r2, r3 distinct
 * and != i, one draw per candidate.  Returns the number of draws m. */
int64_t qpo_de_pick(uint64_t key, int64_t NP, int64_t i, int64_t *r) {
    int64_t m = 0;
    int n = 0;
    while (n < 3) {
        int64_t c = qpo_randint(key, (uint64_t)m, NP);
        ++m;
        int dup = (c == i);
        for (int t = 0; t < n; ++t) dup |= (c == r[t]);
        if (!dup) r[n++] = c;
    }
    return m;
}

/* de_mutate + de_crossover (optimizer.py:247, 250-262) for one individual.
 * Stream positions: 0..m-1 indices, m j_rand, m+1..m+D mask. */
int64_t qpo_de_trial(uint64_t key, int64_t NP, int64_t D, int64_t i, const double *const *genome,
                     double f, double cr, double *trial, int64_t *picks, int64_t *jrand_out) {
    int64_t r[3];
    int64_t m = qpo_de_pick(key, NP, i, r);
    int64_t jrand = qpo_randint(key, (uint64_t)m, D);
    const double *x = genome[i], *x1 = genome[r[0]], *x2 = genome[r[1]], *x3 = genome[r[2]];
    for (int64_t j = 0; j < D; ++j) {
        double u = qpo_u(key, (uint64_t)(m + 1 + j));
        double v = x1[j] + f * (x2[j] - x3[j]);
        trial[j] = (u <= cr || j == jrand) ? v : x[j];
    }
    if (picks) {
        picks[0] = r[0];
        picks[1] = r[1];
        picks[2] = r[2];
    }
    if (jrand_out) *jrand_out = jrand;
    return m;
}

/* gwo_discrete_update (optimizer.py:335-376).  leaders: k int8 projection
 * rows in rank order.  base = first stream position of the 6 x D block. */
void qpo_gwo_discrete(uint64_t key, uint64_t base, int64_t D, int k, const int8_t *const *leaders,
                      double p_dist, double p_sl, double p_flip, double discreteness, int early,
                      double *out) {
    for (int64_t j = 0; j < D; ++j) {
        int cp = 0;
        for (int t = 0; t < k; ++t) cp += leaders[t][j] > 0;
        double p_plus = (double)cp / (double)k;
        if (discreteness != 1.0) p_plus = 0.5 + discreteness * (p_plus - 0.5);
        double us = qpo_u(key, base + (uint64_t)j);
        double upk = qpo_u(key, base + (uint64_t)(D + j));
        double ud = qpo_u(key, base + (uint64_t)(2 * D + j));
        double ust = qpo_u(key, base + (uint64_t)(3 * D + j));
        double upl = qpo_u(key, base + (uint64_t)(4 * D + j));
        double ufl = qpo_u(key, base + (uint64_t)(5 * D + j));
        int64_t pick = (int64_t)(upk * (double)k);
        if (pick > k - 1) pick = k - 1;
        int leader_state = leaders[pick][j];
        int random_state = ust < 0.5 ? 1 : -1;
        int basev;
        if (early) {
            int sampled = upl < p_plus ? 1 : -1;
            basev = ud < p_dist ? random_state : sampled;
        } else {
            int maj = 2 * cp > k ? 1 : (2 * cp < k ? -1 : random_state);
            basev = ufl < p_flip ? -maj : maj;
        }
        out[j] = (double)(us < p_sl ? leader_state : basev);
    }
}

/* gwo_reference_update (optimizer.py:302-332).  L leaders in rank order;
 * stream positions [2mD, 2mD+D) for r1 and [2mD+D, 2mD+2D) for r2. */
void qpo_gwo_continuous(uint64_t key, int64_t D, int L, const double *x, const double *const *leaders,
                        double a, int divide, double *out) {
    double moved[16];
    double two_a = 2.0 * a;
    for (int64_t j = 0; j < D; ++j) {
        for (int m = 0; m < L; ++m) {
            double r1 = qpo_u(key, (uint64_t)(2 * m * D + j));
            double r2 = qpo_u(key, (uint64_t)(2 * m * D + D + j));
            double av = two_a * r1 - a;
            double cv = 2.0 * r2;
            double xm = leaders[m][j];
            double dist = fabs(cv * xm - x[j]);
            moved[m] = xm - av * dist;
        }
        double denom = 0.0;
        for (int m = 0; m < L; ++m) denom = (m == 0) ? fabs(moved[0]) : denom + fabs(moved[m]);
        double acc = 0.0;
        for (int m = 0; m < L; ++m) {
            double w = denom > 0.0 ? fabs(moved[m]) / denom : 1.0 / (double)L;
            double p = w * moved[m];
            acc = (m == 0) ? p : acc + p;
        }
        if (divide) acc /= (double)L;
        out[j] = acc;
    }
}

/* ------------------------------------------------------------------------ */
/* Run drivers (optimizer.py:400-592)                                        */
/* ------------------------------------------------------------------------ */

typedef struct {
    int algorithm; /* 0 hybrid, 1 de, 2 gwo */
    int64_t NP, D, G;
    int64_t seed;
    /* DEParams (optimizer.py:84-101) */
    double f_max, f_min, cr, x_min, x_max;
    /* GWOParams (optimizer.py:104-133) */
    double gwo_a, gwo_a_final;
    int leader_count;
    double discreteness_factor;
    int divide_by_leader_count;
    /* Schedules (optimizer.py:136-173) */
    double p_dist0, p_sl0, p_flip0, phase_split, decay_strength;
    double theta_low_frac, theta_high_frac, range_trigger_frac;
    double explore_boost, exploit_factor, conv_threshold;
    int conv_window;
    int adaptive_branches;
    /* run_gwo bounds (optimizer.py:546) */
    double gwo_lo, gwo_hi;
    int threads;
    /* stop after this many generations (bounded CPU-baseline samples); <0 = G */
    int64_t stop_after;
} qpo_params;

typedef struct {
    double *genome; /* NP x D */
    int8_t *proj;   /* NP x D */
    double *fit;    /* NP */
} qpo_pop;

static void qpo_project_row(const double *g, int64_t D, int8_t *p) {
    for (int64_t j = 0; j < D; ++j) p[j] = g[j] >= 0.0 ? 1 : -1;
}

/* init_population (optimizer.py:207-226) */
void qpo_init_population(int64_t NP, int64_t D, double lo, double hi, int64_t seed, double *genome) {
    double span = hi - lo;
    for (int64_t i = 0; i < NP; ++i) {
        uint64_t key = qpo_key3(seed, 0, i);
        for (int64_t j = 0; j < D; ++j) genome[i * D + j] = lo + qpo_u(key, (uint64_t)j) * span;
    }
}

/* adaptive_f_update (optimizer.py:277-299) */
double qpo_adaptive_f(const qpo_params *p, int64_t g, int64_t total, double pop_std, double fit_range,
                      double conv, double decay, double baseline) {
    double progress = total > 0 ? (double)g / (double)total : 0.0;
    double f = p->f_min + (p->f_max - p->f_min) * cos(0.5 * M_PI * progress);
    if (p->adaptive_branches) {
        double tl = p->theta_low_frac * baseline;
        double th = p->theta_high_frac * baseline;
        double rt = p->range_trigger_frac * baseline;
        if (pop_std < tl || conv < p->conv_threshold) f *= p->explore_boost;
        if (pop_std > th || fit_range < rt) f *= p->exploit_factor;
    }
    f *= decay;
    double lo = f > p->f_min ? f : p->f_min; /* max(f, f_min) */
    return lo < p->f_max ? lo : p->f_max;    /* min(., f_max) */
}

static void qpo_trace_row(double *row, int64_t g, const double *fit, int64_t n, double fval,
                          double *scratch, double *mx_out, double *mn_out, double *std_out) {
    double mx = fit[0], mn = fit[0];
    for (int64_t i = 1; i < n; ++i) {
        if (fit[i] > mx) mx = fit[i];
        if (fit[i] < mn) mn = fit[i];
    }
    double mean, std;
    qpo_mean_std(fit, n, &mean, &std, scratch);
    row[0] = (double)g;
    row[1] = mx;
    row[2] = mean;
    row[3] = fval;
    row[4] = std;
    if (mx_out) *mx_out = mx;
    if (mn_out) *mn_out = mn;
    if (std_out) *std_out = std;
}


/* per-generation work shared by the parallel loop bodies below */
typedef struct {
    const qpo_params *p;
    int64_t g, NP, D;
    double F, a_now, p_dist, p_sl, p_flip;
    int early, k;
    const double **rows;
    double *genome;
    const int8_t **lp;
    const double **lrows;
    double *tgen;
    int8_t *tproj;
    int64_t *mcount;
    uint64_t *keys;
    const int64_t *movers;
} qpo_gen_ctx;

static void qpo_de_body(void *vctx, int64_t i) {
    qpo_gen_ctx *c = (qpo_gen_ctx *)vctx;
    const int64_t D = c->D;
    c->keys[i] = qpo_key3(c->p->seed, c->g, i);
    c->mcount[i] = qpo_de_trial(c->keys[i], c->NP, D, i, c->rows, c->F, c->p->cr, c->tgen + i * D, NULL, NULL);
    qpo_project_row(c->tgen + i * D, D, c->tproj + i * D);
}

static void qpo_gwo_body(void *vctx, int64_t t) {
    qpo_gen_ctx *c = (qpo_gen_ctx *)vctx;
    const int64_t D = c->D, i = c->movers[t];
    uint64_t base = (uint64_t)(c->mcount[i] + 1 + D);
    qpo_gwo_discrete(c->keys[i], base, D, c->k, c->lp, c->p_dist, c->p_sl, c->p_flip,
                     c->p->discreteness_factor, c->early, c->tgen + t * D);
    qpo_project_row(c->tgen + t * D, D, c->tproj + t * D);
}

static void qpo_gwoc_body(void *vctx, int64_t t) {
    qpo_gen_ctx *c = (qpo_gen_ctx *)vctx;
    const int64_t D = c->D, i = c->movers[t];
    uint64_t key = qpo_key3(c->p->seed, c->g, i);
    qpo_gwo_continuous(key, D, 3, c->genome + i * D, c->lrows, c->a_now, c->p->divide_by_leader_count,
                       c->tgen + t * D);
    qpo_project_row(c->tgen + t * D, D, c->tproj + t * D);
}

/*
 * Full run.  trace: (G+1) x 5 rows (generation, best, mean, F|a, pop_std).
 * best_genome (D), best_proj (D), best_fit (1).  Returns number of trace rows.
 */
static double qpo_now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

static int64_t qpo_run_impl(const qpo_problem *P, const qpo_params *p, double *trace, double *best_genome,
                            int8_t *best_proj, double *best_fit, double *t_end);

int64_t qpo_run(const qpo_problem *P, const qpo_params *p, double *trace, double *best_genome,
                int8_t *best_proj, double *best_fit) {
    return qpo_run_impl(P, p, trace, best_genome, best_proj, best_fit, NULL);
}

/* The same run, with t_end[g] = monotonic seconds when generation g's trace
 * row is complete (g = 0: the initial population): benchmark windows time
 * generations w+1..w+k as t_end[w+k] - t_end[w] inside one run. */
int64_t qpo_run_timed(const qpo_problem *P, const qpo_params *p, double *trace, double *best_genome,
                      int8_t *best_proj, double *best_fit, double *t_end) {
    return qpo_run_impl(P, p, trace, best_genome, best_proj, best_fit, t_end);
}

static int64_t qpo_run_impl(const qpo_problem *P, const qpo_params *p, double *trace, double *best_genome,
                            int8_t *best_proj, double *best_fit, double *t_end) {
    const int64_t NP = p->NP, D = p->D, G = p->G;
    const int64_t stop = p->stop_after >= 0 && p->stop_after < G ? p->stop_after : G;
    const int threads = p->threads;
    double *genome = (double *)malloc(sizeof(double) * NP * D);
    int8_t *proj = (int8_t *)malloc((size_t)NP * D);
    double *fit = (double *)malloc(sizeof(double) * NP);
    double *tgen = (double *)malloc(sizeof(double) * NP * D);
    int8_t *tproj = (int8_t *)malloc((size_t)NP * D);
    double *tfit = (double *)malloc(sizeof(double) * NP);
    int64_t *mcount = (int64_t *)malloc(sizeof(int64_t) * NP);
    uint64_t *keys = (uint64_t *)malloc(sizeof(uint64_t) * NP);
    double *scratch = (double *)malloc(sizeof(double) * NP);
    int64_t *movers = (int64_t *)malloc(sizeof(int64_t) * NP);
    const double **rows = (const double **)malloc(sizeof(double *) * NP);
    char *win = (char *)calloc((size_t)(p->conv_window > 1 ? p->conv_window : 1), 1);
    int64_t rows_out = 0;
    qpo_gen_ctx c;
    memset(&c, 0, sizeof(c));
    c.p = p;
    c.NP = NP;
    c.D = D;
    c.rows = rows;
    c.genome = genome;
    c.tgen = tgen;
    c.tproj = tproj;
    c.mcount = mcount;
    c.keys = keys;
    c.movers = movers;

    if (p->algorithm == 2)
        qpo_init_population(NP, D, p->gwo_lo, p->gwo_hi, p->seed, genome);
    else
        qpo_init_population(NP, D, p->x_min, p->x_max, p->seed, genome);
    for (int64_t i = 0; i < NP; ++i) qpo_project_row(genome + i * D, D, proj + i * D);
    qpo_evaluate_block(P, proj, NP, fit, threads);
    for (int64_t i = 0; i < NP; ++i) rows[i] = genome + i * D;

    if (p->algorithm == 2) {
        /* ---------------- run_gwo (optimizer.py:543-592) ---------------- */
        int64_t bi;
        qpo_reduce_best(fit, NP, 1, &bi);
        memcpy(best_genome, genome + bi * D, sizeof(double) * D);
        memcpy(best_proj, proj + bi * D, (size_t)D);
        *best_fit = fit[bi];
        qpo_trace_row(trace, 0, fit, NP, p->gwo_a, scratch, NULL, NULL, NULL);
        rows_out = 1;
        if (t_end) t_end[0] = qpo_now_s();
        for (int64_t g = 1; g <= stop; ++g) {
            double progress = G ? (double)g / (double)G : 0.0;
            c.g = g;
            c.a_now = p->gwo_a_final + (p->gwo_a - p->gwo_a_final) * (1.0 - progress);
            int64_t lead[3];
            qpo_reduce_best(fit, NP, 3, lead);
            const double *lrows[3] = {genome + lead[0] * D, genome + lead[1] * D, genome + lead[2] * D};
            c.lrows = lrows;
            int64_t nm = 0;
            for (int64_t i = 0; i < NP; ++i)
                if (i != lead[0] && i != lead[1] && i != lead[2]) movers[nm++] = i;
            qpo_parallel_for(nm, threads, qpo_gwoc_body, &c);
            qpo_evaluate_block(P, tproj, nm, tfit, threads);
            for (int64_t t = 0; t < nm; ++t) {
                int64_t i = movers[t];
                memcpy(genome + i * D, tgen + t * D, sizeof(double) * D);
                memcpy(proj + i * D, tproj + t * D, (size_t)D);
                fit[i] = tfit[t];
            }
            qpo_reduce_best(fit, NP, 1, &bi);
            if (fit[bi] > *best_fit) {
                memcpy(best_genome, genome + bi * D, sizeof(double) * D);
                memcpy(best_proj, proj + bi * D, (size_t)D);
                *best_fit = fit[bi];
            }
            qpo_trace_row(trace + 5 * g, g, fit, NP, c.a_now, scratch, NULL, NULL, NULL);
            rows_out = g + 1;
            if (t_end) t_end[g] = qpo_now_s();
        }
        goto done;
    }

    /* ---------------- run_hybrid / run_de (optimizer.py:400-540) ---------------- */
    double mx, mn, std;
    qpo_trace_row(trace, 0, fit, NP, p->f_max, scratch, &mx, &mn, &std);
    double baseline_std = std;
    double F = p->f_max;
    double best_prev = mx;
    int win_len = 0, win_head = 0;
    const int win_cap = p->conv_window > 1 ? p->conv_window : 1;
    rows_out = 1;
    if (t_end) t_end[0] = qpo_now_s();
    const int k = p->leader_count;
    c.k = k;

    for (int64_t g = 1; g <= stop; ++g) {
        /* DE phase (optimizer.py:429-439) */
        c.g = g;
        c.F = F;
        qpo_parallel_for(NP, threads, qpo_de_body, &c);
        qpo_evaluate_block(P, tproj, NP, tfit, threads);
        for (int64_t i = 0; i < NP; ++i) {
            if (tfit[i] > fit[i]) {
                memcpy(genome + i * D, tgen + i * D, sizeof(double) * D);
                memcpy(proj + i * D, tproj + i * D, (size_t)D);
                fit[i] = tfit[i];
            }
        }
        if (p->algorithm == 0) {
            /* leaders and wolf phase (optimizer.py:441-467) */
            int64_t lead[4];
            qpo_reduce_best(fit, NP, k, lead);
            const int8_t *lp[4];
            for (int t = 0; t < k; ++t) lp[t] = proj + lead[t] * D;
            c.lp = lp;
            double prog = G ? (double)g / (double)G : 0.0;
            c.p_dist = G ? p->p_dist0 * (1.0 - prog) : 0.0;
            c.p_sl = G ? p->p_sl0 * (1.0 - prog) : 0.0;
            c.p_flip = G ? p->p_flip0 * (1.0 - prog) : 0.0;
            c.early = prog < p->phase_split;
            int64_t nm = 0;
            for (int64_t i = 0; i < NP; ++i) {
                int is_l = 0;
                for (int t = 0; t < k; ++t) is_l |= (lead[t] == i);
                if (!is_l) movers[nm++] = i;
            }
            qpo_parallel_for(nm, threads, qpo_gwo_body, &c);
            qpo_evaluate_block(P, tproj, nm, tfit, threads);
            for (int64_t t = 0; t < nm; ++t) {
                int64_t i = movers[t];
                if (tfit[t] > fit[i]) {
                    memcpy(genome + i * D, tgen + t * D, sizeof(double) * D);
                    memcpy(proj + i * D, tproj + t * D, (size_t)D);
                    fit[i] = tfit[t];
                }
            }
        }
        /* parameter update and trace (optimizer.py:469-485) */
        double row[5];
        qpo_trace_row(row, g, fit, NP, 0.0, scratch, &mx, &mn, &std);
        double best_now = mx;
        char improved = best_now > best_prev;
        if (win_len < win_cap) {
            win[(win_head + win_len) % win_cap] = improved;
            ++win_len;
        } else {
            win[win_head] = improved;
            win_head = (win_head + 1) % win_cap;
        }
        best_prev = best_now;
        int cnt = 0;
        for (int t = 0; t < win_len; ++t) cnt += win[t];
        double conv = win_len ? (double)cnt / (double)win_len : 1.0;
        double prog = G ? (double)g / (double)G : 0.0;
        double decay = 1.0 - p->decay_strength * prog * prog;
        F = qpo_adaptive_f(p, g, G, std, mx - mn, conv, decay, baseline_std);
        row[3] = F;
        memcpy(trace + 5 * g, row, sizeof(row));
        rows_out = g + 1;
        if (t_end) t_end[g] = qpo_now_s();
    }
    {
        int64_t bi;
        qpo_reduce_best(fit, NP, 1, &bi);
        memcpy(best_genome, genome + bi * D, sizeof(double) * D);
        memcpy(best_proj, proj + bi * D, (size_t)D);
        *best_fit = fit[bi];
    }
done:
    free(genome);
    free(proj);
    free(fit);
    free(tgen);
    free(tproj);
    free(tfit);
    free(mcount);
    free(keys);
    free(scratch);
    free(movers);
    free(rows);
    free(win);
    return rows_out;
}
