/*
 * qpm_b200.h -- C ABI of the B200-native HWSDA population engine.
 *
 * One shared library (paper_2511_01255_b200/libqpm_b200.so, sm_100a) exports
 * everything below.  Plain pointers and sizes only; no torch or C++ types
 * cross the boundary.  Every entry point returns QPM_OK (0) or a negative
 * status; qpm_last_error() returns a message for the calling thread.  Device
 * pointers are CUDA global memory on the current device; `stream` is a
 * cudaStream_t (NULL = legacy default stream).  Nothing allocates on the
 * per-generation path: problems and engines allocate once at creation.
 *
 * Which reference interface each group replaces (paths relative to
 * /root/reference/pkg/src/qpmdesign/):
 *
 *   qpm_uniform_fill, qpm_fold_key  -> _kernels.uniform_fill (_kernels.py:144-151,
 *                                      87-98), rng.fold_key (rng.py:31-36)
 *   qpm_problem_*                   -> ShgEvaluator/ThgEvaluator tables
 *                                      (physics.py:277-356) + PatternObjective
 *                                      (objectives.py:72-123)
 *   qpm_fitness_bits, qpm_evaluate_block_host
 *                                   -> PatternObjective.evaluate_block
 *                                      (objectives.py:110-120) via
 *                                      _kernels.thg_abs_block / shg_abs_block
 *                                      (_kernels.py:134-142, 168-169)
 *   qpm_sum_block_host              -> _kernels.thg_block / shg_block
 *                                      (_kernels.py:124-132)
 *   qpm_pack_signs                  -> Individual.from_genome projection
 *                                      (optimizer.py:52-56), bit-packed
 *   qpm_reduce_best                 -> parexec.reduce_best (parexec.py:123-154)
 *   qpm_sweep_spectrum              -> physics.sweep_spectrum (physics.py:378-395),
 *   qpm_wavelength_scalars          -> the per-wavelength Sellmeier / moment precompute (physics.py:97-339),
 *                                      batched over patterns
 *   qpm_brute_force                 -> bench.brute_force_oracle (bench.py:179-209)
 *                                      with bench.lexicographic_signs (:169-176)
 *   qpm_engine_*                    -> optimizer.run_hybrid / run_de / run_gwo
 *                                      (optimizer.py:400-616) including
 *                                      de_mutate/de_crossover/de_select,
 *                                      rank_leaders, gwo_discrete_update,
 *                                      gwo_reference_update, adaptive_f_update
 */
#ifndef QPM_B200_H
#define QPM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QPM_OK 0
#define QPM_ERR_ARG -1
#define QPM_ERR_CUDA -2
#define QPM_ERR_STATE -3
#define QPM_ERR_NCCL -4

#define QPM_PROCESS_SHG 0
#define QPM_PROCESS_THG 1

/* fitness arithmetic: exact replays numba's sequential per-domain order
 * bit-for-bit (parity tool); fast is the segmented FP64 quad-table scan. */
#define QPM_MODE_FAST 0
#define QPM_MODE_EXACT 1

#define QPM_ALGO_HYBRID 0
#define QPM_ALGO_DE 1
#define QPM_ALGO_GWO 2

/* columns of the per-generation schedule table (host-computed with Python
 * float arithmetic so device decisions equal the reference's) */
#define QPM_SCHED_F_ENV 0   /* f_min + (f_max - f_min) cos(pi g / 2G)      optimizer.py:290 */
#define QPM_SCHED_DECAY 1   /* 1 - decay_strength (g/G)^2                   optimizer.py:166-168 */
#define QPM_SCHED_P_DIST 2  /* p_dist0 (1 - g/G)                            optimizer.py:157-158 */
#define QPM_SCHED_P_SL 3    /* p_sl0 (1 - g/G)                              optimizer.py:160-161 */
#define QPM_SCHED_P_FLIP 4  /* p_flip0 (1 - g/G)                            optimizer.py:163-164 */
#define QPM_SCHED_EARLY 5   /* 1.0 if g/G < phase_split                     optimizer.py:170-171 */
#define QPM_SCHED_A_NOW 6   /* a_final + (a - a_final)(1 - g/G)   (run_gwo) optimizer.py:563-564 */
#define QPM_SCHED_COLS 8

const char *qpm_last_error(void);
int qpm_version(void);
/* number of SMs and compute capability of the current device */
int qpm_device_info(int *sm_count, int *cc_major, int *cc_minor);

/* Engines return their device buffers to a process-wide cache on destroy so
 * the next run of the same shape skips cudaMalloc/cudaFree; this frees the
 * idle cached blocks (no engine may be mid-destruction on another thread).
 * No reference counterpart (the reference allocates numpy arrays per run). */
int qpm_release_cached_memory(void);

/* ------------------------------------------------------------------ RNG */
uint64_t qpm_fold_key(int64_t seed, int npath, const int64_t *path);
int qpm_uniform_fill(uint64_t key, uint64_t start, int64_t n, double *out_dev, void *stream);

/* -------------------------------------------------------------- problem */
typedef struct qpm_problem qpm_problem;

/* Tables are host arrays, complex values interleaved (re, im):
 *   e1[n_wl][D][2], b[n_wl][D][2] (THG only, else NULL),
 *   w[n_wl][2] (w12 for THG, w1 for SHG), hconst[n_wl][2] (THG, else NULL).
 * scale: divisor applied to |d_eff| (L or L^2/2), 1.0 for raw.
 * multi: 1 for the multi-wavelength objective -(sum|g0-g| + beta(max-min)).
 * seg_chunks: fast-scan segment length in 128-domain chunks, 0 = the
 * default for D and n_wl.  It fixes the fitness stitch tree (S segments in
 * min(8, S) super-blocks), so fast-mode values depend on it (at the 1e-15
 * level) and on nothing else -- not the batch, not the GPU count.  A
 * multi-GPU run of W ranks needs min(8, S) >= W. */
int qpm_problem_create(qpm_problem **out, int process, int multi, int n_wl, int64_t D, const double *e1,
                       const double *b, const double *w, const double *hconst, double scale, double g0,
                       double beta, int seg_chunks);
int qpm_problem_destroy(qpm_problem *p);
/* u32 words per bit-packed row (domains padded to a multiple of 128) */
int64_t qpm_problem_row_words(const qpm_problem *p);
/* the fast scan's segment length (chunks), segment count S and stitch
 * super-block count min(8, S) */
int qpm_problem_layout(const qpm_problem *p, int *seg_chunks, int *segments, int *super_blocks);

/* pack int8 +/-1 rows [rows][D] into bit rows (bit 1 = -1) of stride row_words */
int qpm_pack_signs(const int8_t *signs_dev, int64_t rows, int64_t D, uint32_t *bits_dev, int64_t row_words,
                   void *stream);

/* fitness of bit-packed rows.  row_index (device, may be NULL): row r reads
 * bits_dev + row_index[r] * row_words.  out_dev: f64 [rows]. */
int qpm_fitness_bits(qpm_problem *p, const uint32_t *bits_dev, int64_t row_words, const int32_t *row_index_dev,
                     int64_t rows, double *out_dev, int mode, void *stream);

/* host-buffer plugin path: int8 [rows][D] host -> f64 [rows] host (sync) */
int qpm_evaluate_block_host(qpm_problem *p, const int8_t *signs, int64_t rows, double *out, int mode);
/* complex kernel sums (thg_block / shg_block) of wavelength wl, host in/out:
 * out[rows][2]; always the exact numba order */
int qpm_sum_block_host(qpm_problem *p, int wl, const int8_t *signs, int64_t rows, double *out);

/* -------------------------------------------------------------- leaders */
/* top-k indices by (-value, index) of values_dev[n]; idx_out_dev int32 [k]; k <= 64 */
int qpm_reduce_best(const double *values_dev, int64_t n, int k, int32_t *idx_out_dev, void *stream);

/* -------------------------------------------------------------- spectra */
/* |d_eff| of P patterns at M pump wavelengths (physics.sweep_spectrum): the
 * phase tables exp(-i dk z_j), z_j = j t, are generated on the device
 * (sincos of the same double product j*t*dk numpy forms) instead of being
 * uploaded, one CTA per (wavelength, pattern).
 *   process QPM_PROCESS_SHG: d = w[m] * sum_j s_j e1_j
 *   process QPM_PROCESS_THG: d = w[m] * sum_j s_j P_j b_j + hphi[m] * sum_j e1_j b_j
 *     (w = w12, hphi = t^2 phi(i dk1 t, i dk2 t): hconst = hphi * sum e1 b)
 * signs: host int8 [P][D]; dk, w, hphi: host [M][2]; out: host f64 [P][M]
 * |d|.  Accuracy: the device sincos differs from libm by <= 1 ulp per phase;
 * |d| agrees with the reference to ~1e-12 relative.  Synchronous. */
int qpm_sweep_spectrum(int process, double thickness, int64_t D, const int8_t *signs, int64_t P, const double *dk,
                       const double *w, const double *hphi, int64_t M, double *out);

/* Per-wavelength scalars of a Sellmeier dispersion model on the device
 * (replaces the host loop of physics.sweep_spectrum / ThgEvaluator over pump
 * wavelengths: physics.py:97-110 refractive index, 184-197 mismatches,
 * 224-270 moment integrals, 285-293 / 325-339 w and the cascade factor).
 * sellmeier_terms[6] = {a1 + b1 ft, a6, a2 + b2 ft, (a3 + b3 ft)**2, a4 + b4 ft,
 * a5**2} with ft = (T - 24.5)(T + 570.82), computed by the caller (Python's
 * x**2 is libm pow).  wavelengths_nm: host [M] (the caller checks the model's
 * validity range).  Out (host [M][2]): dk = (dk1, dk2) bit-identical to the
 * host formula; w (w1 for SHG, w12 for THG) and hphi = t^2 phi(i dk1 t, i dk2 t)
 * within ~1e-16 relative (device exp/sincos).  QPM_ERR_ARG with *bad_index =
 * the first wavelength whose n^2 <= 1; else *bad_index = -1.  Synchronous. */
int qpm_wavelength_scalars(int process, double thickness, const double *sellmeier_terms, const double *wavelengths_nm,
                           int64_t M, double *dk, double *w, double *hphi, int64_t *bad_index);

/* ------------------------------------------------------ exhaustive search */
/* Global optimum over all 2^n sign patterns of a problem with D = n (n <= 63):
 * pattern `index` has sign j = -1 iff bit n-1-j of index is set (+1 sorts
 * first), patterns are generated on the device chunk_rows at a time, scored
 * with `mode` and reduced; ties go to the lowest index.  Returns the index
 * and its fitness.  Synchronous on `stream`. */
int qpm_brute_force(qpm_problem *p, int n, int mode, int64_t chunk_rows, int64_t *best_index, double *best_fit,
                    void *stream);

/* --------------------------------------------------------------- engine */
typedef struct {
    int algorithm; /* QPM_ALGO_* */
    int fitness_mode;
    int64_t NP, G;
    int64_t seed;
    /* DEParams (optimizer.py:84-101) */
    double f_max, f_min, cr, x_min, x_max;
    /* GWOParams (optimizer.py:104-133) */
    int leader_count;
    double discreteness_factor;
    int divide_by_leader_count;
    /* Schedules thresholds (optimizer.py:136-155) */
    double theta_low_frac, theta_high_frac, range_trigger_frac;
    double explore_boost, exploit_factor, conv_threshold;
    int conv_window;
    int adaptive_branches;
    /* run_gwo bounds and a0 (trace row 0) */
    double gwo_lo, gwo_hi, gwo_a0;
    /* column shard of a multi-GPU run: this engine owns the genes under the
     * fitness segments [floor(rank S / world), floor((rank+1) S / world)) of
     * every individual (S = segments of the problem); 0, 1 for one GPU */
    int shard_rank, shard_world;
} qpm_run_params;

typedef struct qpm_engine qpm_engine;

/* sched: host [G+1][QPM_SCHED_COLS] (see QPM_SCHED_*).  The problem must
 * outlive the engine.  stream is captured by the engine's generation graph;
 * NULL makes the engine create (and own) a non-blocking stream. */
int qpm_engine_create(qpm_engine **out, qpm_problem *prob, const qpm_run_params *params, const double *sched,
                      void *stream);
int qpm_engine_destroy(qpm_engine *e);
/* device bytes held by the engine */
int64_t qpm_engine_device_bytes(const qpm_engine *e);
/* init_population + generation-0 evaluation and trace row (async); once per
 * engine (a second call returns QPM_ERR_STATE) */
int qpm_engine_init(qpm_engine *e);
/* run n generations (async).  use_graph != 0: CUDA-graph replays (one
 * graph of 10 generations plus a one-generation graph for the remainder),
 * captured on first use -- except that an engine without graphs runs a step
 * of fewer than 256 generations with eager launches, which is cheaper than
 * capturing for so short a run (same kernels, bit-identical results);
 * qpm_engine_prepare forces the capture. */
int qpm_engine_step(qpm_engine *e, int64_t n, int use_graph);
/* capture, instantiate and upload every graph a graph-mode step of n
 * generations replays, without running a generation (synchronous); a later
 * qpm_engine_step then only launches.  Lets a caller keep the one-time
 * capture cost out of a timed region. */
int qpm_engine_prepare(qpm_engine *e, int64_t n);
/* select the final best (top-1 of the current population, or best-ever for
 * run_gwo) into the result buffer (async) */
int qpm_engine_finalize(qpm_engine *e);
int qpm_engine_generation(const qpm_engine *e, int64_t *g_done);
/* copies (synchronous on the engine stream) */
int qpm_engine_read_trace(qpm_engine *e, int64_t first_row, int64_t n_rows, double *host_rows);
int qpm_engine_read_best(qpm_engine *e, double *genome, int8_t *proj, double *fitness);
/* qpm_engine_read_best and qpm_engine_read_trace in one call (one pinned
 * staging copy, one synchronisation): what optimizer.run returns. */
int qpm_engine_read_result(qpm_engine *e, int64_t first_row, int64_t n_rows, double *host_rows, double *genome,
                           int8_t *proj, double *fitness);
int qpm_engine_read_population(qpm_engine *e, double *genome, double *fitness);
/* ------------------------------------------------------------ multi-GPU
 * One process per GPU; the genes are sharded in contiguous column ranges
 * aligned to the fitness stitch super-blocks (qpm_run_params.shard_rank /
 * shard_world): rank k of W owns super-blocks [floor(k B / W),
 * floor((k+1) B / W)), B = min(8, S).  Every rank runs the per-gene work (DE
 * trials, wolf moves, draws, fitness segment scans) on its columns of all NP
 * individuals and pre-stitches its super-blocks; those partials (NP x 48 B
 * per owned super-block and wavelength) are all-gathered over NCCL inside
 * the generation graph and every rank finishes and scores all rows, so
 * selection, leaders, statistics and the F update run replicated on
 * identical data.  The stitch tree is the single-GPU one, so a sharded run
 * is bit-identical to the same run on one GPU (fast mode).  Replaces the
 * reference's in-process thread pool (parexec.py:73-120). */
/* rank 0 creates the NCCL id (128 bytes) and broadcasts it to the others */
int qpm_nccl_unique_id(uint8_t *id_out);
/* before qpm_engine_init; rank / world must match the engine's shard */
int qpm_engine_set_comm(qpm_engine *e, int rank, int world, const uint8_t *id);
/* this engine's genes [g0, g0 + d) of the run (0, D on one GPU); genomes and
 * projections read back from a shard cover these columns */
int qpm_engine_columns(const qpm_engine *e, int64_t *g0, int64_t *d);
int qpm_engine_phases(const qpm_engine *e);
int qpm_engine_run_phase(qpm_engine *e, int phase);
/* emulated ranks on one GPU (no communicator): qpm_engine_init stops after
 * the generation-0 fitness scan; exchange, then qpm_engine_init_finish */
int qpm_engine_init_finish(qpm_engine *e);
/* emulated exchange before a phase (or before qpm_engine_init_finish): copy
 * src's super-block partial slot into dst (synchronous) */
int qpm_engine_exchange_from(qpm_engine *dst, qpm_engine *src, int phase);
/* Host-staged exchange (the sharded protocol across a process boundary
 * without NCCL, e.g. over a torch.distributed gloo group; tests use it to
 * run real shard engines in separate processes on one GPU): after a phase,
 * read this rank's partial slot to the host, all-gather the slots, write
 * every peer's slot back, then run the next phase (or qpm_engine_init_finish).
 * slot_doubles: doubles per rank slot.  All three are synchronous. */
int qpm_engine_partials_info(const qpm_engine *e, int64_t *slot_doubles, int *world, int *rank);
int qpm_engine_partials_read(qpm_engine *e, double *host_out);
int qpm_engine_partials_write(qpm_engine *e, int rank, const double *host_in);
/* Wait for the engine's queued work with failure detection: polls the stream
 * and ncclCommGetAsyncError; an asynchronous NCCL error, or no progress
 * within timeout_ms (< 0: no limit), aborts the communicator
 * (ncclCommAbort) and returns QPM_ERR_NCCL -- a peer that died or hangs
 * cannot block this rank forever.  qpm_engine_step also polls the error
 * state between graph launches.  After QPM_ERR_NCCL the engine refuses
 * further steps.  Replaces the reference's BatchEvaluationError failure
 * contract (parexec.py:27-33) on the multi-GPU path. */
int qpm_engine_wait(qpm_engine *e, int64_t timeout_ms);
/* Checkpoint / resume (the counter RNG needs no state): a
 * synchronous host snapshot of an initialised engine -- state (g, F, window,
 * baseline std, leaders, best-ever), fitness, trace rows 0..g, the current
 * individuals (genome rows, sign bits, ±1 flags) in individual order and the
 * best-row buffer.  qpm_engine_restore loads it into a freshly created engine
 * of the same run (algorithm, mode, NP, D, G, seed, schedule, shard) in place
 * of qpm_engine_init; the resumed run is bit-identical to an uninterrupted
 * one.  No reference counterpart (the reference has no mid-run checkpoint). */
int64_t qpm_engine_checkpoint_bytes(const qpm_engine *e);
int qpm_engine_checkpoint(qpm_engine *e, void *host_buf, int64_t bytes);
int qpm_engine_restore(qpm_engine *e, const void *host_buf, int64_t bytes);
/* Invariant checks (builds with -DQPM_CHECKS=1, libqpm_b200_checks.so): after
 * every generation a kernel verifies the slot permutation, the planner's DE
 * picks and j_rand, the leaders, finite fitness and trace, and the planner's
 * generation counter; flags = violation bits (0 = clean), detail = the first
 * violation (code << 24 | index).  QPM_ERR_STATE in other builds. */
int qpm_engine_check_status(qpm_engine *e, uint32_t *flags, uint32_t *detail);
int qpm_engine_cand_ptr(qpm_engine *e, double **cand_dev);
int qpm_engine_stream(qpm_engine *e, void **stream);

/* run n generations eagerly with CUDA events between the stages of each
 * generation (advances the run); stage_ms[k] = mean ms of stage k, names
 * are written as n_stages fixed-width strings of name_len bytes */
int qpm_engine_profile(qpm_engine *e, int64_t n, double *stage_ms, int *n_stages, char *names, int name_len);
/* kernel launches issued by one generation of this engine */
int qpm_engine_launches_per_generation(const qpm_engine *e);
/* device pointer to the fitness vector of individuals [NP] (for tests) */
int qpm_engine_fitness_ptr(qpm_engine *e, double **fit_dev);

#ifdef __cplusplus
}
#endif
#endif /* QPM_B200_H */
