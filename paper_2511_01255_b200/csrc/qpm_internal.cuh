// qpm_internal.cuh -- host-side internals shared by the .cu translation units.
#pragma once

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <mutex>
#include <string>

#include <cuda_runtime.h>

#include <utility>
#include <vector>

#include "../../include/qpm_b200.h"

namespace qpm {

void set_error(const char *fmt, ...);

#define QPM_CUDA_TRY(expr)                                                                           \
    do {                                                                                             \
        cudaError_t _e = (expr);                                                                     \
        if (_e != cudaSuccess) {                                                                     \
            ::qpm::set_error("%s:%d %s -> %s", __FILE__, __LINE__, #expr, cudaGetErrorString(_e)); \
            return QPM_ERR_CUDA;                                                                     \
        }                                                                                            \
    } while (0)

#define QPM_LAUNCH_CHECK()                                                                                 \
    do {                                                                                                   \
        cudaError_t _e = cudaGetLastError();                                                               \
        if (_e != cudaSuccess) {                                                                           \
            ::qpm::set_error("%s:%d kernel launch failed: %s", __FILE__, __LINE__, cudaGetErrorString(_e)); \
            return QPM_ERR_CUDA;                                                                           \
        }                                                                                                  \
    } while (0)

#define QPM_ARG_CHECK(cond, msg)                               \
    do {                                                       \
        if (!(cond)) {                                         \
            ::qpm::set_error("invalid argument: %s", (msg));   \
            return QPM_ERR_ARG;                                \
        }                                                      \
    } while (0)

#ifndef QPM_FIT_THREADS
#define QPM_FIT_THREADS 128
#endif
constexpr int kFitThreads = QPM_FIT_THREADS;  // rows per fast-fitness CTA (one lane per row), several wavelengths
#ifndef QPM_FIT_THREADS1
#define QPM_FIT_THREADS1 256
#endif
constexpr int kFitThreadsMax = QPM_FIT_THREADS1;  // ... one wavelength (and the launch bound)
constexpr int kQuadsPerChunk = 32;    // 128 domains = 4 u32 words per chunk
// complex entries per quad of the fast scan's tables: B[8], E[8], I[8] by the
// 3 relative signs (s0 applied by XOR in the scan).  One table is one
// 128-byte shared-memory row, so a quarter-warp's 16-byte loads never
// conflict (measured: folding s0 into 16-entry tables cut the scan's
// instructions by 31 % but made it shared-memory-wavefront bound, C5 fitness
// 2029 -> 3241 us)
constexpr int kQuadIdx = 8;
constexpr int kQuadEntries = 3 * kQuadIdx;
constexpr int kPartDoubles = 6;       // acc, P, T (complex) per (row, wavelength, segment)

inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

// device-resident problem (one PatternObjective)
struct Problem {
    int process = 1, multi = 0, n_wl = 1;
    int64_t D = 0;
    int64_t W = 0;        // u32 words per bit row (multiple of 4)
    int64_t nquads = 0;   // W * 8
    int64_t nchunks = 0;  // W / 4
    int seg_chunks = 1;   // chunks per fast-scan segment
    int S = 1;            // segments per row
    int nsb = 1;          // stitch super-blocks, min(8, S) (qpm_finish.cuh)
    double scale = 1.0, g0 = 2.0, beta = 1.0;
    double2 *e1 = nullptr;  // [n_wl][D]
    double2 *b = nullptr;   // [n_wl][D] (thg)
    double2 *qt = nullptr;  // [n_wl][nquads][24]
    double2 *w = nullptr;   // [n_wl]
    double2 *h = nullptr;   // [n_wl]
    // scratch of the problem's own entry points (qpm_fitness_bits, host path);
    // every engine owns its scratch, so engines sharing a problem never race
    struct FitScratch *own = nullptr;
    // recorded after every use of `own` on whatever stream made it; the next
    // user's stream waits on it, so qpm_fitness_bits on a caller's stream and
    // the host paths on hp_stream never overlap in the shared scratch, and
    // the scratch is only regrown or released once its last user is done
    cudaEvent_t own_ev = nullptr;
    // host plugin path buffers
    int8_t *hp_signs = nullptr;
    uint32_t *hp_bits = nullptr;
    double *hp_out = nullptr;
    int64_t hp_rows = 0;
    uint32_t *hp_pinned = nullptr;  // host-packed bit rows (pinned) of the host paths
    int64_t hp_pinned_rows = 0;
    cudaStream_t hp_stream = nullptr;
    int64_t device_bytes = 0;
    // serialises the host-synchronous entry points (evaluate_block_host,
    // sum_block_host, brute_force): the reference's parexec calls
    // evaluate_block from several worker threads at once (parexec.py:88-105)
    // and they share hp_* and the scratch
    std::mutex *mu = nullptr;
};

// per-row segment partials and per-wavelength gains of one fitness launch
struct FitScratch {
    double *part = nullptr;
    double *gains = nullptr;
    int64_t rows = 0;
    int64_t bytes = 0;
    size_t part_bytes = 0, gains_bytes = 0;
};
// Process-wide cache of device blocks (exact-size reuse): engines created
// and destroyed back to back (one run_hybrid call after another) skip
// cudaMalloc / cudaFree, whose implicit device synchronisation and page
// mapping otherwise cost tens of milliseconds per run.
void *dev_cache_alloc(size_t bytes);
void dev_cache_release(void *p, size_t bytes);
void dev_cache_trim();

int scratch_reserve(const Problem *p, FitScratch *fs, int64_t rows);
void scratch_free(FitScratch *fs);
// launch the fitness of `rows` bit rows (row_index may be null) into out
int launch_fitness(const Problem *p, FitScratch *fs, const uint32_t *bits, int64_t row_words,
                   const int32_t *row_index, int64_t rows, double *out, int mode, cudaStream_t stream, int *launches,
                   bool pdl = false);
// Programmatic dependent launch: a kernel launched with pdl = true is staged
// while its stream predecessor runs and starts when the predecessor exits, so
// the launch latency overlaps the predecessor's tail.  It must call pdl_wait()
// before touching anything the predecessor wrote (a no-op when launched
// without the attribute).  No kernel triggers its dependents early
// (griddepcontrol.launch_dependents): measured on B200, an early trigger let
// dependents observe stale data in about one C2 run in eight, and the early
// residents slowed the primary down.
// (Measured again with the device timeline, tools/timeline.py: triggering
// dependents once every CTA has passed its wait made the C2 generation
// 119.7 -> 133.3 us; the early-resident k_fit_finish CTAs doubled k_fit_fast.)
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// Optional early trigger (build knob QPM_PDL_TRIGGER, a bitmask: 1 trial, 2
// fitness scan, 4 fused finish + selection, 8 wolf apply): the kernel lets its
// dependent grid launch once every CTA has passed its wait, so the dependent's
// CTAs are resident when it ends.  Safe because every kernel of the chain
// waits (griddepcontrol.wait) before touching anything and before exiting:
// a dependent's wait then covers the whole chain behind it.
#ifndef QPM_PDL_TRIGGER
#define QPM_PDL_TRIGGER 0
#endif
template <int BIT>
__device__ __forceinline__ void pdl_trigger() {
    if (QPM_PDL_TRIGGER & BIT) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Device-side kernel timeline (development builds with -DQPM_TRACE only):
// thread 0 of every CTA stamps %globaltimer at entry, after pdl_wait and at
// exit; the last CTA of a launch logs (min entry, min start, max exit).  The
// graph-replayed generation can then be read back as it really ran (PDL
// overlap included), which CUDA events between stages cannot show.
// Ids: 0 de_trial, 1 fit_fast, 2 fit_finish, 3 select_topk, 4 gwo_apply,
// 5 select_stats, 6 plan_rows, 7 plan_bump, 8 plan_wolf.  Each translation unit has its own log.
constexpr int kTraceIds = 9, kTraceLen = 4096;
#ifdef QPM_TRACE
struct TraceAcc {
    unsigned long long t_entry, t_start, t_end;
    unsigned int done, launch;
};
static __device__ TraceAcc g_tacc[kTraceIds];
static __device__ unsigned long long g_tlog[kTraceIds][kTraceLen][3];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
struct TraceScope {
    int id;
    __device__ __forceinline__ static bool lead() { return threadIdx.x == 0 && threadIdx.y == 0 && threadIdx.z == 0; }
    __device__ explicit TraceScope(int i) : id(i) {
        if (lead()) atomicMin(&g_tacc[id].t_entry, gtimer());
    }
    __device__ void started() {
        if (lead()) atomicMin(&g_tacc[id].t_start, gtimer());
    }
    __device__ ~TraceScope() {
        if (!lead()) return;
        atomicMax(&g_tacc[id].t_end, gtimer());
        __threadfence();
        const unsigned n = atomicAdd(&g_tacc[id].done, 1u);
        if (n + 1 == gridDim.x * gridDim.y * gridDim.z) {
            __threadfence();
            const unsigned L = g_tacc[id].launch % kTraceLen;
            g_tlog[id][L][0] = atomicExch(&g_tacc[id].t_entry, ~0ULL);
            g_tlog[id][L][1] = atomicExch(&g_tacc[id].t_start, ~0ULL);
            g_tlog[id][L][2] = atomicExch(&g_tacc[id].t_end, 0ULL);
            g_tacc[id].done = 0;
            g_tacc[id].launch += 1;
            __threadfence();
        }
    }
};
#define QTRACE(id) ::qpm::TraceScope qtrace_scope_(id)
#define QTRACE_STARTED() qtrace_scope_.started()
// intra-kernel stamps of CTA 0, thread 0: g_stamp[id][launch % 64][slot]
static __device__ unsigned long long g_stamp[kTraceIds][64][8];
#define QSTAMP(slot)                                                                                   \
    do {                                                                                               \
        if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && ::qpm::TraceScope::lead())        \
            ::qpm::g_stamp[qtrace_scope_.id][::qpm::g_tacc[qtrace_scope_.id].launch % 64][slot] =      \
                ::qpm::gtimer();                                                                       \
    } while (0)
// the same from a single calling thread of any CTA (e.g. a last-CTA tail)
#define QSTAMP_ANY(slot)                                                                               \
    do {                                                                                               \
        ::qpm::g_stamp[qtrace_scope_.id][::qpm::g_tacc[qtrace_scope_.id].launch % 64][slot] =          \
            ::qpm::gtimer();                                                                           \
    } while (0)
// the same for an explicit kernel id, outside the kernel's own scope
#define QSTAMP_ID(kid, slot)                                                                           \
    do {                                                                                               \
        ::qpm::g_stamp[kid][::qpm::g_tacc[kid].launch % 64][slot] = ::qpm::gtimer();                   \
    } while (0)
// host: reset the accumulators / copy the log of this translation unit
static inline int trace_reset_tu() {
    std::vector<TraceAcc> init(kTraceIds, TraceAcc{~0ULL, ~0ULL, 0ULL, 0u, 0u});
    return cudaMemcpyToSymbol(g_tacc, init.data(), sizeof(TraceAcc) * kTraceIds) == cudaSuccess ? 0 : -1;
}
static inline int trace_read_tu(unsigned long long *log, unsigned int *launches) {
    std::vector<TraceAcc> acc(kTraceIds);
    if (cudaMemcpyFromSymbol(acc.data(), g_tacc, sizeof(TraceAcc) * kTraceIds) != cudaSuccess) return -1;
    for (int i = 0; i < kTraceIds; ++i) launches[i] = acc[i].launch;
    return cudaMemcpyFromSymbol(log, g_tlog, sizeof(g_tlog)) == cudaSuccess ? 0 : -1;
}
static inline int trace_stamps_tu(unsigned long long *out) {
    return cudaMemcpyFromSymbol(out, g_stamp, sizeof(g_stamp)) == cudaSuccess ? 0 : -1;
}
#else
#define QTRACE(id)
#define QTRACE_STARTED()
#define QSTAMP(slot)
#define QSTAMP_ANY(slot)
#define QSTAMP_ID(kid, slot)
#endif

template <typename... KArgs, typename... Args>
cudaError_t launch_k(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                     Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

int launch_reduce_best(const double *values, int64_t n, int k, int32_t *idx_out, cudaStream_t stream);
// fast-mode segment scan into part ([n_wl][rows][S_stride][6], S_stride >= p->S)
int launch_fitness_scan(const Problem *p, const uint32_t *bits, int64_t row_words, const int32_t *row_index,
                        int64_t rows, double *part, int S_stride, cudaStream_t stream, int *launches, bool pdl);
// stitch + objective (the layout of f.part is in the FinishArgs, qpm_finish.cuh)
int launch_fitness_finish(const struct FinishArgs &f, double *out, cudaStream_t stream, int *launches, bool pdl);
// a column shard's owned super-block partials into its all-gather slot
int launch_prestitch(const Problem *p, const double *part, int S_loc, int seg_lo, int rank, int world, int SB_slot,
                     int64_t rows, double *slot, cudaStream_t stream, int *launches, bool pdl);
int launch_fitness_partials(const Problem *p, FitScratch *fs, const uint32_t *bits, int64_t row_words,
                            const int32_t *row_index, int64_t rows, int mode, cudaStream_t stream, int *launches,
                            bool pdl, int *S_out);
}  // namespace qpm
struct qpm_problem;
namespace qpm {
int problem_slice(const Problem *p, int64_t g0, int64_t Dl, qpm_problem **out);

}  // namespace qpm

struct qpm_problem {
    qpm::Problem p;
};
