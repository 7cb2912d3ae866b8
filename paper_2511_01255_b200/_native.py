"""ctypes binding of libqpm_b200.so (the C ABI declared in include/qpm_b200.h).

The library is the only compute path: there is no CPU fallback.  Loading
fails loudly if the .so is missing, and every call that returns a non-zero
status raises QpmError with the library's last-error message.
"""

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libqpm_b200.so")

QPM_OK, QPM_ERR_ARG, QPM_ERR_CUDA, QPM_ERR_STATE, QPM_ERR_NCCL = 0, -1, -2, -3, -4
QPM_PROCESS_SHG, QPM_PROCESS_THG = 0, 1
QPM_MODE_FAST, QPM_MODE_EXACT = 0, 1
QPM_ALGO = {"hybrid": 0, "de": 1, "gwo": 2}
SCHED_COLS = 8
(SCHED_F_ENV, SCHED_DECAY, SCHED_P_DIST, SCHED_P_SL, SCHED_P_FLIP, SCHED_EARLY, SCHED_A_NOW) = range(7)

# every symbol include/qpm_b200.h declares (checked by tests/test_native_abi.py)
EXPORTS = (
    "qpm_last_error", "qpm_version", "qpm_device_info", "qpm_release_cached_memory", "qpm_fold_key", "qpm_uniform_fill",
    "qpm_problem_create", "qpm_problem_destroy", "qpm_problem_row_words", "qpm_problem_layout", "qpm_pack_signs",
    "qpm_fitness_bits", "qpm_evaluate_block_host", "qpm_sum_block_host", "qpm_reduce_best", "qpm_brute_force", "qpm_sweep_spectrum",
    "qpm_wavelength_scalars",
    "qpm_engine_create", "qpm_engine_destroy", "qpm_engine_device_bytes", "qpm_engine_init",
    "qpm_engine_step", "qpm_engine_prepare", "qpm_engine_finalize", "qpm_engine_generation", "qpm_engine_read_trace",
    "qpm_engine_read_best", "qpm_engine_read_result", "qpm_engine_read_population", "qpm_engine_profile", "qpm_engine_launches_per_generation",
    "qpm_engine_fitness_ptr", "qpm_nccl_unique_id", "qpm_engine_set_comm", "qpm_engine_columns",
    "qpm_engine_init_finish",
    "qpm_engine_phases", "qpm_engine_run_phase", "qpm_engine_exchange_from", "qpm_engine_cand_ptr",
    "qpm_engine_stream", "qpm_engine_partials_info", "qpm_engine_partials_read", "qpm_engine_partials_write",
    "qpm_engine_wait", "qpm_engine_check_status", "qpm_engine_checkpoint_bytes", "qpm_engine_checkpoint",
    "qpm_engine_restore",
)


class QpmError(RuntimeError):
    """A libqpm_b200 call failed; the message is the library's last error."""


class RunParams(ctypes.Structure):
    """Mirror of qpm_run_params (include/qpm_b200.h)."""

    _fields_ = [
        ("algorithm", ctypes.c_int),
        ("fitness_mode", ctypes.c_int),
        ("NP", ctypes.c_int64),
        ("G", ctypes.c_int64),
        ("seed", ctypes.c_int64),
        ("f_max", ctypes.c_double),
        ("f_min", ctypes.c_double),
        ("cr", ctypes.c_double),
        ("x_min", ctypes.c_double),
        ("x_max", ctypes.c_double),
        ("leader_count", ctypes.c_int),
        ("discreteness_factor", ctypes.c_double),
        ("divide_by_leader_count", ctypes.c_int),
        ("theta_low_frac", ctypes.c_double),
        ("theta_high_frac", ctypes.c_double),
        ("range_trigger_frac", ctypes.c_double),
        ("explore_boost", ctypes.c_double),
        ("exploit_factor", ctypes.c_double),
        ("conv_threshold", ctypes.c_double),
        ("conv_window", ctypes.c_int),
        ("adaptive_branches", ctypes.c_int),
        ("gwo_lo", ctypes.c_double),
        ("gwo_hi", ctypes.c_double),
        ("gwo_a0", ctypes.c_double),
        ("shard_rank", ctypes.c_int),
        ("shard_world", ctypes.c_int),
    ]


_lib = None


def lib():
    """Load (once) and return the library with typed signatures."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("QPM_LIB", LIB_PATH)  # A/B builds of the same library (development)
    if not os.path.exists(path):
        raise QpmError(f"{path} is missing: build it with `python -m paper_2511_01255_b200.build` "
                       "(there is no CPU fallback)")
    L = ctypes.CDLL(path)
    P, I64, I32, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
    sig = {
        "qpm_last_error": (ctypes.c_char_p, []),
        "qpm_version": (I32, []),
        "qpm_release_cached_memory": (I32, []),
        "qpm_device_info": (I32, [P, P, P]),
        "qpm_fold_key": (ctypes.c_uint64, [I64, I32, P]),
        "qpm_uniform_fill": (I32, [ctypes.c_uint64, ctypes.c_uint64, I64, P, P]),
        "qpm_problem_create": (I32, [P, I32, I32, I32, I64, P, P, P, P, D, D, D, I32]),
        "qpm_problem_layout": (I32, [P, P, P, P]),
        "qpm_problem_destroy": (I32, [P]),
        "qpm_problem_row_words": (I64, [P]),
        "qpm_pack_signs": (I32, [P, I64, I64, P, I64, P]),
        "qpm_fitness_bits": (I32, [P, P, I64, P, I64, P, I32, P]),
        "qpm_evaluate_block_host": (I32, [P, P, I64, P, I32]),
        "qpm_sum_block_host": (I32, [P, I32, P, I64, P]),
        "qpm_reduce_best": (I32, [P, I64, I32, P, P]),
        "qpm_brute_force": (I32, [P, I32, I32, I64, P, P, P]),
        "qpm_sweep_spectrum": (I32, [I32, ctypes.c_double, I64, P, I64, P, P, P, I64, P]),
        "qpm_wavelength_scalars": (I32, [I32, ctypes.c_double, P, P, I64, P, P, P, P]),
        "qpm_engine_create": (I32, [P, P, ctypes.POINTER(RunParams), P, P]),
        "qpm_engine_destroy": (I32, [P]),
        "qpm_engine_device_bytes": (I64, [P]),
        "qpm_engine_init": (I32, [P]),
        "qpm_engine_step": (I32, [P, I64, I32]),
        "qpm_engine_prepare": (I32, [P, I64]),
        "qpm_engine_finalize": (I32, [P]),
        "qpm_engine_generation": (I32, [P, P]),
        "qpm_engine_read_trace": (I32, [P, I64, I64, P]),
        "qpm_engine_read_best": (I32, [P, P, P, P]),
        "qpm_engine_read_result": (I32, [P, I64, I64, P, P, P, P]),
        "qpm_engine_read_population": (I32, [P, P, P]),
        "qpm_engine_profile": (I32, [P, I64, P, P, P, I32]),
        "qpm_engine_launches_per_generation": (I32, [P]),
        "qpm_engine_fitness_ptr": (I32, [P, P]),
        "qpm_nccl_unique_id": (I32, [P]),
        "qpm_engine_set_comm": (I32, [P, I32, I32, P]),
        "qpm_engine_columns": (I32, [P, P, P]),
        "qpm_engine_init_finish": (I32, [P]),
        "qpm_engine_phases": (I32, [P]),
        "qpm_engine_run_phase": (I32, [P, I32]),
        "qpm_engine_exchange_from": (I32, [P, P, I32]),
        "qpm_engine_cand_ptr": (I32, [P, P]),
        "qpm_engine_stream": (I32, [P, P]),
        "qpm_engine_partials_info": (I32, [P, P, P, P]),
        "qpm_engine_partials_read": (I32, [P, P]),
        "qpm_engine_partials_write": (I32, [P, I32, P]),
        "qpm_engine_wait": (I32, [P, I64]),
        "qpm_engine_check_status": (I32, [P, P, P]),
        "qpm_engine_checkpoint_bytes": (I64, [P]),
        "qpm_engine_checkpoint": (I32, [P, P, I64]),
        "qpm_engine_restore": (I32, [P, P, I64]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return _lib


def check(rc: int, what: str = "") -> None:
    if rc != 0:
        msg = lib().qpm_last_error().decode(errors="replace")
        raise QpmError(f"{what or 'libqpm_b200'} failed (status {rc}): {msg}")


def require_cuda():
    """The device the engine runs on; raises when there is none."""
    import torch

    if not torch.cuda.is_available():
        raise QpmError("no CUDA device: paper_2511_01255_b200 runs only on the GPU (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)
