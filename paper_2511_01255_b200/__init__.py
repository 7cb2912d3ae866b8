"""B200-native HWSDA population engine (drop-in for the qpmdesign hot path).

The reference's optimiser / fitness API is kept:

    from paper_2511_01255_b200 import (ObjectiveSpec, make_objective, run_hybrid,
                                       default_dispersion)
    obj = make_objective(ObjectiveSpec("single_thg", (1404.0,)), default_dispersion(),
                         thickness_um=1.0, count=1000)
    result = run_hybrid(obj, dimension=1000, pop_size=50, generations=500, seed=0)

Compute runs only in libqpm_b200.so (hand-written sm_100a CUDA, C ABI in
include/qpm_b200.h); there is no CPU fallback.  Host-side modules hold the
setup that the reference also does on the host (dispersion and phase tables,
schedule scalars).
"""

from . import _native
from .objectives import (
    GpuPatternObjective,
    ObjectiveSpec,
    PatternObjective,
    fitness_multi,
    fitness_single,
    make_objective,
    multi_objective,
)
from .optimizer import (
    ALGORITHMS,
    AdaptiveState,
    DEParams,
    Engine,
    GWOParams,
    Individual,
    Population,
    RunResult,
    Schedules,
    adaptive_f_update,
    run,
    run_de,
    run_gwo,
    run_hybrid,
    schedule_table,
)
from .search import brute_force_oracle, lexicographic_signs
from .spectrum import sweep_spectra, sweep_spectrum
from .trials import ComparisonReport, RunStatistics, TrialRecord, compare_algorithms, run_trials
from .parexec import BatchEvaluationError, BatchJob, TimingReport, evaluate_batch, reduce_best, time_run
from .tables import (
    SELLMEIER_SETS,
    DispersionModel,
    DomainPattern,
    MismatchTable,
    PhaseMismatchPair,
    default_dispersion,
    phase_mismatches,
    refractive_index,
)

__version__ = "0.1.0"


def kernel_backend() -> str:
    return "cuda-sm_100a"
