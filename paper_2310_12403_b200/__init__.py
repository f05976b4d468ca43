"""coopbatch on B200: the cooperative sample + dedup + feature-gather path of
arXiv 2310.12403, as hand-written sm_100a kernels behind a C-ABI
(include/coopbatch_cuda.h) with a host mirror of the reference's API."""
from .coopbatch import (  # noqa: F401
    KAPPA_INFINITY, MODE_COOP, MODE_INDEP, BipartiteBlock, CapacityError, CoopSampleResult,
    UncertifiedError,
    CudaError, ExchangeRecord, cross_edge_ratio, FeatureStore, FormatError, Graph, InputError, LayerStack,
    PartitionMap,
    Plan, SamplerConfig, SamplerKind, SeedSchedule, coop_sample, expand, hash_bits,
    hash_uniform, indep_sample, load_inputs, mix64, partition_from_owner, partition_random,
    sample_block, sample_full, sample_labor0, sample_ns, sample_rw, schedule_advance, LayerMetrics, PeMetrics, step_metrics,
    parse_result)
from .cache import (  # noqa: F401
    BatchMode, CacheOutcome, CacheStats, ClockCache, DependentExperimentResult, DependentStepRow,
    LruCache,
    MinibatchSchedule, feature_load_sim, lru_access, nested_batches, run_dependent_experiment,
    shuffled_order, stack_fingerprint)
from .train import GcnModel, TrainStepResult, coop_train_step, indep_train_step  # noqa: F401,E402
from .analysis import (  # noqa: F401,E402
    ConcavityEntry, ConcavityReport, SeedMode, WorkCurve, WorkCurvePoint, concavity_check,
    work_curve)
