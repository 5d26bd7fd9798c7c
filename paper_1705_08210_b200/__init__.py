"""B200-native Proportional Similarity (Czekanowski) metric engine.

Drop-in for the hot path of ``propsim`` (reference __init__.py:5-36): the
same entry points ``run_2way`` / ``run_3way`` and domain types, computed by
hand-written sm_100a kernels in ``_lib/libpsim.so`` (C ABI: include/psim.h).
There is no CPU fallback: without the library or a GPU, runs raise.
"""

__version__ = "0.1.0"

from .api import RunResult, TrafficStats, resolve_kernel, run_2way, run_3way  # noqa: F401
from .domain import (  # noqa: F401
    ConfigError,
    DataError,
    DecompGrid,
    EngineError,
    MetricRecord,
    Problem,
    RankCoords,
    TupleId,
    coords_of_rank,
    iter_pairs,
    iter_triples,
    pair_index,
    pair_unindex,
    rank_of_coords,
    triple_index,
    triple_unindex,
    unique_tuple_count,
)
from .plan import owns_pair, owns_triple, plan_2way, plan_3way, stage_range  # noqa: F401
from .vectorfile import VectorFileSpec, write_vectors  # noqa: F401
from .synthetic import (  # noqa: F401
    Checksum128,
    SyntheticSpec,
    checksum,
    combine_checksums,
    gen_analytic,
    gen_random_exact,
    gen_uniform,
    mix64,
    value_bits,
)
from .output import (  # noqa: F401
    MetricOutputSpec,
    dequantize_byte,
    owned_tuples,
    quantize_byte,
    read_metrics,
    read_run_output,
    read_run_values,
    reconstruct_index,
    write_metrics,
    write_run_output,
)
