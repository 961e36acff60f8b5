"""B200-native batched strategy simulator -- the hot path of arXiv 2002.06790's dfsim.

Drop-in surface (same names and signatures as the reference's pkg/src/dfsim/__init__.py:6-43
for the hot path): ``simulate``, ``critical_path``, ``estimate_all``,
``expand_data_parallel``, and the schedule consumers ``summarize`` / ``to_trace``;
batched entry points: ``sweep`` / ``sweep_variants`` / ``sweep_sharded`` (multi-GPU) (``SweepResult.summaries`` / ``.trace`` report on the
schedules left in HBM).  Every compute call runs
hand-written sm_100a kernels from ``libdfsim_b200.so`` through the C-ABI in
``include/dfsim_b200.h``; there is no CPU fallback.
"""

from .errors import (  # noqa: F401
    ConfigError,
    CycleError,
    DfsimError,
    FitError,
    FitQualityWarning,
    MissingDurationError,
    NativeError,
    PatternWarning,
    UnknownCollectiveError,
    UnknownOpError,
)
from .model import (  # noqa: F401
    CollectiveConfig,
    DataflowGraph,
    DeviceSpec,
    DurationEntry,
    DurationTable,
    ExpandedGraph,
    LinearCostModel,
    LinkRecord,
    OpNode,
    OpSignature,
    ProfileDB,
    ProfileRecord,
    Schedule,
    ScheduledNode,
    StrategyConfig,
    TensorShape,
    load_profiles,
    make_graph,
    parse_config,
    parse_graph,
    serialize_graph,
    utilization,
)
from .batch import SweepResult, TopologyClass, gather_best, sweep, sweep_variants  # noqa: F401
from .sharded import sweep_sharded  # noqa: F401
from .estimate import estimate_all, estimate_batch  # noqa: F401
from .expansion import expand_class, expand_data_parallel  # noqa: F401
from .lowering import fit_for_grid, fit_for_grid_many, fit_linear, fit_linear_many, node_features  # noqa: F401
from .document import DocumentGraph, load_graph  # noqa: F401
from .ps import expand_parameter_server  # noqa: F401
from .reporting import SummaryReport, render_summary_text, summarize, to_trace, trace_intervals  # noqa: F401
from .simulator import critical_path, simulate  # noqa: F401
from .scalar import (  # noqa: F401
    allreduce_time,
    apply_overrides,
    comm_batch,
    comm_time_us,
    predict,
    predict_batch,
    query_exact,
    query_grid,
    query_link,
    topological_order,
    transfer_time,
)

__version__ = "0.1.0"
