"""paper_1702_04739_b200: B200-native isoperimetric-tree clustering.

Drop-in for the clustering path of the reference package `isoclust`
(/root/reference/pkg/src/isoclust, arXiv 1702.04739): `run_pipeline(points,
k, ...)` returns the same PipelineRun / MisoResult structures, bit-exact
labels, and runs every arithmetic stage as hand-written sm_100a CUDA kernels
behind the C ABI in include/isoclust_b200.h (libisoclust_b200.so).
"""
from ._lib import InfeasibleSubpartitionError
from .harness import (
    BENCH_CSV_HEADER,
    BenchRecord,
    DataFormatError,
    DepthSchedule,
    WorkerPool,
    benchmark,
    class_count,
    generate_random,
    load_labels,
    load_points,
    misclassification_rate,
    save_labels,
    save_points,
    standardize,
    write_bench_csv,
)
from .pipeline import (
    ENGINES,
    WORKERS_ENV_VAR,
    auto_sigma_points,
    decide,
    extrema,
    minimum_spanning_tree,
    node_weights_points,
    par_decide,
    par_solve_miso,
    resolve_workers,
    run_pipeline,
    solve_miso,
    summarize,
    tree_from_parent_list,
)
from .stages import (
    MAX_POINTS,
    auto_sigma,
    brute_force_miso,
    distance_matrix,
    exclusive_scan,
    extract_labels,
    flow,
    min_reduce,
    node_weights,
    potentials,
    prim_mst,
    reverse_bfs_order,
    subpartition_cost,
    sum_reduce,
    total_distance,
    validate_distance_matrix,
    vertex_weights,
)
from .types import (
    BRACKET_EPS,
    MAX_ITERATIONS,
    NO_VERTEX,
    DecisionOutcome,
    Extrema,
    MisoResult,
    NodeWeights,
    PipelineRun,
    RootedTree,
    miso_results_equal,
    outcomes_equal,
)

__version__ = "0.1.0"

__all__ = [
    "BENCH_CSV_HEADER", "BenchRecord", "DataFormatError", "DepthSchedule", "WorkerPool", "benchmark",
    "class_count", "generate_random", "load_labels", "load_points", "misclassification_rate", "save_labels",
    "save_points", "standardize", "write_bench_csv",
    "BRACKET_EPS", "DecisionOutcome", "ENGINES", "Extrema", "InfeasibleSubpartitionError",
    "MAX_ITERATIONS", "MAX_POINTS", "MisoResult", "NO_VERTEX", "NodeWeights", "PipelineRun", "RootedTree",
    "WORKERS_ENV_VAR", "auto_sigma", "auto_sigma_points", "brute_force_miso", "decide", "distance_matrix", "exclusive_scan",
    "extract_labels", "extrema", "flow", "min_reduce", "minimum_spanning_tree", "miso_results_equal",
    "node_weights", "node_weights_points", "outcomes_equal", "par_decide", "par_solve_miso", "potentials",
    "prim_mst", "resolve_workers", "reverse_bfs_order", "run_pipeline", "solve_miso", "subpartition_cost",
    "sum_reduce", "summarize", "total_distance", "tree_from_parent_list", "validate_distance_matrix",
    "vertex_weights", "__version__",
]
