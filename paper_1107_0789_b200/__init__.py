"""B200-native DFC hot path (arXiv 1107.0789): Python view of libdfcg.so.

The product is the C-ABI library ``_lib/libdfcg.so`` (include/dfcg.h): hand-written sm_100a
FP64 CUDA kernels for the APG base solvers and the DFC combiners, driven by a C++ host
orchestrator. This module is a thin ctypes mirror of that ABI with the reference's names
(P/include/dfc/*.hpp): ``apg_mc``, ``apg_rmf``, ``column_project``, ``gen_nystrom``,
``average_estimates``, ``random_project``, ``svd_of_product``, ``dfc_run``.

There is no CPU fallback: importing works anywhere, but every compute call needs the CUDA
library and a GPU and raises if either is missing.
"""
import os as _os

# Concurrent block solves use two streams each; 32 hardware work queues keep them from aliasing
# onto shared queues (read at CUDA context creation: effective when this package is imported
# before the process initialises CUDA; bench.py sets it first thing).
_os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

from ._lib import (  # noqa: F401,E402
    ApgConfig,
    BlockError,
    DfcError,
    ParseError,
    Estimate,
    McSolver,
    Observed,
    Report,
    apg_mc,
    apg_rmf,
    average_estimates,
    build,
    column_project,
    context,
    dfc_run,
    gen_nystrom,
    high_accuracy,
    lib,
    lib_path,
    project_block,
    random_project,
    svd_of_product,
)
from .host import (  # noqa: F401,E402
    extract_columns,
    extract_subproblems,
    extract_rows,
    format_triplets,
    gen_mc_instance,
    load_triplets,
    parse_triplets,
    save_triplets,
    gen_recsys_instance,
    launch_count,
    work_counters,
    prof_collect,
    prof_enable,
    gen_rmf_instance,
    median_rank,
    partition_columns,
    sample_without_replacement,
    SeededRng,
)
