"""B200-native MDOT-PNCG hot path (arxiv 2307.08507).

Thin ctypes binding of the C ABI in include/mdot.h; every O(n^2) and O(n)
step runs in the CUDA library libmdot_b200.so (built in-tree for sm_100a by
paper_2307_08507_b200/build.py).  There is no CPU fallback: importing this
package raises if the library is missing or cannot be loaded.

Python names mirror the C entry points:
    mdot_solve, mdot_sinkhorn, mdot_solve_batch, mdot_marginals, mdot_round,
    mdot_get_unique_id, mdot_comm_create, mdot_comm_destroy,
    mdot_solve_sharded, mdot_solve_sharded_2d, mdot_last_error, mdot_last_screen_stats
Arrays may be CUDA torch tensors (MDOT_MEM_DEVICE, used in place on the
current stream) or host numpy arrays / CPU tensors (MDOT_MEM_HOST, copied in
and out inside the call).
"""
from ._binding import (  # noqa: F401
    LIB_PATH,
    MDOT_BETA_PFR,
    MDOT_BETA_PPR,
    MDOT_BETA_PPR_AF,
    MDOT_BETA_PPR_PLUS,
    MDOT_COST_DENSE_F32,
    MDOT_COST_DENSE_F64,
    MDOT_COST_SQEUCLID_DOT_F32,
    MDOT_COST_SQEUCLID_F32,
    MDOT_PREC_AUTO,
    MDOT_PREC_F32P,
    MDOT_PREC_F64P,
    MDOT_PROJ_NCG,
    MDOT_PROJ_PNCG_JACOBI,
    MDOT_PROJ_PNCG,
    MDOT_PROJ_SINKHORN,
    MDOT_SCHED_ADAPTIVE,
    MDOT_SCHED_DOUBLING,
    MDOT_SCHED_EXPLICIT,
    MDOT_SCHED_FIXED,
    MDOT_WARM_CARRY,
    MDOT_WARM_SCALED,
    MDOT_WARM_ZERO,
    STATUS_NAMES,
    TraceRec,
    MdotError,
    lib,
    mdot_comm_create,
    mdot_comm_create_local,
    mdot_comm_enable_peer,
    mdot_comm_destroy,
    mdot_get_unique_id,
    mdot_last_error,
    mdot_last_screen_stats,
    mdot_marginals,
    mdot_round,
    mdot_sinkhorn,
    mdot_solve,
    mdot_solve_batch,
    mdot_solve_sharded,
    mdot_solve_sharded_2d,
    options,
    read_trace,
    schedule,
)
