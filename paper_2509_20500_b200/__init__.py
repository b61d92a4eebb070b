"""B200-native (sm_100a) hot path of arXiv 2509.20500: asynchronous SP-LiDAR dead-time Markov chain.

    P~0 = rownorm((1 lambda^T) . exp.(-Lambda L - D))       (§3.4)   build_base
    P~  = J_l P~0,  l = ceil((t_d mod t_r) / Delta)         (Thm 2)   apply_deadtime / folded
    pi P~ = pi               stationary, sweep

The compute path is libsplidar.so (include/splidar.h); this package only marshals arguments.
"""
from .splidar import (  # noqa: F401
    ENOCONV, EINVAL, ENOSPACE, ECUDA, EZEROROW, OK, F32, F64, LIB_PATH, Plan, SolveInfo, SplidarError,
    apply_deadtime, build_base, build_base_batched, build_info, empty_matrix, flux_vectors, leading_dim,
    lib_path, shift, solve_host, stationary, sweep, workspace, workspace_bytes,
    SpectralInfo, bin_trajectory, flux_items, mixing_steps, second_eigenvalue, second_eigenvalue_dense,
    stationary_structured,
    structured_workspace, StructPlan, build_eq4, monte_carlo, lambda2_of, build_base_rows, ShardPlan,
    stationary_multi, plan_cache_clear,
)
