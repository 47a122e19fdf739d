"""B200-native partial-update MACE (arXiv 1911.09278) — the reconstruction hot path.

Drop-in for the reference package's hot-path API (``macetomo``): the same
entry points, types and error behaviour, backed by hand-written sm_100a
kernels in ``libmace_b200.so`` (see include/mace_b200.h).
"""

from .denoisers import DenoiserSpec, denoise, make_denoiser
from .geometry import (Geometry, SparseViewMatrix, ViewSubset, back_project, build_system_matrix, forward_project,
                       load_system_matrix, partition_views, roi_mask, save_system_matrix)
from .icd import (REFRESH_EVERY, AgentWorkspace, ConvergenceError, icd_map_solve, partial_update_prox,
                  pixel_update, prox_solve)
from .mace import (ConvergenceLog, EquitCounter, MaceConfig, MaceResult, PeerComm, ResidualReport, WorkerPool, average,
                   consensus_G, consensus_GH, equilibrium_residuals, mace_pnp_solve, mace_solve, mann_step,
                   new_stack, nrmse, reflect_G, mace_solve_batch)
from .models import QGGMRF, QUADRATIC, PriorParams, ReconProblem, book_to_reference_beta, map_cost, map_gradient, neighbor_table

__version__ = "0.1.0"
