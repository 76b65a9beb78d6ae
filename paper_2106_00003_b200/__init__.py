"""B200-native (sm_100a) data-parallel hot path of arXiv 2106.00003 (Hamze): circle-method
round-robin schedule, block-parallel Givens forward on an n x m batch (or I -> U), and the
replay backward (dX, dtheta) with a deterministic dtheta reduction over the m columns.

The compute lives in libgivens.so (include/givens.h); this package is the thin binding.
"""
from .ops import (GivensApply, fast_apply, fast_build_U, HostPipeline, Layout, apply, gemm_apply, gemm_backward, gemm_workspace, backward, build_U, givens_apply, index_trace, mask_from_dims,  # noqa: F401
                  mask_from_keep, n_eff, num_angles, schedule, u_apply, u_backward, u_build_U, u_supported, version,
                  workspace, workspace_bytes)
from ._lib import (GivensError, OP_APPLY, OP_BACKWARD, OP_BUILD_U, OP_U_APPLY, OP_U_BACKWARD,  # noqa: F401
                   OP_U_BUILD_U)
