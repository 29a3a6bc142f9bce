"""B200-native DPV-SLAM hot path: patch-graph correlation lookup and the
Gauss-Newton / Levenberg-Marquardt bundle-adjustment step.

Drop-in for the reference ``patchslam`` modules on that path
(``geometry.reproject_grid``, ``graph.PatchGraph``, ``ba.*``,
``block_cholesky.block_cholesky``) plus the correlation op the reference
leaves out (``corr.corr``).  All numerics run in sm_100a kernels behind the
C-ABI in include/dpvslam_b200.h; see DESIGN.md.
"""

from . import ba, block_cholesky, corr, geometry, graph, synthetic  # noqa: F401
from .errors import NativeUnavailable, PatchSlamError, SingularSystem  # noqa: F401
from .geometry import Intrinsics, Patch, Pose  # noqa: F401
from .graph import LOOP, ODOMETRY, PatchGraph  # noqa: F401

__version__ = "0.1.0"
