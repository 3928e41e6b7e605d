"""mgtrace-b200: B200-native (sm_100a) hot path of the deflated Hutchinson
estimator for tr(A^-1) (arXiv:1909.12234), behind the reference's
(`mgtrace`) Python API.

Host side: Python/PyTorch (device memory, streams, torch.distributed).
Compute: hand-written CUDA kernels in `libmgtrace_b200.so` behind the C ABI
of `include/mgtrace_b200.h`.  There is no CPU fallback.
"""

from .lattice import (
    DENSE_GUARD,
    GeometryError,
    LatticeGeometry,
    SizeGuardError,
    WilsonOperator,
    build_lattice,
    build_wilson,
    gamma5_pattern,
)
from .gauge import GaugeField, gauge_from_array, generate_gauge
from .krylov import SolveConfig, SolveReport, TruncatedInverse, bicgstab_solve, truncated_inverse
from .probing import NoiseVector, ProbeGroup, ProbeSet, build_probe_set, make_noise
from .trace import TraceEstimate, hutchinson, jackknife, tsm_correction
from .mgsolve import Hierarchy, MultigridSolver, build_hierarchy, dump_hierarchy, load_hierarchy
from . import experiments

__version__ = "0.1.0"
