"""B200-native randomized skeletonization (sketched LUPP ID / CUR).

Drop-in for the hot path of the reference package `randskel`
(`/root/reference/pkg/src/randskel/__init__.py:9-86`): same public names,
signatures, result types, statuses and exceptions for the interpolative and
CUR entry points, with the arithmetic in hand-written sm_100a kernels
(librskel.so, C ABI in include/rskel.h).  There is no CPU fallback: without a
CUDA device or the built library the entry points raise DeviceError.
"""

from .errors import (
    DeviceError,
    DimensionError,
    NumericalError,
    RankDeficientError,
    SingularError,
)
from .sketching import (
    GaussianSketch,
    RngStream,
    SketchSpec,
    SparseSignSketch,
    SrttSketch,
    apply_sketch,
    make_gaussian,
    make_sketch,
    make_sparse_sign,
    make_srtt,
)
from .dense import (
    LUFactors,
    frobenius_norm,
    gemm,
    invert_permutation,
    lupp,
    lupp_blocked_step,
    row_permute,
    triangular_solve,
)
from .skeleton import (
    STATUS_ILL_CONDITIONED,
    STATUS_NOT_CONVERGED,
    STATUS_OK,
    STATUS_RANK_EXHAUSTED,
    ErrorTrace,
    SkeletonResult,
    TraceRecord,
    column_id,
    rand_lupp,
    rand_lupp_adaptive,
)
from .lu_state import (
    BlockedLUState,
    ResidualEstimates,
    adaptive_init,
    adaptive_step,
    draw_residual_sample,
    interpolation_matrix,
    residual_ur_estimates,
)
from .cur import CurFactors, cur_decompose, cur_decompose_adaptive, pinv_apply, two_sided_id
from .evaluate import row_id_error, stable_row_id_error
from ._ozaki import set_sketch_engine, sketch_engine
from .zoo import gen_chan, gen_fast_decay, gen_fast_decay_hadamard, gen_kahan, gen_nonneg_lowrank

__version__ = "0.1.0"
