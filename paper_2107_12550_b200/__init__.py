"""B200-native DD/TD/QD dense direct solver — drop-in for the reference's
Python API (/root/reference/pkg/src/mpcore/__init__.py:62-78) on the hot
path: multi-component containers, LU with partial pivoting, triangular
solves, GEMM/GEMV/batch kernels (all sm_100a CUDA in libmpcore.so, called
through ctypes) and the mixed-precision iterative-refinement driver (long
residual on the host, short solves on the GPU).

    import paper_2107_12550_b200 as mpcore
"""

__version__ = "0.1.0"

from .errors import (  # noqa: F401
    ArithmeticOverflowError, DimensionError, DivideByZeroError, DomainError,
    GenerationError, MpcoreError, ParseError, SingularMatrixError)
from .linalg import (  # noqa: F401
    BfDomain, DenseMatrix, DeviceMatrix, DeviceVector, McDomain, PivotRecord,
    PrecisionTag, Vector, axpy_batch, convert_matrix, convert_vector,
    elementwise_add_batch, elementwise_div_batch, elementwise_mul_batch,
    lu_factor_pp, lu_solve, mat_mul_blocked, mat_norm_fro, mat_vec,
    max_rel_err, vec_norm2)
from .bigfloat import (  # noqa: F401
    BigFloat, PrecisionContext, bf_from_multicomp, bf_parse_decimal,
    bf_to_multicomp)
from .longfloat import LF  # noqa: F401
from .mcfloat import (  # noqa: F401
    MultiComp, mc_add, mc_div, mc_mul, mc_sqrt, mc_sub)
from .refine import (  # noqa: F401
    RefineConfig, RefineReport, check_stop, iterative_refinement,
    iterative_refinement_td_mp)
from .paper import (  # noqa: F401
    DDLUdecompPM, TDLUdecompPM, QDLUdecompPM, SolveDDLSPM, SolveTDLSPM,
    SolveQDLSPM)


def simd_enabled():
    """Reads MPCORE_SIMD like the reference (simd.py:31-33); there is a
    single (device) execution path either way."""
    from . import _native
    return bool(_native.lib().mpcore_simd_enabled())


__all__ = [
    "__version__",
    "MpcoreError", "ArithmeticOverflowError", "DivideByZeroError",
    "DomainError", "SingularMatrixError", "DimensionError", "ParseError",
    "GenerationError",
    "MultiComp", "mc_add", "mc_sub", "mc_mul", "mc_div", "mc_sqrt",
    "BigFloat", "PrecisionContext", "bf_parse_decimal",
    "bf_to_multicomp", "bf_from_multicomp", "LF",
    "McDomain", "BfDomain", "Vector", "DenseMatrix", "PivotRecord",
    "lu_factor_pp", "lu_solve", "mat_vec", "mat_mul_blocked",
    "vec_norm2", "mat_norm_fro", "max_rel_err",
    "convert_vector", "convert_matrix",
    "RefineConfig", "RefineReport", "check_stop", "iterative_refinement",
    "simd_enabled",
    "DDLUdecompPM", "TDLUdecompPM", "QDLUdecompPM",
    "SolveDDLSPM", "SolveTDLSPM", "SolveQDLSPM",
]
