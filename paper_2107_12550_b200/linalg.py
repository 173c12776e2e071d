"""Dense linear algebra over DD/TD/QD, executed by libmpcore on the GPU.

Drop-in for the short-precision surface of the reference's linalg module
(/root/reference/pkg/src/mpcore/linalg.py): same containers (planar numpy
``.data`` of shape (k, ...), simd.py:36-48), same entry points and errors:

  lu_factor_pp    linalg.py:452-469   in place, returns PivotRecord
  lu_solve        linalg.py:524-538   new Vector, b untouched
  mat_vec         linalg.py:545-574
  mat_mul_blocked linalg.py:577-617   (block only tiled the reference's
                                       scalar loop; accepted and ignored)
  axpy_batch / elementwise_add_batch / elementwise_mul_batch  (624-673)

Every McDomain operation runs in sm_100a kernels (libmpcore.so) and is
bitwise identical to the reference's lane path.  ``simd`` is accepted for
signature compatibility; there is exactly one execution path.  BigFloat
(long-precision) containers live in ``longfloat`` and stay on the host.
"""

import ctypes
import math

import numpy as np

from . import _native as nat
from .errors import DimensionError, DomainError, SingularMatrixError
from .longfloat import BfDomain, LF

__all__ = [
    "McDomain", "BfDomain", "Vector", "DenseMatrix", "PivotRecord",
    "lu_factor_pp", "lu_solve", "mat_vec", "mat_mul_blocked", "axpy_batch",
    "elementwise_add_batch", "elementwise_mul_batch", "vec_norm2",
    "mat_norm_fro", "max_rel_err", "convert_vector", "convert_matrix",
    "DeviceMatrix", "DeviceVector",
]

_TAGS = {"dd": 2, "td": 3, "qd": 4}
_NAMES = {2: "dd", 3: "td", 4: "qd"}


class PrecisionTag:
    """DD (k=2), TD (k=3), QD (k=4)  (mcfloat.py:361-401)."""

    __slots__ = ("name", "k", "bits", "rel_bound")

    def __init__(self, name, k, rel_exp):
        self.name, self.k, self.bits = name, k, 53 * k
        self.rel_bound = 2.0 ** rel_exp

    def __repr__(self):
        return "PrecisionTag(%s)" % self.name

    @classmethod
    def from_name(cls, name):
        try:
            return _REGISTRY[name.lower()]
        except (KeyError, AttributeError):
            raise DomainError("unknown precision tag %r" % (name,)) from None

    @classmethod
    def from_k(cls, k):
        for t in _REGISTRY.values():
            if t.k == k:
                return t
        raise DomainError("unknown component count %r" % (k,))


DD = PrecisionTag("dd", 2, -99)
TD = PrecisionTag("td", 3, -152)
QD = PrecisionTag("qd", 4, -205)
_REGISTRY = {"dd": DD, "td": TD, "qd": QD}


class McDomain:
    """Scalar domain of k-component values (linalg.py:74-145)."""

    kind = "mc"

    def __init__(self, tag):
        if isinstance(tag, str):
            tag = PrecisionTag.from_name(tag)
        self.tag = tag
        self.k = tag.k
        self.name = tag.name
        self.one = (1.0,) + (0.0,) * (tag.k - 1)
        self.zero = (0.0,) * tag.k

    def __repr__(self):
        return "McDomain(%s)" % self.name

    def compatible(self, other):
        return isinstance(other, McDomain) and other.k == self.k

    def pivot_mag(self, a):
        # linalg.py:115-119: magnitude of the leading component
        return abs(a[0])

    def is_zero(self, a):
        return a[0] == 0.0

    def coerce(self, value):
        from .mcfloat import MultiComp
        if isinstance(value, MultiComp):
            if value.k != self.k:
                raise DomainError("expected %d components, got %d"
                                  % (self.k, value.k))
            return value.components
        if isinstance(value, LF):
            return value.to_components(self.k)
        if isinstance(value, (int, float)) and not isinstance(value, bool):
            x = float(value)
            if not math.isfinite(x):
                raise DomainError("non-finite element %r" % (x,))
            return (x,) + (0.0,) * (self.k - 1)
        if isinstance(value, tuple) and len(value) == self.k:
            return tuple(float(c) for c in value)
        raise DomainError("cannot store %r in %r" % (value, self))

    def wrap(self, raw):
        from .mcfloat import MultiComp
        return MultiComp(tuple(raw), validate=False)

    def to_long(self, raw, prec=None):
        return LF.from_components(raw, prec)

    def from_long(self, value):
        return value.to_components(self.k)


# containers at least this large keep their planes page-locked (when the
# device is present), so lu_factor_pp / lu_solve / mat_mul_blocked move
# them at DMA speed instead of through pageable staging
PINNED_MIN_BYTES = 1 << 20


def _planes_zeros(k, shape):
    if isinstance(shape, int):
        shape = (shape,)
    shape = (k,) + tuple(shape)
    if 8 * int(np.prod(shape)) >= PINNED_MIN_BYTES and nat.device_available():
        return nat.pinned_zeros(shape)
    return np.zeros(shape, dtype=np.float64)


def _planes_copy(a):
    out = _planes_zeros(a.shape[0], a.shape[1:])
    out[...] = a
    return out


class Vector:
    """Dense column vector (linalg.py:221-281)."""

    __slots__ = ("domain", "n", "data")

    def __init__(self, domain, n, data):
        self.domain, self.n, self.data = domain, n, data

    @classmethod
    def zeros(cls, domain, n):
        if n < 1:
            raise DimensionError("vector length must be positive")
        if domain.kind == "mc":
            return cls(domain, n, _planes_zeros(domain.k, n))
        return cls(domain, n, [domain.zero] * n)

    @classmethod
    def from_values(cls, domain, values):
        values = list(values)
        v = cls.zeros(domain, len(values))
        for i, val in enumerate(values):
            v.set(i, val)
        return v

    def get(self, i):
        if self.domain.kind == "mc":
            return self.domain.wrap(tuple(self.data[:, i].tolist()))
        return self.data[i]

    def set(self, i, value):
        raw = self.domain.coerce(value)
        if self.domain.kind == "mc":
            self.data[:, i] = raw
        else:
            self.data[i] = raw

    def copy(self):
        if self.domain.kind == "mc":
            return Vector(self.domain, self.n, _planes_copy(self.data))
        return Vector(self.domain, self.n, list(self.data))

    def to_list(self):
        return [self.get(i) for i in range(self.n)]

    def _extract(self):
        if self.domain.kind == "mc":
            return [tuple(col) for col in zip(*self.data.tolist())]
        return list(self.data)


class DenseMatrix:
    """Dense row-major matrix (linalg.py:284-337)."""

    __slots__ = ("domain", "rows", "cols", "data")

    def __init__(self, domain, rows, cols, data):
        self.domain, self.rows, self.cols, self.data = domain, rows, cols, data

    @classmethod
    def zeros(cls, domain, rows, cols):
        if rows < 1 or cols < 1:
            raise DimensionError("matrix dimensions must be positive")
        if domain.kind == "mc":
            return cls(domain, rows, cols,
                       _planes_zeros(domain.k, (rows, cols)))
        return cls(domain, rows, cols,
                   [[domain.zero] * cols for _ in range(rows)])

    @classmethod
    def from_rows(cls, domain, rows):
        rows = [list(r) for r in rows]
        if not rows or any(len(r) != len(rows[0]) for r in rows):
            raise DimensionError("ragged or empty row data")
        m = cls.zeros(domain, len(rows), len(rows[0]))
        for i, r in enumerate(rows):
            for j, val in enumerate(r):
                m.set(i, j, val)
        return m

    def get(self, i, j):
        if self.domain.kind == "mc":
            return self.domain.wrap(tuple(self.data[:, i, j].tolist()))
        return self.data[i][j]

    def set(self, i, j, value):
        raw = self.domain.coerce(value)
        if self.domain.kind == "mc":
            self.data[:, i, j] = raw
        else:
            self.data[i][j] = raw

    def copy(self):
        if self.domain.kind == "mc":
            return DenseMatrix(self.domain, self.rows, self.cols,
                               _planes_copy(self.data))
        return DenseMatrix(self.domain, self.rows, self.cols,
                           [list(r) for r in self.data])

    def _extract_rows(self):
        if self.domain.kind == "mc":
            return [[tuple(e) for e in row]
                    for row in self.data.transpose(1, 2, 0).tolist()]
        return self.data


def _require_same_domain(*objs):
    d = objs[0].domain
    for o in objs[1:]:
        if not d.compatible(o.domain):
            raise DomainError("domain mismatch: %r vs %r" % (d, o.domain))
    return d


class PivotRecord:
    """Row exchange sequence (linalg.py:348-386): swaps[j] = r >= j."""

    __slots__ = ("swaps",)

    def __init__(self, swaps):
        self.swaps = [int(s) for s in swaps]
        for j, r in enumerate(self.swaps):
            if r < j or r >= len(self.swaps):
                raise DomainError("invalid swap %d at step %d" % (r, j))

    @property
    def n(self):
        return len(self.swaps)

    def permutation(self):
        order = list(range(self.n))
        for j, r in enumerate(self.swaps):
            if r != j:
                order[j], order[r] = order[r], order[j]
        return order

    def apply(self, v):
        out = v.copy()
        if v.domain.kind == "mc":
            for j, r in enumerate(self.swaps):
                if r != j:
                    out.data[:, [j, r]] = out.data[:, [r, j]]
        else:
            for j, r in enumerate(self.swaps):
                if r != j:
                    out.data[j], out.data[r] = out.data[r], out.data[j]
        return out


# ---------------------------------------------------------------------------
# device-resident objects (handle level)
# ---------------------------------------------------------------------------

class DeviceMatrix:
    """A k-component matrix resident in HBM (one libmpcore handle)."""

    def __init__(self, k, rows, cols):
        self.k, self.rows, self.cols = k, rows, cols
        self._h = nat.Handle(nat.new_matrix(k, rows, cols))

    @property
    def handle(self):
        return self._h.h

    @classmethod
    def from_planes(cls, planes):
        planes = np.ascontiguousarray(planes, dtype=np.float64)
        k, rows, cols = planes.shape
        m = cls(k, rows, cols)
        nat.set_planes(m.handle, planes)
        return m

    def upload(self, planes):
        nat.set_planes(self.handle, planes)

    def download(self, out=None):
        return nat.get_planes(self.handle, (self.k, self.rows, self.cols), out)

    def generate(self, slot, system_n, seed):
        nat.check(nat.lib().mpcore_generate(self.handle, slot, system_n,
                                            seed), "generate")

    def copy_from(self, other):
        nat.check(nat.lib().mpcore_copy(other.handle, self.handle), "copy")

    def device_ptr(self):
        """Address of component plane 0, element 0 (planar, row-major)."""
        p = ctypes.c_uint64()
        nat.check(nat.lib().mpcore_object_device_ptr(self.handle,
                                                     ctypes.byref(p)), "ptr")
        return p.value

    def lu_factor(self, nb=0):
        """In-place factorisation -> (PivotHandle)."""
        st, piv, step = nat.lu_factor(self.handle, nb)
        if st == nat.SINGULAR:
            raise SingularMatrixError(
                "no nonzero pivot at elimination step %d" % step, step=step)
        nat.check(st, "lu_factor")
        return PivotHandle(piv, self.rows)


class DeviceVector:
    def __init__(self, k, n):
        self.k, self.n = k, n
        self._h = nat.Handle(nat.new_vector(k, n))

    @property
    def handle(self):
        return self._h.h

    @classmethod
    def from_planes(cls, planes):
        planes = np.ascontiguousarray(planes, dtype=np.float64)
        v = cls(planes.shape[0], planes.shape[1])
        nat.set_planes(v.handle, planes)
        return v

    def upload(self, planes):
        nat.set_planes(self.handle, planes)

    def device_ptr(self):
        """Address of component plane 0, element 0 (planar)."""
        p = ctypes.c_uint64()
        nat.check(nat.lib().mpcore_object_device_ptr(self.handle,
                                                     ctypes.byref(p)), "ptr")
        return p.value

    def download(self, out=None):
        return nat.get_planes(self.handle, (self.k, self.n), out)

    def generate(self, slot, system_n, seed):
        nat.check(nat.lib().mpcore_generate(self.handle, slot, system_n,
                                            seed), "generate")


class PivotHandle:
    def __init__(self, h, n):
        self._h = nat.Handle(h)
        self.n = n

    @property
    def handle(self):
        return self._h.h

    @classmethod
    def from_swaps(cls, swaps):
        return cls(nat.pivot_new(swaps), len(swaps))

    def swaps(self):
        return nat.pivot_get(self.handle, self.n)


def device_solve(lu, piv, b, x):
    nat.check(nat.lib().mpcore_lu_solve(lu.handle, piv.handle, b.handle,
                                        x.handle), "lu_solve")


def device_solve_system(A, b, x, nb=0):
    """x = A^-1 b in one call (mpcore_solve_system): A is left holding its
    LU factors and the PivotHandle is returned, exactly as
    ``A.lu_factor(nb)`` + ``device_solve`` would leave them; b rides along
    the factorisation as an extra column (its forward substitution), so only
    the back substitution runs afterwards."""
    h = ctypes.c_uint64()
    step = ctypes.c_int32(-1)
    st = nat.lib().mpcore_solve_system(A.handle, b.handle, x.handle, int(nb),
                                       ctypes.byref(h), ctypes.byref(step))
    if st == nat.SINGULAR:
        raise SingularMatrixError(
            "no nonzero pivot at elimination step %d" % step.value,
            step=step.value)
    nat.check(st, "solve_system")
    return PivotHandle(h.value, A.rows)


# ---------------------------------------------------------------------------
# reference entry points
# ---------------------------------------------------------------------------

def _mc_only(dom, what):
    if dom.kind != "mc":
        raise DomainError("%s on %r runs on the host long-precision path; "
                          "use longfloat" % (what, dom))


def lu_factor_pp(A, simd=None, nb=0):
    """Factor A in place as P*A = L*U with partial pivoting (GPU).

    linalg.py:452-469: U on/above the diagonal, unit-lower multipliers
    below; returns the PivotRecord; raises SingularMatrixError(step).
    """
    if A.rows != A.cols:
        raise DimensionError("LU needs a square matrix, got %dx%d"
                             % (A.rows, A.cols))
    if A.domain.kind != "mc":
        from .longfloat import lu_factor_long
        return PivotRecord(lu_factor_long(A))
    dm = DeviceMatrix.from_planes(A.data)
    st, piv, step = nat.lu_factor(dm.handle, nb)
    if st == nat.SINGULAR:
        dm.download(A.data)
        raise SingularMatrixError(
            "no nonzero pivot at elimination step %d" % step, step=step)
    nat.check(st, "lu_factor")
    pv = PivotHandle(piv, A.rows)
    dm.download(A.data)
    return PivotRecord(pv.swaps())


def lu_solve(lu, piv, b, simd=None):
    """Solve P*A = L*U against one right-hand side (GPU); b unchanged."""
    dom = _require_same_domain(lu, b)
    if lu.rows != lu.cols:
        raise DimensionError("factored matrix must be square")
    if piv.n != lu.rows or b.n != lu.rows:
        raise DimensionError("size mismatch: lu %d, pivots %d, rhs %d"
                             % (lu.rows, piv.n, b.n))
    if dom.kind != "mc":
        from .longfloat import lu_solve_long
        return lu_solve_long(lu, piv, b)
    dm = DeviceMatrix.from_planes(lu.data)
    pv = PivotHandle.from_swaps(piv.swaps)
    bv = DeviceVector.from_planes(b.data)
    xv = DeviceVector(dom.k, b.n)
    device_solve(dm, pv, bv, xv)
    return Vector(dom, b.n, xv.download())


def mat_vec(A, x, simd=None):
    """A*x, accumulating left to right over columns (linalg.py:545-574)."""
    dom = _require_same_domain(A, x)
    if A.cols != x.n:
        raise DimensionError("mat_vec size mismatch: %dx%d times %d"
                             % (A.rows, A.cols, x.n))
    if dom.kind != "mc":
        from .longfloat import mat_vec_long
        return mat_vec_long(A, x)
    dm = DeviceMatrix.from_planes(A.data)
    xv = DeviceVector.from_planes(x.data)
    yv = DeviceVector(dom.k, A.rows)
    nat.check(nat.lib().mpcore_mat_vec(dm.handle, xv.handle, yv.handle),
              "mat_vec")
    return Vector(dom, A.rows, yv.download())


def mat_mul_blocked(A, B, simd=None, block=64):
    """A*B, inner index ascending globally (linalg.py:577-617)."""
    dom = _require_same_domain(A, B)
    if A.cols != B.rows:
        raise DimensionError("mat_mul size mismatch: %dx%d times %dx%d"
                             % (A.rows, A.cols, B.rows, B.cols))
    if dom.kind != "mc":
        from .longfloat import mat_mul_long
        return mat_mul_long(A, B)
    da = DeviceMatrix.from_planes(A.data)
    db = DeviceMatrix.from_planes(B.data)
    dc = DeviceMatrix(dom.k, A.rows, B.cols)
    nat.check(nat.lib().mpcore_mat_mul(da.handle, db.handle, dc.handle),
              "mat_mul")
    return DenseMatrix(dom, A.rows, B.cols, dc.download())


def axpy_batch(alpha, x, y, simd=None):
    """In-place y <- y + alpha*x (alpha applied from the right); returns y."""
    dom = _require_same_domain(x, y)
    if x.n != y.n:
        raise DimensionError("axpy size mismatch: %d vs %d" % (x.n, y.n))
    raw = dom.coerce(alpha)
    _mc_only(dom, "axpy_batch")
    xv = DeviceVector.from_planes(x.data)
    yv = DeviceVector.from_planes(y.data)
    al = np.ascontiguousarray(raw, dtype=np.float64)
    nat.check(nat.lib().mpcore_axpy(nat.dptr(al), dom.k, xv.handle,
                                    yv.handle), "axpy")
    yv.download(y.data)
    return y


def _elementwise(op, x, y):
    dom = _require_same_domain(x, y)
    if x.n != y.n:
        raise DimensionError("size mismatch: %d vs %d" % (x.n, y.n))
    _mc_only(dom, "elementwise")
    xv = DeviceVector.from_planes(x.data)
    yv = DeviceVector.from_planes(y.data)
    ov = DeviceVector(dom.k, x.n)
    nat.check(nat.lib().mpcore_elementwise(op, xv.handle, yv.handle,
                                           ov.handle), "elementwise")
    return Vector(dom, x.n, ov.download())


def elementwise_add_batch(x, y, simd=None):
    return _elementwise(0, x, y)


def elementwise_mul_batch(x, y, simd=None):
    return _elementwise(1, x, y)


def elementwise_div_batch(x, y):
    """Elementwise x / y via _div_t (mcfloat.py:304-318)."""
    return _elementwise(2, x, y)


# ---------------------------------------------------------------------------
# norms, errors, conversion (host long-precision side; linalg.py:680-770)
# ---------------------------------------------------------------------------

def vec_norm2(v):
    from .longfloat import vec_norm2_any
    return vec_norm2_any(v)


def mat_norm_fro(A):
    from .longfloat import mat_norm_fro_any
    return mat_norm_fro_any(A)


def max_rel_err(x, ref, ctx=None):
    from .longfloat import max_rel_err as _m
    return _m(x, ref, ctx)


def convert_vector(v, domain):
    from .longfloat import convert_vector as _c
    return _c(v, domain)


def convert_matrix(A, domain):
    from .longfloat import convert_matrix as _c
    return _c(A, domain)
