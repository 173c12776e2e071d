"""Host long-precision side (the paper's "MP" role): correctly rounded
binary floating point at a fixed precision, on mpmath's raw mpf tuples.

The reference's long side is its own BigFloat (bigfloat.py); every scalar
operation there rounds once, to nearest-even, at the context precision, as
mpmath's mpf_add/mpf_sub/mpf_mul/mpf_div/mpf_sqrt do with rnd='n' (SURVEY
finding 10).  The loops below are written in the reference's operation
order (linalg.py:545-574 scalar mat_vec, 680-700 norms, 740-770
conversions; refine.py:163-194) so residual histories match bit for bit.

This module is the host-side long-precision engine the north star keeps on
the CPU; the short-precision factor/solve never runs here.
"""

import math
import re

from mpmath import libmp as L

from .errors import (ArithmeticOverflowError, DimensionError,
                     DivideByZeroError, DomainError, ParseError,
                     SingularMatrixError)

RND = "n"
FZERO = L.fzero

__all__ = ["BigFloat", "LF", "PrecisionContext", "BfDomain", "parse_decimal",
           "format_decimal", "convert_vector", "convert_matrix"]


class PrecisionContext:
    """Target significand width in bits (bigfloat.py:52-71)."""

    __slots__ = ("p",)

    def __init__(self, p):
        p = int(p)
        if p < 2:
            raise DomainError("precision must be at least 2 bits, got %d" % p)
        self.p = p

    def __repr__(self):
        return "PrecisionContext(%d)" % self.p

    def __eq__(self, other):
        return isinstance(other, PrecisionContext) and other.p == self.p

    def __hash__(self):
        return hash(("PrecisionContext", self.p))


class BigFloat:
    """One long-precision value (the reference's BigFloat, bigfloat.py:73-158):
    value = sign * man * 2**exp, prec = the precision it was last rounded to
    (bookkeeping only: comparisons and hashing ignore it).

    Stored as mpmath's raw mpf tuple ``v`` (odd mantissa; the reference's
    _strip form), so every operation of this module is one correctly
    rounded mpmath call.  ``BigFloat(sign, man, exp, prec)`` is the
    reference constructor; the module's own results are built through
    ``LF(v, prec)`` (a subclass: every LF is a BigFloat).
    """

    __slots__ = ("v", "prec")

    def __init__(self, sign, man, exp, prec):
        sign, man, exp = int(sign), int(man), int(exp)
        if sign == 0 or man == 0:
            self.v = FZERO
        else:
            if man < 0:
                man, sign = -man, -sign
            tz = (man & -man).bit_length() - 1
            man, exp = man >> tz, exp + tz
            self.v = (1 if sign < 0 else 0, man, exp, man.bit_length())
        self.prec = int(prec)

    def to_float(self):
        """Nearest binary64 (bf_to_binary64, bigfloat.py:375-387)."""
        r = L.to_float(self.v, rnd=RND)
        if math.isinf(r):
            raise ArithmeticOverflowError("value does not fit in binary64")
        return r

    def to_components(self, k):
        """Peel k rounded binary64 heads (bf_to_multicomp, 419-432)."""
        comps = []
        r = self.v
        for _ in range(k):
            c = L.to_float(r, rnd=RND)
            if math.isinf(c):
                raise ArithmeticOverflowError("value does not fit in binary64")
            comps.append(c)
            if c != 0.0:
                r = L.mpf_sub(r, L.from_float(c))
        return tuple(comps)

    def round(self, p):
        if self.v == FZERO:
            return LF(FZERO, p)
        if self.v[3] <= p:
            return self if self.prec == p else LF(self.v, p)
        return LF(L.mpf_pos(self.v, p, RND), p)

    # the reference's attribute surface (sign in {-1, 0, 1}, man >= 0)
    @property
    def sign(self):
        if not self.v[1]:
            return 0
        return -1 if self.v[0] else 1

    @property
    def man(self):
        return int(self.v[1])

    @property
    def exp(self):
        return int(self.v[2]) if self.v[1] else 0

    def is_zero(self):
        return not self.v[1]

    # operators round at the larger operand precision (BigFloat._ctx)
    def _p(self, other):
        return max(self.prec, other.prec)

    def __add__(self, other):
        if not isinstance(other, BigFloat):
            return NotImplemented
        return lf_add(self, other, self._p(other))

    def __sub__(self, other):
        if not isinstance(other, BigFloat):
            return NotImplemented
        return lf_sub(self, other, self._p(other))

    def __mul__(self, other):
        if not isinstance(other, BigFloat):
            return NotImplemented
        return lf_mul(self, other, self._p(other))

    def __truediv__(self, other):
        if not isinstance(other, BigFloat):
            return NotImplemented
        return lf_div(self, other, self._p(other))

    def __neg__(self):
        return lf_neg(self)

    def __abs__(self):
        return lf_abs(self)

    def __float__(self):
        return self.to_float()

    def __eq__(self, other):
        if not isinstance(other, BigFloat):
            return NotImplemented
        return L.mpf_cmp(self.v, other.v) == 0

    def __ne__(self, other):
        eq = self.__eq__(other)
        return eq if eq is NotImplemented else not eq

    def __lt__(self, other):
        if not isinstance(other, BigFloat):
            return NotImplemented
        return L.mpf_cmp(self.v, other.v) < 0

    def __le__(self, other):
        if not isinstance(other, BigFloat):
            return NotImplemented
        return L.mpf_cmp(self.v, other.v) <= 0

    def __gt__(self, other):
        if not isinstance(other, BigFloat):
            return NotImplemented
        return L.mpf_cmp(self.v, other.v) > 0

    def __ge__(self, other):
        if not isinstance(other, BigFloat):
            return NotImplemented
        return L.mpf_cmp(self.v, other.v) >= 0

    def __hash__(self):
        return hash(self.v)

    def __repr__(self):
        return "BigFloat(%s, prec=%d)" % (format_hex(self), self.prec)


class LF(BigFloat):
    """A BigFloat built from a raw mpf tuple (this module's internal
    constructor): ``LF(v, prec)``."""

    __slots__ = ()

    def __init__(self, v, prec):
        self.v = v
        self.prec = prec

    # -- conversions -------------------------------------------------------
    @classmethod
    def from_int(cls, n, prec=None):
        v = L.from_int(int(n))
        if prec is None:
            return cls(v, max(v[3], 2))
        return cls(L.normalize(v[0], v[1], v[2], v[3], prec, RND)
                   if v[1] else FZERO, prec)

    @classmethod
    def from_float(cls, x):
        x = float(x)
        if not math.isfinite(x):
            raise DomainError("cannot convert non-finite value %r" % (x,))
        return cls(L.from_float(x), 53)

    @classmethod
    def from_components(cls, comps, prec=None):
        """Exact sum of binary64 components, rounded once to prec
        (bf_from_multicomp, bigfloat.py:404-416)."""
        acc = FZERO
        for c in comps:
            if c != 0.0:
                acc = L.mpf_add(acc, L.from_float(float(c)))
        if prec is None:
            return cls(acc, max(acc[3], 53))
        return cls(L.mpf_pos(acc, prec, RND), prec)


def lf_add(a, b, p):
    return LF(L.mpf_add(a.v, b.v, p, RND), p)


def lf_sub(a, b, p):
    return LF(L.mpf_sub(a.v, b.v, p, RND), p)


def lf_mul(a, b, p):
    return LF(L.mpf_mul(a.v, b.v, p, RND), p)


def lf_div(a, b, p):
    if not b.v[1]:
        raise DivideByZeroError("division by zero")
    return LF(L.mpf_div(a.v, b.v, p, RND), p)


def lf_sqrt(a, p):
    if a.sign < 0:
        raise DomainError("square root of a negative value")
    if not a.v[1]:
        return LF(FZERO, p)
    return LF(L.mpf_sqrt(a.v, p, RND), p)


def lf_neg(a):
    """Exact negation (bf_neg keeps the precision tag)."""
    return LF(L.mpf_neg(a.v), a.prec)


def lf_abs(a):
    return LF(L.mpf_abs(a.v), a.prec)


def lf_cmp(a, b):
    return L.mpf_cmp(a.v, b.v)


# ---------------------------------------------------------------- text ----
_DEC_RE = re.compile(
    r"^([+-]?)(?:(\d+)(?:\.(\d*))?|\.(\d+))(?:[eE]([+-]?\d+))?$")
_HEX_RE = re.compile(
    r"^([+-]?)0[xX]([0-9a-fA-F]+)(?:\.([0-9a-fA-F]*))?[pP]([+-]?\d+)$")


def parse_decimal(text, prec):
    """Correctly rounded decimal literal (bf_parse_decimal, 445-466)."""
    m = _DEC_RE.match(text.strip())
    if not m:
        raise ParseError("malformed decimal literal %r" % (text,))
    sign_s, int_s, frac_s, bare, exp_s = m.groups()
    if bare is not None:
        int_s, frac_s = "", bare
    frac_s = frac_s or ""
    digits = (int_s or "") + frac_s
    d = int(digits) if digits else 0
    if d == 0:
        return LF(FZERO, prec)
    if sign_s == "-":
        d = -d
    e10 = (int(exp_s) if exp_s else 0) - len(frac_s)
    if e10 >= 0:
        return LF(L.from_int(d * 10 ** e10, prec, RND), prec)
    return LF(L.from_rational(d, 10 ** -e10, prec, RND), prec)


def parse_hex(text, prec=None):
    """Exact hex-float literal (bf_parse_hex, 538-555)."""
    m = _HEX_RE.match(text.strip())
    if not m:
        raise ParseError("malformed hex literal %r" % (text,))
    sign_s, int_s, frac_s, exp_s = m.groups()
    frac_s = frac_s or ""
    man = int(int_s + frac_s, 16)
    if man == 0:
        return LF(FZERO, prec or 2)
    if sign_s == "-":
        man = -man
    v = L.from_man_exp(man, int(exp_s) - 4 * len(frac_s))
    if prec is None:
        return LF(v, max(v[3], 2))
    return LF(L.mpf_pos(v, prec, RND), prec)


def format_hex(a):
    """Canonical exact hex form (bf_format_hex, bigfloat.py:520-535)."""
    if not a.v[1]:
        return "0x0.0p+0"
    neg, man, exp, bc = a.v
    nbits = bc - 1
    e = exp + nbits
    sign_s = "-" if neg else ""
    if nbits == 0:
        return "%s0x1p%+d" % (sign_s, e)
    pad = (-nbits) % 4
    frac = (man - (1 << nbits)) << pad
    width = (nbits + pad) // 4
    return "%s0x1.%sp%+d" % (sign_s, format(frac, "0%dx" % width), e)


def _rn_int(num, den):
    q, r = divmod(num, den)
    r2 = r << 1
    if r2 > den or (r2 == den and q & 1):
        q += 1
    return q


def format_decimal(a, digits=None):
    """Scientific decimal with `digits` significant figures, correctly
    rounded (the algorithm of bf_format_decimal, bigfloat.py:483-509)."""
    if digits is None:
        digits = int(math.ceil(a.prec * 0.3010299956639812)) + 2
    if digits < 1:
        raise DomainError("need at least one digit")
    if not a.v[1]:
        frac = "0" * (digits - 1)
        return "0." + frac + "e+0" if frac else "0.e+0"
    neg, man, exp, bc = a.v
    top = exp + bc
    d_exp = math.floor(top * 0.30102999566398114)
    scaled = 0
    for _ in range(4):
        t = digits - 1 - d_exp
        num, den = man, 1
        if t >= 0:
            num *= 10 ** t
        else:
            den = 10 ** -t
        if exp >= 0:
            num <<= exp
        else:
            den <<= -exp
        scaled = _rn_int(num, den)
        lo, hi = 10 ** (digits - 1), 10 ** digits
        if scaled >= hi:
            d_exp += 1
        elif scaled < lo:
            d_exp -= 1
        else:
            break
    s = str(scaled)
    sign_s = "-" if neg else ""
    frac = s[1:]
    return ("%s%s.%se%+d" % (sign_s, s[0], frac, d_exp) if frac
            else "%s%s.e%+d" % (sign_s, s[0], d_exp))


# -------------------------------------------------------------- domain ----
class BfDomain:
    """Scalar domain of long values at a fixed precision (linalg.py:148-214)."""

    kind = "bf"

    def __init__(self, bits):
        self.ctx = bits if isinstance(bits, PrecisionContext) \
            else PrecisionContext(bits)
        self.p = self.ctx.p
        self.name = "bf%d" % self.p
        self.one = LF.from_int(1, self.p)
        self.zero = LF(FZERO, self.p)

    def __repr__(self):
        return "BfDomain(%d)" % self.p

    def compatible(self, other):
        return isinstance(other, BfDomain) and other.p == self.p

    def add(self, a, b):
        return lf_add(a, b, self.p)

    def sub(self, a, b):
        return lf_sub(a, b, self.p)

    def mul(self, a, b):
        return lf_mul(a, b, self.p)

    def div(self, a, b):
        return lf_div(a, b, self.p)

    def sqrt(self, a):
        return lf_sqrt(a, self.p)

    def neg(self, a):
        return lf_neg(a)

    def is_zero(self, a):
        return a.is_zero()

    def pivot_mag(self, a):
        return lf_abs(a)

    def coerce(self, value):
        from .mcfloat import MultiComp
        if isinstance(value, LF):
            return value.round(self.p)
        if isinstance(value, MultiComp):
            return LF.from_components(value.components, self.p)
        if isinstance(value, bool):
            raise DomainError("cannot store %r in %r" % (value, self))
        if isinstance(value, int):
            return LF.from_int(value, self.p)
        if isinstance(value, float):
            return LF.from_float(value).round(self.p)
        if isinstance(value, str):
            return parse_decimal(value, self.p)
        raise DomainError("cannot store %r in %r" % (value, self))

    def wrap(self, raw):
        return raw

    def to_long(self, raw, prec=None):
        return raw if prec is None else raw.round(prec)

    def from_long(self, value):
        return value.round(self.p)


def _transfer_prec(src, dst):
    # linalg.py:743-747
    bits = 0
    for d in (src, dst):
        bits = max(bits, d.p if d.kind == "bf" else 53 * d.k + 64)
    return bits + 8


def convert_vector(v, domain):
    """Re-represent a vector in another domain (linalg.py:751-758)."""
    from .linalg import Vector
    p = _transfer_prec(v.domain, domain)
    out = Vector.zeros(domain, v.n)
    if v.domain.kind == "mc" and domain.kind == "bf":
        cols = v.data.T.tolist()
        out.data = [LF.from_components(c, p).round(domain.p) for c in cols]
    elif v.domain.kind == "bf" and domain.kind == "mc":
        import numpy as np
        comps = [s.round(p).to_components(domain.k) for s in v.data]
        out.data = np.ascontiguousarray(np.array(comps, dtype=np.float64).T)
    elif v.domain.kind == "bf":
        out.data = [s.round(p).round(domain.p) for s in v.data]
    else:
        cols = v.data.T.tolist()
        import numpy as np
        comps = [LF.from_components(c, p).to_components(domain.k)
                 for c in cols]
        out.data = np.ascontiguousarray(np.array(comps, dtype=np.float64).T)
    return out


def convert_matrix(A, domain):
    """Re-represent a matrix in another domain (linalg.py:761-770)."""
    import numpy as np
    from .linalg import DenseMatrix
    p = _transfer_prec(A.domain, domain)
    out = DenseMatrix.zeros(domain, A.rows, A.cols)
    if A.domain.kind == "mc":
        elems = A.data.transpose(1, 2, 0).tolist()
        if domain.kind == "bf":
            out.data = [[LF.from_components(e, p).round(domain.p)
                         for e in row] for row in elems]
        else:
            vals = [[LF.from_components(e, p).to_components(domain.k)
                     for e in row] for row in elems]
            out.data = np.ascontiguousarray(
                np.moveaxis(np.array(vals, dtype=np.float64), -1, 0))
    else:
        if domain.kind == "bf":
            out.data = [[s.round(p).round(domain.p) for s in row]
                        for row in A.data]
        else:
            vals = [[s.round(p).to_components(domain.k) for s in row]
                    for row in A.data]
            out.data = np.ascontiguousarray(
                np.moveaxis(np.array(vals, dtype=np.float64), -1, 0))
    return out


# -------------------------------------------------------- scalar loops ----
def mat_vec_long(A, x):
    """Scalar-path mat_vec (linalg.py:566-574): acc = add(acc, mul(a, x))."""
    from .linalg import Vector
    dom = A.domain
    p = dom.p
    xs = x.data
    vals = []
    add, mul = L.mpf_add, L.mpf_mul
    xv = [s.v for s in xs]
    for row in A.data:
        acc = FZERO
        for a, b in zip(row, xv):
            acc = add(acc, mul(a.v, b, p, RND), p, RND)
        vals.append(LF(acc, p))
    out = Vector.zeros(dom, A.rows)
    out.data = vals
    return out


def mat_mul_long(A, B):
    from .linalg import DenseMatrix
    dom = A.domain
    p = dom.p
    vals = [[dom.zero] * B.cols for _ in range(A.rows)]
    for i in range(A.rows):
        for j in range(B.cols):
            acc = FZERO
            for q in range(A.cols):
                acc = L.mpf_add(acc, L.mpf_mul(A.data[i][q].v,
                                               B.data[q][j].v, p, RND), p, RND)
            vals[i][j] = LF(acc, p)
    out = DenseMatrix.zeros(dom, A.rows, B.cols)
    out.data = vals
    return out


def lu_factor_long(A):
    """_lu_rows (linalg.py:393-419) over long values."""
    dom = A.domain
    rows = A.data
    n = len(rows)
    swaps = []
    for j in range(n):
        best = j
        bestmag = dom.pivot_mag(rows[j][j])
        for i in range(j + 1, n):
            m = dom.pivot_mag(rows[i][j])
            if lf_cmp(m, bestmag) > 0:
                best, bestmag = i, m
        if best != j:
            rows[j], rows[best] = rows[best], rows[j]
        swaps.append(best)
        piv = rows[j][j]
        if dom.is_zero(piv):
            raise SingularMatrixError(
                "no nonzero pivot at elimination step %d" % j, step=j)
        recip = dom.div(dom.one, piv)
        rowj = rows[j]
        for i in range(j + 1, n):
            rowi = rows[i]
            m = dom.mul(rowi[j], recip)
            rowi[j] = m
            negm = dom.neg(m)
            for c in range(j + 1, n):
                rowi[c] = dom.add(rowi[c], dom.mul(negm, rowj[c]))
    return swaps


def lu_solve_long(lu, piv, b):
    """_solve_rows (linalg.py:476-493) over long values."""
    dom = lu.domain
    rows = lu.data
    x = list(b.data)
    n = len(rows)
    for j, r in enumerate(piv.swaps):
        if r != j:
            x[j], x[r] = x[r], x[j]
    for j in range(n):
        xj = x[j]
        for i in range(j + 1, n):
            x[i] = dom.add(x[i], dom.mul(dom.neg(rows[i][j]), xj))
    for j in range(n - 1, -1, -1):
        xj = dom.div(x[j], rows[j][j])
        x[j] = xj
        negxj = dom.neg(xj)
        for i in range(j):
            x[i] = dom.add(x[i], dom.mul(rows[i][j], negxj))
    out = b.copy()
    out.data = x
    return out


def _norm_acc(values, p):
    acc = FZERO
    for s in values:
        acc = L.mpf_add(acc, L.mpf_mul(s.v, s.v, p, RND), p, RND)
    return LF(acc, p)


def vec_norm2_any(v):
    """vec_norm2 (linalg.py:680-689) in the vector's own domain."""
    dom = v.domain
    if dom.kind == "bf":
        return lf_sqrt(_norm_acc(v.data, dom.p), dom.p)
    raise DomainError("short-precision norms are not on the device path")


def mat_norm_fro_any(A):
    """mat_norm_fro (linalg.py:692-700), row-major accumulation."""
    dom = A.domain
    if dom.kind == "bf":
        acc = FZERO
        p = dom.p
        for row in A.data:
            for s in row:
                acc = L.mpf_add(acc, L.mpf_mul(s.v, s.v, p, RND), p, RND)
        return lf_sqrt(LF(acc, p), p)
    raise DomainError("short-precision norms are not on the device path")


def max_rel_err(x, ref, ctx=None):
    """Worst per-entry relative error at 240 bits (linalg.py:706-727)."""
    if x.n != ref.n:
        raise DimensionError("size mismatch: %d vs %d" % (x.n, ref.n))
    p = ctx.p if ctx is not None else 240

    def at(v, i):
        if v.domain.kind == "bf":
            return v.data[i].round(p)
        return LF.from_components(tuple(v.data[:, i].tolist()), p)

    best = None
    for i in range(x.n):
        r = at(ref, i)
        xi = at(x, i)
        if r.is_zero():
            q = lf_abs(xi)
        else:
            q = lf_div(lf_abs(lf_sub(xi, r, p)), lf_abs(r), p)
        if best is None or lf_cmp(q, best) > 0:
            best = q
    return best.to_float()
