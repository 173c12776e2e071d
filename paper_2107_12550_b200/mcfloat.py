"""MultiComp value type (mcfloat.py:404-551 of the reference) and the
scalar mc_* operations.

The arithmetic of a MultiComp is executed by the same sm_100a kernels as the
batched paths (libmpcore elementwise entry point with a batch of one), so a
scalar result is bitwise what the dense kernels compute; there is no host
implementation of the DD/TD/QD kernels in this package.
"""

import math

import numpy as np

from . import _native as nat
from .errors import ArithmeticOverflowError, DivideByZeroError, DomainError
from .linalg import PrecisionTag, DD, TD, QD  # noqa: F401

__all__ = ["MultiComp", "PrecisionTag", "mc_add", "mc_sub", "mc_mul",
           "mc_div", "mc_sqrt", "mc_neg", "mc_abs", "mc_cmp", "from_binary64",
           "to_binary64"]


def _validate_components(comps):
    # mcfloat.py:404-413
    if comps[0] == 0.0:
        for c in comps:
            if c != 0.0:
                raise DomainError("zero head with nonzero tail %r" % (comps,))
        return
    for i in range(len(comps) - 1):
        if abs(comps[i + 1]) > 0.5 * math.ulp(comps[i]):
            raise DomainError("components overlap at position %d: %r"
                              % (i, comps))


class MultiComp:
    """Ordered tuple of k binary64 components, canonical form."""

    __slots__ = ("components", "k")

    def __init__(self, components, validate=True):
        comps = tuple(float(c) for c in components)
        if len(comps) not in (2, 3, 4):
            raise DomainError("component count must be 2, 3 or 4")
        if validate:
            for c in comps:
                if not math.isfinite(c):
                    raise DomainError("non-finite component %r" % (c,))
            _validate_components(comps)
        object.__setattr__(self, "components", comps)
        object.__setattr__(self, "k", len(comps))

    def __setattr__(self, name, value):
        raise AttributeError("MultiComp is immutable")

    @property
    def tag(self):
        return PrecisionTag.from_k(self.k)

    def __repr__(self):
        return "MultiComp(%s)" % ", ".join(repr(c) for c in self.components)

    def __float__(self):
        return self.components[0]

    def _coerce(self, other):
        if isinstance(other, MultiComp):
            if other.k != self.k:
                raise DomainError("mixed component widths %d and %d"
                                  % (self.k, other.k))
            return other
        if isinstance(other, (int, float)):
            return from_binary64(float(other), self.k)
        return NotImplemented

    def __add__(self, o):
        o = self._coerce(o)
        return o if o is NotImplemented else mc_add(self, o)

    __radd__ = __add__

    def __sub__(self, o):
        o = self._coerce(o)
        return o if o is NotImplemented else mc_sub(self, o)

    def __rsub__(self, o):
        o = self._coerce(o)
        return o if o is NotImplemented else mc_sub(o, self)

    def __mul__(self, o):
        o = self._coerce(o)
        return o if o is NotImplemented else mc_mul(self, o)

    __rmul__ = __mul__

    def __truediv__(self, o):
        o = self._coerce(o)
        return o if o is NotImplemented else mc_div(self, o)

    def __rtruediv__(self, o):
        o = self._coerce(o)
        return o if o is NotImplemented else mc_div(o, self)

    def __neg__(self):
        return mc_neg(self)

    def __abs__(self):
        return mc_abs(self)

    def __eq__(self, o):
        o = self._coerce(o)
        return o if o is NotImplemented else mc_cmp(self, o) == 0

    def __ne__(self, o):
        eq = self.__eq__(o)
        return eq if eq is NotImplemented else not eq

    def __lt__(self, o):
        o = self._coerce(o)
        return o if o is NotImplemented else mc_cmp(self, o) < 0

    def __le__(self, o):
        o = self._coerce(o)
        return o if o is NotImplemented else mc_cmp(self, o) <= 0

    def __gt__(self, o):
        o = self._coerce(o)
        return o if o is NotImplemented else mc_cmp(self, o) > 0

    def __ge__(self, o):
        o = self._coerce(o)
        return o if o is NotImplemented else mc_cmp(self, o) >= 0

    def __hash__(self):
        return hash(self.components)


def _same_width(a, b):
    if a.k != b.k:
        raise DomainError("mixed component widths %d and %d" % (a.k, b.k))
    return a.k


def _device_op(op, a, b):
    k = a.k
    x = np.array(a.components, dtype=np.float64).reshape(k, 1)
    y = np.array((b if b is not None else a).components,
                 dtype=np.float64).reshape(k, 1)
    hx, hy, ho = (nat.Handle(nat.new_vector(k, 1)) for _ in range(3))
    nat.set_planes(hx.h, x)
    nat.set_planes(hy.h, y)
    nat.check(nat.lib().mpcore_elementwise(op, hx.h, hy.h, ho.h),
              "elementwise")
    out = nat.get_planes(ho.h, (k, 1))[:, 0]
    for c in out:
        if not math.isfinite(c):
            raise ArithmeticOverflowError(
                "multi-component result left the binary64 range")
    return MultiComp(tuple(out.tolist()), validate=False)


def mc_add(a, b):
    _same_width(a, b)
    return _device_op(0, a, b)


def mc_sub(a, b):
    _same_width(a, b)
    return _device_op(0, a, mc_neg(b))


def mc_mul(a, b):
    _same_width(a, b)
    return _device_op(1, a, b)


def mc_div(a, b):
    _same_width(a, b)
    if b.components[0] == 0.0:
        raise DivideByZeroError("division by zero")
    return _device_op(2, a, b)


def mc_sqrt(a):
    """Square root (mcfloat.py:596-601, _sqrt_t 324-340): Newton on
    1/sqrt(a) then one Heron correction, on the device (elementwise op 3).
    Raises DomainError for a negative value; sqrt(0) is exactly zero."""
    if a.components[0] < 0.0:
        raise DomainError("square root of a negative value")
    return _device_op(3, a, None)


def mc_neg(a):
    return MultiComp(tuple(-c for c in a.components), validate=False)


def mc_abs(a):
    return mc_neg(a) if a.components[0] < 0.0 else a


def mc_cmp(a, b):
    """Exact three-way comparison (mcfloat.py:343-354): sign of the
    correctly rounded sum of the joint term list."""
    _same_width(a, b)
    terms = list(a.components) + [-c for c in b.components]
    try:
        s = math.fsum(terms)
    except OverflowError:
        s = math.fsum(t * 2.0 ** -60 for t in terms)
    return (s > 0.0) - (s < 0.0)


def from_binary64(x, k):
    x = float(x)
    if not math.isfinite(x):
        raise DomainError("cannot widen non-finite value %r" % (x,))
    return MultiComp((x,) + (0.0,) * (k - 1), validate=False)


def to_binary64(a):
    return a.components[0]
