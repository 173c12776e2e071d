"""The reference's bigfloat module surface (bigfloat.py:52-555) over this
package's long-precision engine (longfloat.py: mpmath raw mpf, one correct
rounding per operation, bit for bit the reference's single-rounding rules;
SURVEY finding 10).  Names, argument meaning and errors follow the
reference so code written against ``mpcore.bigfloat`` runs unchanged:

  BigFloat(sign, man, exp, prec), PrecisionContext(p)
  bf_add/bf_sub/bf_mul/bf_div/bf_sqrt(a, b, ctx)   correctly rounded at ctx.p
  bf_neg/bf_abs/bf_cmp, bf_from_int, bf_from_binary64, bf_to_binary64
  bf_from_multicomp(m, ctx=None)  exact component sum, rounded once (404-416)
  bf_to_multicomp(a, k)           k peeled binary64 heads (419-432)
  bf_parse_decimal(text, ctx), bf_format_decimal(a, digits=None),
  bf_format_hex(a), bf_parse_hex(text, ctx=None)

This is the host ("MP") side the north star keeps on the CPU; nothing here
touches the short-precision GPU path.
"""

from mpmath import libmp as _L

from .errors import DomainError
from .longfloat import (BigFloat, LF, PrecisionContext, format_decimal,
                        format_hex, lf_abs, lf_add, lf_cmp, lf_div, lf_mul,
                        lf_neg, lf_sqrt, lf_sub, parse_decimal, parse_hex)

__all__ = ["BigFloat", "PrecisionContext", "bf_add", "bf_sub", "bf_mul",
           "bf_div", "bf_sqrt", "bf_neg", "bf_abs", "bf_cmp", "bf_from_int",
           "bf_from_binary64", "bf_to_binary64", "bf_from_multicomp",
           "bf_to_multicomp", "bf_parse_decimal", "bf_format_decimal",
           "bf_format_hex", "bf_parse_hex"]


def bf_add(a, b, ctx):
    return lf_add(a, b, ctx.p)


def bf_sub(a, b, ctx):
    return lf_sub(a, b, ctx.p)


def bf_mul(a, b, ctx):
    return lf_mul(a, b, ctx.p)


def bf_div(a, b, ctx):
    return lf_div(a, b, ctx.p)


def bf_sqrt(a, ctx):
    return lf_sqrt(a, ctx.p)


def bf_neg(a):
    return lf_neg(a)


def bf_abs(a):
    return lf_abs(a)


def bf_cmp(a, b):
    return lf_cmp(a, b)


def bf_from_int(n, ctx=None):
    """Exact conversion from int, rounded only if a context is given
    (bigfloat.py:363-372; an exact zero carries prec 2 without one)."""
    n = int(n)
    if n == 0:
        return LF(_L.fzero, ctx.p if ctx else 2)
    return LF.from_int(n, ctx.p if ctx else None)


def bf_from_binary64(x):
    return LF.from_float(x)


def bf_to_binary64(a):
    return a.to_float()


def bf_from_multicomp(m, ctx=None):
    """Exact sum of the components, rounded once to ctx precision
    (exact with ctx=None)."""
    return LF.from_components(m.components, ctx.p if ctx else None)


def bf_to_multicomp(a, k):
    """Nearest k-component value: k peeled rounded binary64 heads, each tail
    the exact remainder of the previous head (canonical form)."""
    from .mcfloat import MultiComp
    return MultiComp(a.to_components(k), validate=False)


def bf_parse_decimal(text, ctx):
    return parse_decimal(text, ctx.p)


def bf_format_decimal(a, digits=None):
    return format_decimal(a, digits)


def bf_format_hex(a):
    return format_hex(a)


def bf_parse_hex(text, ctx=None):
    return parse_hex(text, ctx.p if ctx else None)
