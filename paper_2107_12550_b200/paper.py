"""The paper's BNCamPy entry-point names (Listing 1):
TDLUdecompPM(af, af_ch) factors in place and fills the pivot list;
SolveTDLSPM(xf, af, bf, af_ch) solves into xf.  DD/QD variants likewise.
Arguments are the package's DenseMatrix / Vector containers of the
matching width and a list (af_ch) receiving / holding PivotRecord.swaps."""

from .errors import DomainError
from .linalg import PivotRecord, lu_factor_pp, lu_solve


def _lu(k, af, af_ch):
    if af.domain.kind != "mc" or af.domain.k != k:
        raise DomainError("expected a %d-component matrix" % k)
    piv = lu_factor_pp(af)
    if af_ch is not None:
        af_ch[:] = piv.swaps
    return piv


def _solve(k, xf, af, bf, af_ch):
    if af.domain.kind != "mc" or af.domain.k != k:
        raise DomainError("expected a %d-component matrix" % k)
    x = lu_solve(af, PivotRecord(af_ch), bf)
    xf.data[...] = x.data
    return xf


def DDLUdecompPM(af, af_ch=None):
    return _lu(2, af, af_ch)


def TDLUdecompPM(af, af_ch=None):
    return _lu(3, af, af_ch)


def QDLUdecompPM(af, af_ch=None):
    return _lu(4, af, af_ch)


def SolveDDLSPM(xf, af, bf, af_ch):
    return _solve(2, xf, af, bf, af_ch)


def SolveTDLSPM(xf, af, bf, af_ch):
    return _solve(3, xf, af, bf, af_ch)


def SolveQDLSPM(xf, af, bf, af_ch):
    return _solve(4, xf, af, bf, af_ch)
