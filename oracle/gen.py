"""ORACLE — TEST INFRASTRUCTURE ONLY.

numpy restatement of the seeded planar input recipe (SURVEY.md §8(d)
"Concrete seeded generator"), used by the tests to build inputs on the host
independently of the product's device generator
(paper_2107_12550_b200/csrc/gen.cu), and to check it bit for bit.

  w(i) = RN(mix(S + G*(i+1))) * 2^-63 - 1       (testgen.py:53-59, 100-101:
                                                 splitmix64 step i+1 from
                                                 state S, uniform mapping)
  element e (row-major) of object slot m (A:0, B:1, x:2) in a system of size
  n, component c:  i = ((m*n*n + e)*4 + c)
  c0 = w(i0);  c_j = (c_{j-1} * 2^-53) * w(i_j);  then add_k(c, 0).
"""

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
SEED_BASE = 210712550


def mix(z):
    """splitmix64 output finaliser (testgen.py:57-59) on uint64 arrays."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def uniform(seed, idx):
    """w(i) for uint64 index array idx."""
    idx = np.asarray(idx, dtype=np.uint64)
    with np.errstate(over="ignore"):
        state = np.uint64(seed) + GOLDEN * (idx + np.uint64(1))
    u = mix(state)
    return u.astype(np.float64) * 2.0 ** -63 - 1.0


def raw_planes(k, count, slot, n, seed):
    """Un-normalised (k, count) components for elements 0..count-1."""
    e = np.arange(count, dtype=np.uint64)
    base = (np.uint64(slot) * np.uint64(n) * np.uint64(n) + e) * np.uint64(4)
    out = np.empty((k, count), dtype=np.float64)
    out[0] = uniform(seed, base)
    for c in range(1, k):
        out[c] = (out[c - 1] * 2.0 ** -53) * uniform(seed, base + np.uint64(c))
    return out


def planes(k, shape, slot, n, seed):
    """Renormalised planar (k, *shape) input (add_k(raw, 0) via the oracle)."""
    from . import renormalize_planes
    count = int(np.prod(shape))
    raw = raw_planes(k, count, slot, n, seed)
    return renormalize_planes(raw).reshape((k,) + tuple(shape))


def config_seed(index):
    return SEED_BASE + int(index)
