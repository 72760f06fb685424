"""Parity tolerances of BASELINE.json's north_star, written out.

float64 ttm: each output within 1e-12 * sum_k |A||B| (the a-priori bound of
a K-term fold) AND the whole output within 1e-12 normwise,
||C_gpu - C_ref||_2 / ||C_ref||_2.  float64 inner products: within
1e-12 * sum|a b| of the reference's fold AND within 1e-12 relative of the
exactly rounded value (normwise for a scalar; computed here with exact
products and math.fsum, so a reference fold's own cancellation error cannot
hide a GPU error or fail a correct result).
"""

from __future__ import annotations

import math

import numpy as np

RTOL64 = 1e-12
RTOL32 = 1e-5


def check_ttm(got, want, bound, rtol=RTOL64):
    """Assert both float64 ttm bounds; return (max elementwise ratio, normwise)."""
    got = np.asarray(got, dtype=np.float64).ravel()
    want = np.asarray(want, dtype=np.float64).ravel()
    bound = np.asarray(bound, dtype=np.float64).ravel()
    d = np.abs(got - want)
    assert np.all(d <= rtol * bound + 1e-300), f"elementwise: max |d|/bound = {np.max(d / np.maximum(bound, 1e-300))}"
    nref = float(np.linalg.norm(want))
    normwise = float(np.linalg.norm(got - want)) / nref if nref > 0 else float(np.linalg.norm(got - want))
    assert normwise <= rtol, f"normwise {normwise}"
    ratio = float(np.max(np.where(bound > 0, d / np.where(bound > 0, bound, 1.0), 0.0))) if d.size else 0.0
    return ratio, normwise


def _two_prod(a, b):
    """Exact products a*b = p + e of binary64 arrays (Dekker/Veltkamp split)."""
    p = a * b
    split = 134217729.0  # 2^27 + 1
    def halves(x):
        t = split * x
        hi = t - (t - x)
        return hi, x - hi
    ah, al = halves(a)
    bh, bl = halves(b)
    e = ((ah * bh - p) + ah * bl + al * bh) + al * bl
    return p, e


def exact_dot(a, b, init=0.0):
    """init + sum a_i b_i, exactly rounded (exact products, math.fsum)."""
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    p, e = _two_prod(a, b)
    return math.fsum(np.concatenate([p, e, [float(init)]]))


def check_inner(got, want_ref, a, b, rtol=RTOL64, init=0.0):
    """Assert |got - ref fold| <= rtol sum|ab| and |got - exact| <= rtol |exact|."""
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    bound = float(np.sum(np.abs(a) * np.abs(b)))
    assert abs(got - want_ref) <= rtol * bound + 1e-300, (got, want_ref, bound)
    ex = exact_dot(a, b, init)
    # 1e-28 sum|ab|: the double-double accumulation's own floor (~eps^2), so a
    # sum that cancels to ~0 is not held to a relative bar no binary64 method meets
    assert abs(got - ex) <= rtol * abs(ex) + 1e-28 * bound + 1e-300, ("normwise", got, ex)
    return abs(got - ex) / abs(ex) if ex else abs(got)
