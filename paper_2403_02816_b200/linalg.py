"""Matrix exponential exp(s*A) by diagonal Pade + scaling-and-squaring.

Setup-only (the reference builds exp(f tau A_mu) once per (direction,
fraction) in prepare, before its timer starts: integrators.py:258-262,
operators.py:123-132).  Same degree ladder {3,5,7,9,13}, 1-norm theta
thresholds and squaring rule as linalg.py:17-87, computed on the host with
LAPACK like the reference; the per-step work never touches it.
"""

import math
from fractions import Fraction

import numpy as np

__all__ = ["expm_pade"]

_LADDER = ((3, 1.495585217958292e-2), (5, 2.539398330063230e-1),
           (7, 9.504178996162932e-1), (9, 2.097847961257068e0),
           (13, 5.371920351148152e0))


def _coeffs(p):
    # c_k = (2p-k)! p! / ((2p)! k! (p-k)!), rescaled to c_p = 1, exact
    raw = [Fraction(math.factorial(2 * p - k) * math.factorial(p),
                    math.factorial(k) * math.factorial(p - k)) for k in range(p + 1)]
    return [float(c / raw[p]) for c in raw]


_C = {p: _coeffs(p) for p, _ in _LADDER}


def _rational(b, p):
    c = _C[p]
    eye = np.eye(b.shape[0], dtype=complex)
    b2 = b @ b
    if p == 13:
        b4 = b2 @ b2
        b6 = b2 @ b4
        odd = b @ (b6 @ (c[13] * b6 + c[11] * b4 + c[9] * b2)
                   + c[7] * b6 + c[5] * b4 + c[3] * b2 + c[1] * eye)
        even = (b6 @ (c[12] * b6 + c[10] * b4 + c[8] * b2)
                + c[6] * b6 + c[4] * b4 + c[2] * b2 + c[0] * eye)
    else:
        odd, even, pw = c[1] * eye, c[0] * eye, eye
        for k in range(1, p // 2 + 1):
            pw = pw @ b2
            odd = odd + c[2 * k + 1] * pw
            even = even + c[2 * k] * pw
        odd = b @ odd
    return np.linalg.solve(even - odd, even + odd)


def expm_pade(a, scale=1.0):
    a = np.asarray(a)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise ValueError(f"matrix must be square, got shape {a.shape}")
    if not np.all(np.isfinite(a)):
        raise ValueError("matrix contains non-finite entries")
    if not np.isfinite(scale):
        raise ValueError("scale must be finite")
    b = np.asarray(a, dtype=complex) * scale
    norm = np.linalg.norm(b, 1) if b.size else 0.0
    for p, theta in _LADDER[:-1]:
        if norm <= theta:
            return _rational(b, p)
    theta13 = _LADDER[-1][1]
    sq = max(0, math.ceil(math.log2(norm / theta13))) if norm > theta13 else 0
    f = _rational(b / (2.0 ** sq), 13)
    for _ in range(sq):
        f = f @ f
    return f
