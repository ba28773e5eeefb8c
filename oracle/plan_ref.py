"""TEST INFRASTRUCTURE ONLY — exact F(o,k) transform construction for the oracle.

This restates, independently of the product package, the reference's host construction so the C
oracle (``winoleg_oracle.c``) can be fed the same nearest-double matrices the reference's
``plan_to_float`` produces:

* point ladder 0, 1, -1, 2, -2, ..., closed with infinity  (reference construct.py:62-75)
* B^T row i = ascending coefficients of prod_{j != i}(x - p_j); infinity row = full modulus
  polynomial prod_j (x - p_j)                                   (construct.py:33-42, :161-164, :175-177)
* G[i, j] = p_i^j / prod_{j' != i}(p_i - p_j'); infinity row e_{k-1}   (construct.py:165-171, :178)
* A[i, j] = p_i^j; infinity row e_{o-1}                           (construct.py:172-174, :179)
* monic Legendre p_{n+1} = x p_n - n^2/(4n^2-1) p_{n-1}; P[j, i] = coeff of x^j in p_i; P^-1 by
  unit-upper back substitution                                     (legendre.py:18-37, :53-75)
* G_P = P G, B_P = P B, A_P = P A                                  (construct.py:182-187)
* every Fraction rounded to the nearest double                     (rational.py:62-64)

Only ``tests/``, ``bench.py``'s cpu-baseline leg and ``__graft_entry__.smoke`` may import this.
"""

from __future__ import annotations

from fractions import Fraction

import numpy as np


def ladder(m: int) -> list[Fraction]:
    pts = [Fraction(0)]
    v = 1
    while len(pts) < m - 1:
        pts.append(Fraction(v))
        if len(pts) < m - 1:
            pts.append(Fraction(-v))
        v += 1
    return pts[: m - 1]


def _poly_mul_linear(coeffs: list[Fraction], root: Fraction) -> list[Fraction]:
    out = [Fraction(0)] * (len(coeffs) + 1)
    for i, c in enumerate(coeffs):
        out[i + 1] += c
        out[i] -= root * c
    return out


def roots_poly(roots) -> list[Fraction]:
    c = [Fraction(1)]
    for r in roots:
        c = _poly_mul_linear(c, Fraction(r))
    return c


def toom_cook(o: int, k: int, finite=None):
    """Exact (G [m,k], B^T [m,m], A [m,o]) as nested lists of Fractions, infinity point last."""
    m = o + k - 1
    pts = ladder(m) if finite is None else [Fraction(p) for p in finite]
    assert len(pts) == m - 1
    G = [[Fraction(0)] * k for _ in range(m)]
    BT = [[Fraction(0)] * m for _ in range(m)]
    A = [[Fraction(0)] * o for _ in range(m)]
    for i, p in enumerate(pts):
        others = pts[:i] + pts[i + 1:]
        poly = roots_poly(others)
        BT[i][: len(poly)] = poly
        denom = Fraction(1)
        for q in others:
            denom *= p - q
        for j in range(k):
            G[i][j] = p ** j / denom
        for j in range(o):
            A[i][j] = p ** j
    full = roots_poly(pts)
    BT[m - 1][: len(full)] = full
    G[m - 1][k - 1] = Fraction(1)
    A[m - 1][o - 1] = Fraction(1)
    return G, BT, A


def legendre_pair(m: int):
    """(P, P^-1) exact, P[j][i] = coefficient of x^j in the monic Legendre p_i."""
    polys = [[Fraction(1)], [Fraction(0), Fraction(1)]]
    for n in range(1, m - 1):
        c = Fraction(n * n, 4 * n * n - 1)
        nxt = [Fraction(0)] + polys[n]
        for j, v in enumerate(polys[n - 1]):
            nxt[j] -= c * v
        polys.append(nxt)
    P = [[Fraction(0)] * m for _ in range(m)]
    for i in range(m):
        for j, c in enumerate(polys[i]):
            P[j][i] = c
    # unit upper triangular inverse by back substitution, column by column
    Pi = [[Fraction(0)] * m for _ in range(m)]
    for col in range(m):
        Pi[col][col] = Fraction(1)
        for row in range(col - 1, -1, -1):
            Pi[row][col] = -sum((P[row][t] * Pi[t][col] for t in range(row + 1, col + 1)), Fraction(0))
    return P, Pi


def matmul(X, Y):
    return [[sum((X[i][t] * Y[t][j] for t in range(len(Y))), Fraction(0)) for j in range(len(Y[0]))]
            for i in range(len(X))]


def transpose(X):
    return [list(r) for r in zip(*X)]


def to_f64(X) -> np.ndarray:
    return np.array([[float(v) for v in row] for row in X], dtype=np.float64)


def exact_plan(o: int = 4, k: int = 3):
    G, BT, A = toom_cook(o, k)
    m = o + k - 1
    P, Pi = legendre_pair(m)
    B = transpose(BT)
    return {
        "o": o, "k": k, "m": m, "G": G, "BT": BT, "AT": transpose(A), "P": P, "Pinv": Pi,
        "G_P": matmul(P, G), "BPT": transpose(matmul(P, B)), "APT": transpose(matmul(P, A)),
    }


def packed_f64(o: int = 4, k: int = 3, identity_base: bool = False) -> np.ndarray:
    """fp64 matrices in the C oracle's packed order: G, BT, AT, Pinv, G_P, BPT, APT."""
    ep = exact_plan(o, k)
    if identity_base:  # reference tests/helpers.py:7-13: P = P^-1 = I, G_P=G, B_P=B, A_P=A
        m = ep["m"]
        eye = [[Fraction(int(i == j)) for j in range(m)] for i in range(m)]
        ep = dict(ep, P=eye, Pinv=eye, G_P=ep["G"], BPT=ep["BT"], APT=ep["AT"])
    parts = [to_f64(ep[name]).ravel() for name in ("G", "BT", "AT", "Pinv", "G_P", "BPT", "APT")]
    return np.ascontiguousarray(np.concatenate(parts))
