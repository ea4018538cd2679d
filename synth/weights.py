"""Finite-difference weight generators (seeded-input side; NOT the method).

The paper treats the stencil weights as given data: "the w^{xy}_l are the
R_xy+1 weights for approximating the two dimensional Laplacian" (PAPER.md
l.79, Sec. 1 Eq. 4) and "the w^z_{k,l} are the weights for approximating the
second derivative ... The grid size Delta z_k is absorbed into the w^z_{k,l}"
(Eq. 5). It says they "can be optimized" (l.66-68) but never
gives them. Following SPEC.md l.46-63 we generate maximal-order
(polynomial-exactness) weights with Fornberg's recursion, in exact rationals
or float64, and round once to float32 when handing them to the library and
to the oracle. Both consume the same float32 arrays; neither recomputes them.
"""
from __future__ import annotations

from fractions import Fraction
from typing import Sequence

import numpy as np


def fornberg(x0, nodes: Sequence, m: int = 2):
    """Weights c_j such that sum_j c_j f(nodes[j]) ~ f^{(m)}(x0).

    Fornberg's recursion (Math. Comp. 51, 1988). Works for any number type
    that supports + - * / (Fraction for exact weights, float for float64).
    Returns the list of weights for derivative order ``m``.
    """
    n = len(nodes) - 1
    zero = x0 - x0
    one = zero + 1
    c = [[zero] * (m + 1) for _ in range(n + 1)]
    c1 = one
    c4 = nodes[0] - x0
    c[0][0] = one
    for i in range(1, n + 1):
        mn = min(i, m)
        c2 = one
        c5 = c4
        c4 = nodes[i] - x0
        for j in range(i):
            c3 = nodes[i] - nodes[j]
            c2 = c2 * c3
            if j == i - 1:
                for k in range(mn, 0, -1):
                    c[i][k] = c1 * (k * c[i - 1][k - 1] - c5 * c[i - 1][k]) / c2
                c[i][0] = -c1 * c5 * c[i - 1][0] / c2
            for k in range(mn, 0, -1):
                c[j][k] = (c4 * c[j][k] - k * c[j][k - 1]) / c3
            c[j][0] = c4 * c[j][0] / c3
        c1 = c2
    return [c[j][m] for j in range(n + 1)]


def central_second_derivative(r: int, exact: bool = False):
    """1-D maximal-order central weights c_0..c_r on unit-spaced nodes -r..r."""
    if r < 1:
        raise ValueError("radius must be >= 1")
    if exact:
        nodes = [Fraction(l) for l in range(-r, r + 1)]
        w = fornberg(Fraction(0), nodes, 2)
    else:
        nodes = [float(l) for l in range(-r, r + 1)]
        w = fornberg(0.0, nodes, 2)
    return [w[r + l] for l in range(r + 1)]


def xy_weights(r_xy: int, exact: bool = False):
    """w^xy_0..w^xy_R for the h^2-scaled 2-D Laplacian of Eq. 4.

    w^xy_0 = 2 c_0 (one c_0 from each of the x and y axes), w^xy_l = c_l
    (SPEC.md l.49). Returned as exact Fractions or as float64 numpy array.
    """
    c = central_second_derivative(r_xy, exact=exact)
    w = [2 * c[0]] + list(c[1:])
    if exact:
        return w
    return np.array(w, dtype=np.float64)


def z_coords_ramp(nz: int, r_z: int, dz_top: float, dz_bottom: float) -> np.ndarray:
    """nz + 2 r_z monotone node depths (metres).

    Interior spacing ramps linearly from dz_top to dz_bottom over the nz-1
    interior intervals; the r_z halo nodes above/below extend the edge
    spacing (SURVEY.md Sec. 8(c) reading c4).
    """
    if nz < 2:
        raise ValueError("nz must be >= 2")
    if nz > 2:
        t = np.arange(nz - 1, dtype=np.float64) / (nz - 2)
    else:
        t = np.zeros(1)
    dz = dz_top + (dz_bottom - dz_top) * t
    z_int = np.concatenate([[0.0], np.cumsum(dz)])
    top = z_int[0] - dz[0] * np.arange(r_z, 0, -1, dtype=np.float64)
    bot = z_int[-1] + dz[-1] * np.arange(1, r_z + 1, dtype=np.float64)
    return np.concatenate([top, z_int, bot])


def z_weights(z_coords: Sequence, r_z: int, exact: bool = False):
    """Per-plane weights w^z_{k,l}, l=-r_z..r_z (Eq. 5).

    Row k (interior plane k, 0-based) differentiates at node z_coords[k+r_z]
    using nodes z_coords[k .. k+2 r_z]; stored at column m = l + r_z.
    Units 1/m^2 (Delta z absorbed). Returns (nz, 2 r_z + 1) float64, or a
    list of Fraction rows when ``exact``.
    """
    zc = list(z_coords)
    nz = len(zc) - 2 * r_z
    if nz < 1:
        raise ValueError("too few z nodes for the radius")
    for a, b in zip(zc, zc[1:]):
        if not b > a:
            raise ValueError("z_coords must be strictly increasing")
    rows = []
    for k in range(nz):
        nodes = zc[k:k + 2 * r_z + 1]
        if exact:
            nodes = [Fraction(v) for v in nodes]
            rows.append(fornberg(nodes[r_z], nodes, 2))
        else:
            nodes = [float(v) for v in nodes]
            rows.append(fornberg(nodes[r_z], nodes, 2))
    if exact:
        return rows
    return np.array(rows, dtype=np.float64)
