"""Performance model of the VTI step: the paper's Sec. 2 formulas and this
build's byte model (used by bench.py's roofline fields).

PAPER.md Sec. 2 (l.94-110) gives two computational intensities for the
R_xy / R_z stencils; Sec. 4 (l.272-280) quotes 92 flops per point at
R_xy = 12, R_z = 8, an optimistic CI of 3.3 and a CPU peak fraction of 47 %.
"""
from __future__ import annotations


def flops_per_point(r_xy: int, r_z: int) -> int:
    """The paper's count, 5 R_xy + 4 R_z ("approximatively 92" at 12/8)."""
    return 5 * r_xy + 4 * r_z


def ci_pessimistic(r_xy: int, r_z: int) -> float:
    """Eq. 6: (1/4)(5R_xy + 4R_z)/(4R_xy + 2R_z) flop/byte, loads not cached."""
    return 0.25 * (5 * r_xy + 4 * r_z) / (4 * r_xy + 2 * r_z)


def ci_optimistic(r_xy: int, r_z: int) -> float:
    """Eq. 7: (1/28)(5R_xy + 4R_z) flop/byte, 7 fp32 values per point."""
    return (5 * r_xy + 4 * r_z) / 28.0


def peak_fraction(r_xy: int, r_z: int, peak_gflops: float, bw_gbytes: float, gib: bool = False) -> float:
    """Roofline bound on the fraction of peak flops: CI x bandwidth / peak.

    The paper's "47 %" for 666 GF / 102.4 GB/s is reproduced only when the
    bandwidth is converted as 102.4e9 B/s / 2^30 = 95.4 "G"B/s (gib=True, the
    slip SURVEY.md 2d E3 identifies); with GB/s it is 50.5 %."""
    bw = bw_gbytes * 1e9 * (1e9 / 2 ** 30 if gib else 1.0)
    return ci_optimistic(r_xy, r_z) * bw / (peak_gflops * 1e9)


def bytes_per_point(precision: int = 32) -> int:
    """This build's algorithmic DRAM bytes per point-update: reads
    p^n, q^n, p^{n-1}, q^{n-1}, vx2, vn2, vz2, writes p^{n+1}, q^{n+1}; separable damping."""
    return 9 * precision // 8


def step_flops_per_point(r_xy: int, r_z: int) -> int:
    """Arithmetic of one update in this build's canonical order (fp32 ops per point):
    L: 1 mul + R_xy x (3 add + 1 fma); D: 1 mul + 2R_z fma; vz2*D, 2 fma for F,
    g = gxy*gz, and 2 x (mul, 2 fma, mul) for the two leapfrog updates -> flops
    counting an fma as 2."""
    l_ops = 1 + r_xy * (3 + 2)
    d_ops = 1 + 2 * r_z * 2
    rest = 1 + 2 * 2 + 1 + 2 * (1 + 2 * 2 + 1)
    return l_ops + d_ops + rest
