"""Pins for the weight generators (synth/weights.py): exact rationals and
polynomial exactness. The weights are given data for Eqs. 4-5 (PAPER.md
l.74-87); SPEC.md l.46-63 fixes the examples used here."""
import json
import os
from fractions import Fraction as F

import numpy as np
import pytest

from synth import weights as W

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


@pytest.mark.parametrize("key,r", [("r1", 1), ("r2", 2)])
def test_xy_weights_spec_examples(key, r):
    want = [F(s) for s in GOLD["xy_weights"][key]["w"]]
    assert W.xy_weights(r, exact=True) == want


def test_xy_weights_r4_exact_rationals():
    # c = [-205/72, 8/5, -1/5, 8/315, -1/560] (classic 9-point); w0 = 2 c0
    assert W.xy_weights(4, exact=True) == [F(-205, 36), F(8, 5), F(-1, 5), F(8, 315), F(-1, 560)]


@pytest.mark.parametrize("r", [1, 2, 4, 6, 8, 12])
def test_central_weights_polynomial_exact(r):
    """1-D weights differentiate x^d exactly for d <= 2r (at x0 = 1/3, shifted nodes)."""
    c = W.central_second_derivative(r, exact=True)
    x0 = F(1, 3)
    for d in range(0, 2 * r + 1):
        s = c[0] * x0 ** d + sum(c[l] * ((x0 + l) ** d + (x0 - l) ** d) for l in range(1, r + 1))
        exact = d * (d - 1) * x0 ** (d - 2) if d >= 2 else 0
        assert s == exact, (r, d)
    # and not for degree 2r+2 (maximal order, not more)
    d = 2 * r + 2
    s = c[0] * x0 ** d + sum(c[l] * ((x0 + l) ** d + (x0 - l) ** d) for l in range(1, r + 1))
    assert s != d * (d - 1) * x0 ** (d - 2)


@pytest.mark.parametrize("r", [1, 4, 8, 12])
def test_xy_row_sum_zero(r):
    w = W.xy_weights(r, exact=True)
    assert w[0] + 4 * sum(w[1:]) == 0


def test_z_weights_spec_example():
    g = GOLD["z_weights"]["nodes_0_1_3"]
    rows = W.z_weights([F(s) for s in g["nodes"]], g["r_z"], exact=True)
    assert rows == [[F(s) for s in g["row"]]]


def test_z_weights_uniform_r1():
    dz = F(GOLD["z_weights"]["uniform_r1"]["dz"])
    rows = W.z_weights([dz * i for i in range(5)], 1, exact=True)
    for row in rows:
        assert [v * dz * dz for v in row] == [F(s) for s in GOLD["z_weights"]["uniform_r1"]["row_times_dz2"]]


@pytest.mark.parametrize("rz", [1, 4, 6, 8])
def test_z_weights_nonuniform_polynomial_exact(rz):
    zc = W.z_coords_ramp(12, rz, 5.0, 15.0)
    rows = W.z_weights([F(v) for v in zc], rz, exact=True)
    for k, row in enumerate(rows):
        z0 = F(zc[k + rz])
        nodes = [F(v) for v in zc[k:k + 2 * rz + 1]]
        for d in range(0, 2 * rz + 1):
            s = sum(wm * (zn - z0 + 1) ** d for wm, zn in zip(row, nodes))
            exact = d * (d - 1) if d >= 2 else 0  # d^2/dz^2 (z - z0 + 1)^d at z0
            assert s == exact
        assert sum(row) == 0


def test_z_weights_float64_match_exact_and_scale():
    zc = W.z_coords_ramp(10, 4, 5.0, 15.0)
    wf = W.z_weights(zc, 4)
    we = np.array([[float(v) for v in row] for row in W.z_weights([F(v) for v in zc], 4, exact=True)])
    np.testing.assert_allclose(wf, we, rtol=1e-11, atol=1e-12 * np.abs(we).max())
    # scale covariance: z -> 2z scales weights by 1/4
    np.testing.assert_allclose(W.z_weights(2 * zc, 4), wf / 4, rtol=1e-11, atol=1e-14)


def test_z_weights_uniform_symmetric_and_equal_central():
    dz = 10.0
    zc = np.arange(20) * dz
    wz = W.z_weights(zc, 4)
    c = W.central_second_derivative(4)
    sym = np.array(c[::-1] + c[1:]) / dz ** 2
    np.testing.assert_allclose(wz, np.broadcast_to(sym, wz.shape), rtol=1e-12, atol=1e-16)


def test_z_ramp_monotone_and_halo_extension():
    zc = W.z_coords_ramp(64, 4, 5.0, 15.0)
    d = np.diff(zc)
    assert len(zc) == 64 + 8 and (d > 0).all()
    np.testing.assert_allclose(d[:5], 5.0)
    np.testing.assert_allclose(d[-5:], 15.0)


def test_z_weights_rejects_non_monotone():
    with pytest.raises(ValueError):
        W.z_weights([0.0, 1.0, 1.0, 2.0], 1)
