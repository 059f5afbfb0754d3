"""K1 (coefficient kernel) parity through the C ABI on the B200.

Mirrors the reference's own elemint tests (pkg/tests/test_elemint.py) as
known-answer checks, plus element-wise parity against the reference's golden
table and the CPU oracle.
"""
import numpy as np
import pytest

from conftest import coeff_err, golden, term_scale
from oracle import oracle
from paper_2111_05205_b200 import elemint
from paper_2111_05205_b200.tbasis import BSplineBasis, decomposition_weights, eval_basis

pytestmark = pytest.mark.gpu
C, DT = 1.0, 0.05
POW = {"U": 1, "W": 0, "BU": 0, "BW": -1}


def _random_triangle(rng, span=0.5):
    while True:
        E = rng.uniform(-span, span, (3, 3))
        if np.linalg.norm(np.cross(E[1] - E[0], E[2] - E[0])) >= 0.05:
            return E


def _normal(E):
    n = np.cross(E[1] - E[0], E[2] - E[0])
    return n / np.linalg.norm(n)


@pytest.mark.parametrize("d", [1, 2, 3])
def test_table_matches_reference_golden(d):
    g = golden("coeff_table.npz")
    P, A, B, Cc, s = g["P"], g["A"], g["B"], g["C"], g["s"]
    U, W = elemint.retarded_coeff_table(P, A, B, Cc, g["ez"], s, d, C, DT)
    BU, BW = elemint.retarded_coeff_table(P, A, B, Cc, g["ez"], s, d, C, DT, which="bm", nx=g["nx"])
    for name, got in (("U", U), ("W", W), ("BU", BU), ("BW", BW)):
        sc = term_scale(P, A, B, Cc, s, d, DT, d + POW[name])
        assert coeff_err(got, g[f"{name}{d}"], sc) < 1e-12, (d, name)


@pytest.mark.parametrize("d", [1, 2, 3])
def test_table_matches_oracle_random(d, rng):
    n = 20000
    P = rng.uniform(-1, 1, (n, 3))
    A, B, Cc = (rng.uniform(-0.5, 0.5, (n, 3)) for _ in range(3))
    ez = np.cross(B - A, Cc - A)
    keep = np.linalg.norm(ez, axis=1) > 1e-2
    P, A, B, Cc, ez = P[keep], A[keep], B[keep], Cc[keep], ez[keep]
    ez /= np.linalg.norm(ez, axis=1)[:, None]
    s = rng.uniform(0.01, 3.0, len(P))
    nx = rng.normal(size=P.shape)
    nx /= np.linalg.norm(nx, axis=1)[:, None]
    for which in ("uw", "bm"):
        got = elemint.retarded_coeff_table(P, A, B, Cc, ez, s, d, C, DT, which=which, nx=nx)
        ref = oracle.coeff_table(P, A, B, Cc, ez, s, d, C, DT, which, nx)
        names = ("U", "W") if which == "uw" else ("BU", "BW")
        for k in range(2):
            sc = term_scale(P, A, B, Cc, s, d, DT, d + POW[names[k]])
            assert coeff_err(got[k], ref[k], sc) < 1e-12, (which, k)


def test_nonpositive_gamma_and_not_arrived_are_zero(rng):
    basis = BSplineBasis(2, DT)
    E = _random_triangle(rng)
    xi = rng.uniform(-1, 1, 3)
    assert elemint.single_layer_coeff(xi, E, 0, basis, C) == 0.0
    assert elemint.double_layer_coeff(xi, E, -3, basis, C) == 0.0
    assert elemint.bm_coeffs(xi, [1.0, 0, 0], E, 0, basis, C) == (0.0, 0.0)
    b1 = BSplineBasis(1, DT)
    E2 = np.array([[0.0, 0, 0], [0.01, 0, 0], [0, 0.01, 0]])
    far = np.array([0.0, 0.0, 10.0])
    assert elemint.single_layer_coeff(far, E2, 10, b1, C) == 0.0
    assert elemint.double_layer_coeff(far, E2, 10, b1, C) == 0.0


@pytest.mark.parametrize("d", [1, 2, 3])
def test_self_element_double_layer_free_term(d, rng):
    """Self W = -gamma^d / 2 and the kappa-sum reproduces -N(t)/2 (test_elemint.py:86-104)."""
    basis = BSplineBasis(d, DT)
    E = _random_triangle(rng)
    xi = E.mean(axis=0)
    for gamma in range(1, 8):
        w = elemint.double_layer_coeff(xi, E, gamma, basis, C)
        assert w == pytest.approx(-(gamma ** d) / 2.0, rel=1e-12)
    w = decomposition_weights(d)
    for alpha in range(1, 6):
        summed = sum(w[k] * elemint.double_layer_coeff(xi, E, alpha - k, basis, C) for k in range(d + 2))
        assert summed == pytest.approx(-0.5 * eval_basis(basis, 0, alpha * DT), abs=1e-12)


def test_coplanar_double_layer_vanishes():
    basis = BSplineBasis(2, DT)
    E = np.array([[0.0, 0, 0], [0.4, 0, 0], [0.1, 0.5, 0]])
    xi = np.array([2.0, 1.0, 0.0])
    for gamma in (10, 30, 60):
        assert abs(elemint.double_layer_coeff(xi, E, gamma, basis, C)) < 1e-13


def test_large_time_saturation_d1(rng):
    basis = BSplineBasis(1, DT)
    E = _random_triangle(rng)
    xi = rng.uniform(-1, 1, 3) + np.array([0, 0, 1.0])
    rmax = max(np.linalg.norm(xi - E[k]) for k in range(3))
    g0 = int(np.ceil(rmax / (C * DT))) + 2
    vals = [elemint.single_layer_coeff(xi, E, g, basis, C) for g in range(g0, g0 + 6)]
    diffs = np.diff(vals)
    np.testing.assert_allclose(diffs, diffs[0], rtol=1e-10)


def test_batch_matches_scalar(rng):
    d = 2
    basis = BSplineBasis(d, DT)
    rows = []
    for _ in range(10):
        E = _random_triangle(rng)
        xi = rng.uniform(-1, 1, 3)
        nx = rng.normal(size=3)
        rows.append((xi, E, int(rng.integers(1, 40)), nx / np.linalg.norm(nx)))
    P = np.array([r[0] for r in rows])
    E = np.array([r[1] for r in rows])
    nz = np.array([_normal(r[1]) for r in rows])
    nx = np.array([r[3] for r in rows])
    s = np.array([r[2] * C * DT for r in rows])
    U, W = elemint.retarded_coeff_table(P, E[:, 0], E[:, 1], E[:, 2], nz, s, d, C, DT)
    BU, BW = elemint.retarded_coeff_table(P, E[:, 0], E[:, 1], E[:, 2], nz, s, d, C, DT, which="bm", nx=nx)
    for i, (xi, Ei, gamma, nxi) in enumerate(rows):
        assert U[i] == pytest.approx(elemint.single_layer_coeff(xi, Ei, gamma, basis, C), rel=1e-12, abs=1e-15)
        assert W[i] == pytest.approx(elemint.double_layer_coeff(xi, Ei, gamma, basis, C), rel=1e-12, abs=1e-15)
        bu, bw = elemint.bm_coeffs(xi, nxi, Ei, gamma, basis, C)
        assert BU[i] == pytest.approx(bu, rel=1e-12, abs=1e-15)
        assert BW[i] == pytest.approx(bw, rel=1e-12, abs=1e-15)


def test_argument_errors():
    P = np.zeros((1, 3))
    E = np.eye(3)
    with pytest.raises(ValueError):
        elemint.retarded_coeff_table(P, E[0], E[1], E[2], [0, 0, 1.0], [1.0], 4, C, DT)
    with pytest.raises(ValueError):
        elemint.retarded_coeff_table(P, E[0], E[1], E[2], [0, 0, 1.0], [1.0], 1, C, DT, which="bm")
    with pytest.raises(ValueError):
        elemint.retarded_coeff_table(P, E[0], E[1], E[2], [0, 0, 1.0], [1.0], 1, C, DT, which="xx")


def test_empty_batch():
    z = np.zeros((0, 3))
    U, W = elemint.retarded_coeff_table(z, z, z, z, z, np.zeros(0), 1, C, DT)
    assert U.shape == (0,) and W.shape == (0,)
