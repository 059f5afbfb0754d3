"""MOT parity of the CUDA path (tdw_march through the C ABI) on the B200.

Tolerances (BASELINE.json north_star): per-step relative L2 of the unknown
density <= 1e-9; <= 1e-7 for d = 2 BMBIE, where the paper documents
cancellation of significant digits (PAPER.md 1295-1309).  Golden fixtures come
from the reference's own march (tests/golden/make_golden.py); the C oracle
(oracle/) covers the configurations without fixtures.  At BASELINE's full
sizes (configs 2, 3) size-independent properties are checked as well: exact
linearity in the data (scaling by 2 is exact in binary floating point) and
bit-for-bit determinism.
"""
import warnings

import numpy as np
import pytest

from conftest import GOLDEN, golden, per_step_rel
from oracle import oracle
from paper_2111_05205_b200 import marching, scenarios
from paper_2111_05205_b200.tbasis import BSplineBasis

pytestmark = pytest.mark.gpu
TOL = {1: 1e-9, 2: 1e-7, 3: 1e-7}


def _unknown(h, spec):
    return h.u if spec.phi[0] == 1.0 else h.q


def _oracle(spec, **kw):
    uk, qk = marching.greville_samples(spec)
    return oracle.march(spec.mesh.vertices, spec.mesh.triangles, spec.phi, spec.bie, spec.basis.d,
                        spec.c, spec.basis.dt, spec.nt, uk, qk, **kw)


def test_cfg0_matches_reference_everywhere():
    g = golden("march_cfg0.npz")
    spec = scenarios.build_spec(0)
    trace = []
    h = marching.march(spec, rhs_trace=trace)
    assert h.status == str(g["status"]) and h.n_steps == int(g["n_steps"])
    print(f"cfg0 vs reference: worst step {per_step_rel(h.u, g['u']).max():.3e}")
    assert per_step_rel(h.u, g["u"]).max() < 1e-9
    np.testing.assert_array_equal(h.q, g["q"])
    assert per_step_rel(h.tau, g["tau"]).max() < 1e-9
    sig = np.linalg.norm(h.sigma - g["sigma"], axis=1) / np.linalg.norm(g["u"], axis=1).clip(1e-300)
    assert sig.max() < 1e-9
    assert per_step_rel(np.array(trace), g["rhs"]).max() < 1e-9


def test_cfg1_d2_bmbie_matches_reference():
    g = golden("march_cfg1.npz")
    spec = scenarios.build_spec(1)
    h = marching.march(spec)
    assert h.status == str(g["status"]) and h.n_steps == int(g["n_steps"])
    err = per_step_rel(h.u[:, g["sub"]], g["unknown_sub"])
    print(f"cfg1 vs reference: worst step {err.max():.3e} (256-element sample)")
    assert err.max() < TOL[2], err.max()
    for k, b in enumerate(g["full_steps"]):
        ref = g["unknown_full"][k]
        assert np.linalg.norm(h.u[b] - ref) / np.linalg.norm(ref) < TOL[2]


def test_cfg1_matches_oracle_all_elements():
    spec = scenarios.build_spec(1)
    h = marching.march(spec)
    r = _oracle(spec)
    assert per_step_rel(h.u, r["u"]).max() < TOL[2]
    assert per_step_rel(h.tau, r["tau"]).max() < TOL[2]


@pytest.mark.skipif(not (GOLDEN / "march_cfg2.npz").exists(), reason="config-2 fixture not generated")
def test_cfg2_full_size_matches_reference():
    """BASELINE config 2 at full size (5120 elements, BMBIE d=1 Dirichlet, Nt=256)."""
    g = golden("march_cfg2.npz")
    spec = scenarios.build_spec(2)
    assert np.array_equal(spec.mesh.vertices, g["vertices"])
    h = marching.march(spec)
    assert h.status == str(g["status"]) and h.n_steps == int(g["n_steps"])
    err = per_step_rel(h.q[:, g["sub"]], g["unknown_sub"])
    print(f"cfg2 vs reference: worst step {err.max():.3e} (256-element sample)")
    assert err.max() < TOL[1], err.max()
    for k, b in enumerate(g["full_steps"]):
        ref = g["unknown_full"][k]
        assert np.linalg.norm(h.q[b] - ref) / np.linalg.norm(ref) < TOL[1]
    np.testing.assert_allclose(np.linalg.norm(h.q, axis=1), g["unknown_norm"], rtol=TOL[1], atol=0)


def _mini_spec(d, bie, phi_mode, nt=40, f=4, dt_scale=1.0):
    mesh = scenarios.build_mesh(0, frequency=f)
    dt = scenarios.time_step(mesh) * dt_scale
    sig, t0 = 4 * dt, 24 * dt
    zc, nz = mesh.centroids[:, 2].copy(), mesh.normals[:, 2].copy()
    phi = {"neumann": np.ones(mesh.n_elements), "dirichlet": np.zeros(mesh.n_elements),
           "mixed": (mesh.centroids[:, 0] > 0).astype(float)}[phi_mode]

    def q_data(t):
        a = (t - zc - t0) / sig
        return -(nz * 2.0 * a / sig * np.exp(-a * a))

    def u_data(t):
        a = (t - zc - t0) / sig
        return -np.exp(-a * a)

    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return marching.ProblemSpec(mesh, phi, bie, BSplineBasis(d, dt), 1.0, nt, u_data=u_data, q_data=q_data)


@pytest.mark.parametrize("d,bie,phi_mode", [(1, "obie", "dirichlet"), (2, "obie", "neumann"),
                                            (3, "bmbie", "neumann"), (1, "bmbie", "mixed"),
                                            (2, "bmbie", "dirichlet"), (3, "obie", "mixed")])
def test_parameter_grid_matches_oracle(d, bie, phi_mode):
    spec = _mini_spec(d, bie, phi_mode)
    h = marching.march(spec)
    r = _oracle(spec)
    assert h.status == r["status"] and h.n_steps == r["n_steps"]
    tol = TOL[d] if bie == "bmbie" else 1e-9
    for key in ("u", "q"):
        ref = r[key]
        mask = np.linalg.norm(ref, axis=1) > 0
        assert per_step_rel(getattr(h, key)[mask], ref[mask]).max() < tol, key


def test_header_widths_agree(monkeypatch):
    """Units carry 16-bit pair headers when their bands are <= 31 lags and their
    lag range <= 64 lags, 32-bit headers otherwise.  A small time step makes
    both kinds occur in one store; forcing 32-bit headers everywhere
    (TDW_HDR32=1) must give the same densities bit for bit."""
    spec = _mini_spec(1, "obie", "neumann", nt=120, dt_scale=0.2)
    mixed = marching.BandStore(spec).assemble()
    inf = mixed.info()
    assert 0 < inf["units_hdr32"] < inf["n_units"], inf
    a = marching.march(spec, mats=mixed)
    monkeypatch.setenv("TDW_HDR32", "1")
    wide = marching.BandStore(spec).assemble()
    assert wide.info()["units_hdr32"] == wide.info()["n_units"]
    b = marching.march(spec, mats=wide)
    np.testing.assert_array_equal(a.u, b.u)
    r = _oracle(spec)
    assert a.status == r["status"] and a.n_steps == r["n_steps"]
    assert per_step_rel(a.u, r["u"]).max() < 1e-9


@pytest.mark.parametrize("env", ["TDW_SOLVER=smem+TDW_SOLVE_CL=2", "TDW_SOLVER=smem+TDW_SOLVE_CL=4",
                                 "TDW_SOLVER=smem+TDW_SOLVE_CL=16", "TDW_SOLVER=reg+TDW_HALO=0",
                                 "TDW_SOLVER=reg+TDW_HALO=2", "TDW_SOLVER=reg+TDW_HALO=3"])
def test_solver_variants_agree(monkeypatch, env):
    """Every cluster solver the step-time model can pick (register-resident with
    or without halo rounds, or shared-memory at 2..16 CTAs; at 2 and 4 CTAs a
    thread owns several of the 2560 / 1280 rows) converges to the same densities
    on config 2."""
    spec = scenarios.build_spec(2)
    ref = marching.march(spec)
    for kv in env.split("+"):
        k, v = kv.split("=")
        monkeypatch.setenv(k, v)
    store = marching.BandStore(spec).assemble()
    inf = store.info()
    if "TDW_SOLVE_CL" in env:
        assert inf["solve_cluster"] == int(env.split("TDW_SOLVE_CL=")[1])
    h = marching.march(spec, mats=store)
    assert h.status == ref.status and h.n_steps == ref.n_steps
    assert per_step_rel(h.q, ref.q).max() < 1e-11


@pytest.mark.parametrize("kb,overlap", [(1, 1), (2, 1), (2, 2), (3, 2), (4, 1), (4, 4), (5, 5), (6, 3)])
def test_temporal_block_sizes_match_reference(monkeypatch, kb, overlap):
    """One convolution pass per kb steps, running beside `overlap` solves
    (split lags 2..kb+overlap, their unknown part added by the near terms after
    each solve), reproduces the reference golden march of config 2 for every
    block size and overlap; the config-2 default is (5, 5)."""
    g = golden("march_cfg2.npz")
    spec = scenarios.build_spec(2)
    monkeypatch.setenv("TDW_KB", str(kb))
    monkeypatch.setenv("TDW_OVERLAP", str(overlap))
    store = marching.BandStore(spec).assemble()
    inf = store.info()
    assert inf["steps_per_pass"] == kb and inf["pass_overlap"] == overlap, inf
    h = marching.march(spec, mats=store)
    assert h.status == str(g["status"]) and h.n_steps == int(g["n_steps"])
    assert per_step_rel(h.q[:, g["sub"]], g["unknown_sub"]).max() < TOL[1]
    r = _oracle(_mini_spec(3, "bmbie", "mixed"))
    spec_m = _mini_spec(3, "bmbie", "mixed")
    hm = marching.march(spec_m)
    for key in ("u", "q"):
        mask = np.linalg.norm(r[key], axis=1) > 0
        assert per_step_rel(getattr(hm, key)[mask], r[key][mask]).max() < TOL[3], key


def test_halo_solver_is_bit_identical(monkeypatch):
    """The communication-avoiding solver (h sweeps per cluster barrier, halo rows
    recomputed with the owner's operand order) runs the same Jacobi iterates as
    the plain register solver: with h = 2 and the plain solver testing
    convergence every 2 sweeps, the densities agree bit for bit."""
    spec = scenarios.build_spec(2)
    monkeypatch.setenv("TDW_CHEB", "0")  # plain Jacobi sweeps in the halo solver
    monkeypatch.setenv("TDW_SOLVER", "reg")
    monkeypatch.setenv("TDW_CHECK_EVERY", "2")
    monkeypatch.setenv("TDW_NEAR_IN_SOLVE", "0")  # both solvers: all near terms in near_step_kernel
    monkeypatch.setenv("TDW_HALO", "0")
    plain = marching.BandStore(spec).assemble()
    assert plain.info()["solve_halo"] == 0
    hp = marching.march(spec, mats=plain)
    monkeypatch.setenv("TDW_HALO", "2")
    halo = marching.BandStore(spec).assemble()
    assert halo.info()["solve_halo"] == 2
    hh = marching.march(spec, mats=halo)
    np.testing.assert_array_equal(hh.q, hp.q)
    np.testing.assert_array_equal(hh.u, hp.u)


@pytest.mark.parametrize("cfg", [1, 2])
def test_chebyshev_sweeps_match_jacobi(cfg, monkeypatch):
    """The halo solver's Chebyshev-accelerated sweeps (default; rho from the
    assembly's power iteration) converge to the same densities as plain Jacobi
    sweeps and the reference goldens."""
    spec = scenarios.build_spec(cfg)
    h = marching.march(spec)
    monkeypatch.setenv("TDW_CHEB", "0")
    hj = marching.march(spec)
    x, xj = _unknown(h, spec), _unknown(hj, spec)
    assert per_step_rel(x, xj).max() < 1e-12
    g = golden(f"march_cfg{cfg}.npz")
    tol = TOL[spec.basis.d] if spec.bie == "bmbie" else 1e-9
    assert per_step_rel(x[:, g["sub"]], g["unknown_sub"]).max() < tol


@pytest.mark.parametrize("kb,tail", [("5", "1"), ("5", "2"), ("5", "3"), ("6", "1"), ("6", "2"), ("6", "3")])
def test_near_terms_in_the_solve_tail(monkeypatch, kb, tail):
    """The first split lags' near terms formed in the halo solve's tail from the
    owners' x in DSMEM (TDW_NEAR_IN_SOLVE lags; the rest on the near stream) equal
    the all-near_step_kernel form (TDW_NEAR_IN_SOLVE=0) to round-off (another
    summation order), at kb 5 (the config-2 default: a three-lag tail) and kb 6."""
    spec = scenarios.build_spec(2)
    monkeypatch.setenv("TDW_KB", kb)
    monkeypatch.setenv("TDW_NEAR_IN_SOLVE", "0")
    h0 = marching.march(spec)
    monkeypatch.setenv("TDW_NEAR_IN_SOLVE", tail)
    st = marching.BandStore(spec).assemble()
    h1 = marching.march(spec, mats=st)

    def rel(x, ref):  # per step, floored at 1e-6 of the largest step (the first
        n = np.linalg.norm(ref, axis=1)  # steps before the pulse arrives are round-off)
        return np.linalg.norm(x - ref, axis=1) / np.maximum(n, 1e-6 * n.max())
    assert rel(h1.q, h0.q).max() < 1e-11


def test_window_off_is_equivalent():
    """window=False keeps the whole history (marching.py:296-300): same result."""
    spec = _mini_spec(1, "bmbie", "neumann", nt=60)
    a = marching.march(spec, window=True)
    b = marching.march(spec, window=False)
    r = _oracle(spec, window=False)
    assert per_step_rel(b.u, a.u).max() < 1e-10
    assert per_step_rel(b.u, r["u"]).max() < 1e-9


def test_blowup_detector_matches_oracle():
    """A tiny blow-up threshold stops the march at the same step as the reference rule."""
    spec = _mini_spec(1, "obie", "neumann", nt=40)
    h = marching.march(spec, blowup_factor=1e-6)
    uk, qk = marching.greville_samples(spec)
    r = oracle.march(spec.mesh.vertices, spec.mesh.triangles, spec.phi, spec.bie, 1, 1.0,
                     spec.basis.dt, spec.nt, uk, qk, threshold=1e-6)
    assert h.status == "unstable" == r["status"]
    assert h.n_steps == r["n_steps"] < spec.nt - 1
    n = h.n_steps
    assert per_step_rel(h.u[:n], r["u"][:n]).max() < 1e-9
    assert not h.u[n:].any()


def test_reused_store_and_rhs_trace():
    spec = scenarios.build_spec(0)
    store = marching.build_retarded_matrices(spec)
    h1 = marching.march(spec, mats=store)
    h2 = marching.march(spec, mats=store)
    np.testing.assert_array_equal(h1.u, h2.u)
    with pytest.raises(ValueError):
        marching.march(spec, mats=store, window=False)


@pytest.mark.parametrize("cfg", [2, 3])
def test_full_size_linearity_and_determinism(cfg):
    """Full BASELINE sizes: doubling the data doubles every density bit for bit,
    two runs are identical, the march stays stable and finite."""
    spec = scenarios.build_spec(cfg)
    store = marching.BandStore(spec).assemble()
    h1 = marching.march(spec, mats=store)
    assert h1.status == "stable" and h1.n_steps == spec.nt - 1
    x1 = _unknown(h1, spec)
    assert np.isfinite(x1).all() and np.abs(x1).max() > 0
    h2 = marching.march(spec, mats=store)
    np.testing.assert_array_equal(_unknown(h2, spec), x1)
    if spec.q_data is not None:
        f = spec.q_data
        spec.q_data = lambda t: 2.0 * f(t)
    else:
        f = spec.u_data
        spec.u_data = lambda t: 2.0 * f(t)
    h3 = marching.march(spec, mats=store)
    np.testing.assert_array_equal(_unknown(h3, spec), 2.0 * x1)


@pytest.mark.parametrize("cfg,nt,kb", [(2, 16, "6"), (2, 17, "4"), (0, 9, "6"), (1, 8, "5")])
def test_short_loops_last_pass(cfg, nt, kb, monkeypatch):
    """Loops whose last convolution pass has fewer steps than kb (its history
    slices reach past the last step) run cleanly and match the oracle."""
    monkeypatch.setenv("TDW_KB", kb)
    spec = scenarios.build_spec(cfg, nt=nt)
    h = marching.march(spec)
    uk, qk = marching.greville_samples(spec)
    r = oracle.march(spec.mesh.vertices, spec.mesh.triangles, spec.phi, spec.bie, spec.basis.d, spec.c,
                     spec.basis.dt, spec.nt, uk, qk)
    assert h.status == r["status"] and h.n_steps == r["n_steps"]
    x, xr = (h.u, r["u"]) if spec.phi[0] == 1.0 else (h.q, r["q"])
    n = np.linalg.norm(xr, axis=1)
    err = np.linalg.norm(x - xr, axis=1) / np.maximum(n, 1e-6 * n.max())
    assert err.max() < 1e-9


@pytest.mark.parametrize("cfg", [1, 2])
def test_device_side_boundary_data(cfg):
    """march(device_data=True) samples the incident plane pulse on the device
    (tdw_known_plane_pulse): the same densities as the host-sampled march, to
    the last bits of exp."""
    spec = scenarios.build_spec(cfg)
    store = marching.BandStore(spec).assemble()
    h = marching.march(spec, mats=store)
    hd = marching.march(spec, mats=store, device_data=True)
    assert hd.status == h.status and hd.n_steps == h.n_steps
    for a, b in ((hd.u, h.u), (hd.q, h.q)):
        n = np.linalg.norm(b, axis=1)
        assert (np.linalg.norm(a - b, axis=1) / np.maximum(n, 1e-6 * max(n.max(), 1e-300))).max() < 1e-12
    store.close()


@pytest.mark.parametrize("cfg", [2, 3])
def test_full_size_rhs_matches_reference_form(cfg):
    """Full BASELINE size, every step's right-hand side in the reference's own
    sigma/tau lag-CSR form.  For a seeded sample of rows and steps the oracle
    rebuilds those rows of the reference's per-lag matrices (marching.py:132-181)
    and recomputes b_i^alpha (marching.py:315-327: tilde sums, windowed sums at
    the gamma* window bottom, stock sums) from the GPU's OWN history; the GPU's
    rhs_trace must agree (1e-9, 1e-7 for d = 2 BMBIE), and the GPU's solution
    must pass the reference's residual test on those rows (marching.py:330-333)."""
    spec = scenarios.build_spec(cfg)
    trace = []
    h = marching.march(spec, rhs_trace=trace)
    assert h.status == "stable" and h.n_steps == spec.nt - 1
    rhs = np.array(trace)
    ns, nt, d = spec.mesh.n_elements, spec.nt, spec.basis.d
    gstar = marching.BandStore(spec).gamma_star
    rng = np.random.default_rng(100 + cfg)
    rows = np.sort(rng.choice(ns, size=48, replace=False))
    alphas = sorted({1, 2, d + 2, gstar - 1, gstar, gstar + 1, gstar + d + 2, (nt - 1) // 2,
                     nt - 2, nt - 1} | set(rng.integers(3, nt - 1, size=6).tolist()))
    alphas = [a for a in alphas if 1 <= a <= nt - 1]
    uk, qk = marching.greville_samples(spec)
    b, res = oracle.rhs_rows(spec.mesh.vertices, spec.mesh.triangles, spec.phi, spec.bie, d, spec.c,
                             spec.basis.dt, nt, rows, alphas, uk, qk, h.u, h.q, h.tau, h.sigma)
    got = rhs[np.array(alphas) - 1][:, rows].T            # (rows, alphas)
    err = np.linalg.norm(got - b, axis=0) / np.maximum(np.linalg.norm(b, axis=0), 1e-300)
    # the GPU's solution in the reference's lag-1 matrix against the GPU's own b
    # (res = A x - b_oracle, so A x - b_gpu = res + b - got)
    rel_res = np.linalg.norm(res + b - got, axis=0) / np.maximum(np.linalg.norm(got, axis=0), 1e-300)
    tol = TOL[d] if spec.bie == "bmbie" else 1e-9
    print(f"cfg{cfg} rhs vs reference form: worst step {err.max():.3e} (tol {tol:g}), "
          f"worst residual {rel_res.max():.3e}, steps {alphas}")
    assert err.max() < tol, (err.max(), alphas[int(err.argmax())])
    assert rel_res.max() < 1e-10


def test_pair_restricted_store_matches_reference():
    """build_retarded_matrices(spec, pairs=(ii, jj)) (marching.py:132-181 with the
    pairs argument): the reference's own restricted march (config 0, pairs at
    centroid distance < 1.2; tests/golden/march_pairs_cfg0.npz) is reproduced."""
    g = golden("march_pairs_cfg0.npz")
    spec = scenarios.build_spec(0)
    c = spec.mesh.centroids
    ii, jj = np.nonzero(np.linalg.norm(c[:, None, :] - c[None, :, :], axis=2) < float(g["radius"]))
    assert len(ii) == int(g["n_pairs"])
    store = marching.build_retarded_matrices(spec, pairs=(ii, jj))
    trace = []
    h = marching.march(spec, mats=store, rhs_trace=trace)
    assert h.status == str(g["status"]) and h.n_steps == int(g["n_steps"])
    assert per_step_rel(h.u, g["u"]).max() < 1e-9
    assert per_step_rel(np.array(trace), g["rhs"]).max() < 1e-9
    full = marching.march(spec)
    assert per_step_rel(h.u, full.u).max() > 1e-3   # the restriction really changes the problem


def test_build_step_matrix_and_solve():
    """build_step_matrix (marching.py:279-289): A from the device store equals the
    oracle's w0 (W1 phi - U1 (1 - phi)) entry for entry, and lu.solve(b) on the
    device equals scipy's sparse LU solution."""
    import scipy.sparse.linalg as spla
    for cfg in (0, 2):
        spec = scenarios.build_spec(cfg)
        store = marching.build_retarded_matrices(spec)
        A, lu = marching.build_step_matrix(spec, store)
        mesh, d = spec.mesh, spec.basis.d
        v0, v1, v2 = mesh.element_vertices()
        # every pair arrived by lag 1 (marching.py:93-129): the reference's lag-1 pattern
        cen, rad = mesh.centroids, mesh.element_radii()
        dist = np.maximum(np.linalg.norm(cen[:, None, :] - cen[None, :, :], axis=2) - rad[None, :], 0.0)
        rows, cols = np.nonzero(np.maximum(np.ceil(dist / (spec.c * spec.basis.dt)).astype(int) - 1, 1) == 1)
        kw = dict(which="bm", nx=-mesh.normals[rows]) if spec.bie == "bmbie" else {}
        U1, W1 = oracle.coeff_table(mesh.centroids[rows], v0[cols], v1[cols], v2[cols], mesh.normals[cols],
                                    np.full(len(rows), spec.c * spec.basis.dt), d, spec.c, spec.basis.dt, **kw)
        w0 = spec.basis.weights[0]
        ref = np.zeros((mesh.n_elements, mesh.n_elements))
        ref[rows, cols] = w0 * (W1 * spec.phi[cols] - U1 * (1.0 - spec.phi[cols]))
        # (the device keeps only the pairs whose V^(1) is not identically zero)
        assert np.abs(A.toarray() - ref).max() <= 1e-12 * np.abs(ref).max()
        b = np.random.default_rng(cfg).standard_normal(mesh.n_elements)
        x = lu.solve(b)
        xr = spla.spsolve(A.tocsc(), b)
        assert np.linalg.norm(x - xr) <= 1e-12 * np.linalg.norm(xr)
        store.close()


@pytest.mark.parametrize("cfg", [0, 1, 2])
def test_krylov_solver_matches(cfg, monkeypatch):
    """The BiCGSTAB solve the loop switches to for step matrices with a Jacobi
    bound >= 0.9 (forced here with TDW_SOLVER=krylov) reproduces the reference
    (goldens) like the Jacobi cluster solvers do."""
    monkeypatch.setenv("TDW_SOLVER", "krylov")
    spec = scenarios.build_spec(cfg)
    h = marching.march(spec)
    g = golden(f"march_cfg{cfg}.npz")
    assert h.status == str(g["status"]) and h.n_steps == int(g["n_steps"])
    x = _unknown(h, spec)
    tol = TOL[spec.basis.d] if spec.bie == "bmbie" else 1e-9
    assert per_step_rel(x[:, g["sub"]], g["unknown_sub"]).max() < tol


def test_store_validation():
    """A store is tied to the problem it was assembled for (phi, bie, d, c, dt,
    geometry): march refuses another spec; a gamma_max below the lags march
    needs raises like the reference (marching.py:306-308)."""
    spec = scenarios.build_spec(0)
    store = marching.build_retarded_matrices(spec)
    other = scenarios.build_spec(0)
    other.phi = np.zeros_like(other.phi)
    other.u_data, other.q_data = other.q_data, None
    with pytest.raises(ValueError, match="phi"):
        marching.march(other, mats=store)
    short = marching.build_retarded_matrices(spec, gamma_max=3)
    with pytest.raises(ValueError, match="cover the required lags"):
        marching.march(spec, mats=short)
    marching.march(spec, mats=store)  # the matching spec still runs


@pytest.mark.parametrize("cfg", [0, 1, 2])
def test_on_the_fly_mode_matches_reference(cfg):
    """Coefficient mode ON_THE_FLY (SURVEY 8(b) `mode`; north_star (1)): no banded
    store, every convolution pass re-evaluates the closed forms.  Same reference
    goldens and tolerances as the stored mode, and agreement with the stored
    mode to round-off."""
    spec = scenarios.build_spec(cfg)
    store = marching.build_retarded_matrices(spec, mode="on_the_fly")
    inf = store.info()
    assert inf["coeff_mode"] == 2 and inf["store_bytes"] == 0 and inf["n_band"] > 0
    h = marching.march(spec, mats=store)
    g = golden(f"march_cfg{cfg}.npz")
    assert h.status == str(g["status"]) and h.n_steps == int(g["n_steps"])
    x = _unknown(h, spec)
    tol = TOL[spec.basis.d] if spec.bie == "bmbie" else 1e-9
    assert per_step_rel(x[:, g["sub"]], g["unknown_sub"]).max() < tol
    hs = marching.march(spec, mode="stored")
    assert per_step_rel(x, _unknown(hs, spec)).max() < 1e-11   # the same sums, grouped differently
    ms = store.time_conv(3)
    print(f"cfg{cfg} on-the-fly pass {ms:.3f} ms (kb = {inf['steps_per_pass']})")
    store.close()


@pytest.mark.parametrize("cfg", [0, 2])
def test_streamed_march_matches_preloaded(cfg, monkeypatch):
    """march() with host data callables runs the streamed loop (the device takes
    each chunk of Greville samples as soon as the host has written it,
    tdw_march_stream_begin/finish): the same densities as the loop on data
    uploaded up front (tdw_march_device_known), for plain per-step callables and
    vectorised sources, first call (direct launches) and later calls (graph)."""
    spec = scenarios.build_spec(cfg)
    store = marching.BandStore(spec).assemble()
    uk, qk = marching.greville_samples(spec)
    store.upload_known(uk, qk)
    store.run_resident(1e6 * max(spec.blowup_reference, 1e-30), 1)
    ref = store.download()
    f_u, f_q = spec.u_data, spec.q_data
    plain = type(spec)(spec.mesh, spec.phi, spec.bie, spec.basis, spec.c, spec.nt,
                       u_data=(lambda t: f_u(t)) if f_u else None, q_data=(lambda t: f_q(t)) if f_q else None)
    for s in (plain, plain, spec, spec):
        h = marching.march(s, mats=store)
        assert h.status == ref.status and h.n_steps == ref.n_steps
        np.testing.assert_array_equal(h.u, ref.u)
        np.testing.assert_array_equal(h.q, ref.q)
        # the history arrays are written chunk by chunk while the loop runs
        # (tdw_march_stream_outputs): the same values as the download at the end
        np.testing.assert_array_equal(h.tau, ref.tau)
        np.testing.assert_array_equal(h.sigma, ref.sigma)
    # without registered outputs tdw_march_stream_finish copies everything at the end
    monkeypatch.setenv("TDW_STREAM_OUT", "0")
    h = marching.march(plain, mats=store)
    for name in ("u", "q", "tau", "sigma"):
        np.testing.assert_array_equal(getattr(h, name), getattr(ref, name))


def test_streamed_outputs_of_an_unstable_march():
    """Blow-up inside a streamed march: the rows written while the loop ran equal
    those of the march on preloaded data, zero from n_steps on (marching.py:336-338)."""
    import ctypes as C
    from paper_2111_05205_b200 import _lib
    spec = scenarios.build_spec(0)
    store = marching.BandStore(spec).assemble()
    uk, qk = marching.greville_samples(spec)
    store.upload_known(uk, qk)
    thr = 1e-3 * float(np.abs(qk).max() + np.abs(uk).max())   # tripped after a few steps
    store.run_resident(thr, 1)
    ref = store.download()
    assert ref.status == "unstable" and 0 < ref.n_steps < spec.nt - 1
    h = marching.march(spec, mats=store, blowup_factor=thr / max(spec.blowup_reference, 1e-30))
    assert h.status == "unstable" and h.n_steps == ref.n_steps
    for name in ("u", "q", "tau", "sigma"):
        np.testing.assert_array_equal(getattr(h, name), getattr(ref, name))
    assert not h.u[h.n_steps:].any()
    # arrays that are not page-locked are refused
    lib = _lib.load()
    bad = np.zeros((spec.nt - 1, spec.mesh.n_elements))
    rc = lib.tdw_march_stream_outputs(store.h, _lib.dptr(bad), None, None, None)
    assert rc != 0
    store.close()


def test_streamed_march_aborts_when_the_data_raises():
    """A data callable that raises mid-way stops the device loop (flag -1) and the
    exception reaches the caller; the store stays usable."""
    spec = scenarios.build_spec(0)
    store = marching.BandStore(spec).assemble()
    f = spec.q_data
    calls = [0]

    def bad(t):
        calls[0] += 1
        if calls[0] > 40:
            raise ArithmeticError("boom")
        return f(t)
    broken = type(spec)(spec.mesh, spec.phi, spec.bie, spec.basis, spec.c, spec.nt, q_data=bad)
    with pytest.raises(ArithmeticError, match="boom"):
        marching.march(broken, mats=store)
    good = type(spec)(spec.mesh, spec.phi, spec.bie, spec.basis, spec.c, spec.nt, q_data=lambda t: f(t))
    h = marching.march(good, mats=store)
    assert h.status == "stable" and h.n_steps == spec.nt - 1
    # the same once the loop is a cached graph fed by the chunk server (the first
    # streamed marches of a store are launched kernel by kernel)
    ref = marching.march(good, mats=store)
    calls[0] = 0
    with pytest.raises(ArithmeticError, match="boom"):
        marching.march(broken, mats=store)
    h = marching.march(good, mats=store)
    np.testing.assert_array_equal(h.q, ref.q)
    np.testing.assert_array_equal(h.u, ref.u)


def test_store_closed_with_a_streamed_march_in_flight():
    """tdw_problem_destroy while a streamed march still waits for its data (begin
    without finish): the loop is cancelled and drained before anything is freed."""
    import ctypes as C
    import time
    from paper_2111_05205_b200 import _lib
    spec = scenarios.build_spec(0)
    store = marching.BandStore(spec).assemble()
    marching.march(spec, mats=store)                      # first streamed march: direct launches
    marching.march(spec, mats=store)                      # the cached graph and the chunk server
    lib = _lib.load()
    bu, bq = store.pinned_known(0), store.pinned_known(1)
    flag = store.pinned_flag()
    flag[0] = 0                                           # nothing published, ever
    rc = lib.tdw_march_stream_begin(store.h, 1e30, 0, bu.ctypes.data if spec.u_data else None,
                                    bq.ctypes.data if spec.q_data else None, marching.STREAM_CHUNK,
                                    flag.ctypes.data)
    assert rc == 0
    t0 = time.perf_counter()
    store.close()
    assert time.perf_counter() - t0 < 30.0
    h = marching.march(spec)                              # the device is fine afterwards
    assert h.status == "stable"
