"""Host-side logic: mesh/scenario construction, basis constants, the C ABI surface."""
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT, golden
from paper_2111_05205_b200 import _lib, distributed, marching, scenarios, tbasis
from paper_2111_05205_b200.mesh import MeshError, TriMesh, mesh_stats
from paper_2111_05205_b200.shapes import icosphere


@pytest.mark.parametrize("cfg", [0, 1])
def test_scenario_mesh_is_the_reference_mesh(cfg):
    """shapes.icosphere reproduces the reference's vertex order bit for bit
    (config 2's jitter consumes one random number per vertex in that order)."""
    g = golden(f"march_cfg{cfg}.npz")
    spec = scenarios.build_spec(cfg)
    assert np.array_equal(spec.mesh.vertices, g["vertices"])
    assert np.array_equal(spec.mesh.triangles, g["triangles"])
    assert spec.basis.dt == float(g["dt"])
    assert marching.compute_gamma_star(mesh_stats(spec.mesh), spec.basis, spec.c) == int(g["gamma_star"])


def test_scenario_sizes():
    assert scenarios.build_mesh(2).n_elements == 5120
    assert scenarios.build_mesh(3).n_elements == 20480
    m4 = scenarios.build_mesh(4)
    assert m4.n_elements == 40960 and abs(mesh_stats(m4).max_diameter - 5.0) < 1e-9


def test_icosphere_counts():
    for f in (1, 2, 3, 5):
        assert icosphere(f).n_elements == 20 * f * f


def test_weight_tables():
    np.testing.assert_allclose(tbasis.decomposition_weights(1), [1, -2, 1])
    np.testing.assert_allclose(tbasis.decomposition_weights(2), [0.5, -1.5, 1.5, -0.5])
    np.testing.assert_allclose(tbasis.decomposition_weights(3), [1 / 6, -2 / 3, 1, -2 / 3, 1 / 6])
    for d in range(1, 9):
        assert sum(tbasis.decomposition_weights_exact(d)) == 0
    with pytest.raises(ValueError):
        tbasis.decomposition_weights(0)


def test_problem_spec_validation():
    m = icosphere(2)
    with pytest.raises(ValueError):
        marching.ProblemSpec(m, np.ones(3), "obie", tbasis.BSplineBasis(1, 0.1), 1.0, 8)
    with pytest.raises(ValueError):
        marching.ProblemSpec(m, np.ones(m.n_elements), "xbie", tbasis.BSplineBasis(1, 0.1), 1.0, 8)
    with pytest.raises(ValueError):
        marching.ProblemSpec(m, np.ones(m.n_elements), "obie", tbasis.BSplineBasis(1, 0.1), 1.0, 1)
    with pytest.warns(UserWarning):
        marching.ProblemSpec(m, np.ones(m.n_elements), "obie", tbasis.BSplineBasis(1, 0.01), 1.0, 8)


def test_degenerate_mesh_rejected():
    with pytest.raises(MeshError):
        TriMesh(np.array([[0, 0, 0], [1, 0, 0], [2, 0, 0.0]]), np.array([[0, 1, 2]]))


def test_greville_samples_match_reference_recipe():
    g = golden("march_cfg0.npz")
    spec = scenarios.build_spec(0)
    uk, qk = marching.greville_samples(spec)
    # the reference's march consumes these through the tilde sums: its stored q is q_known
    np.testing.assert_array_equal(qk, g["q"])
    assert not uk.any()


def _header_functions():
    text = (ROOT / "include" / "tdw.h").read_text()
    return sorted(set(re.findall(r"^int\s+(tdw_\w+)\(|^const char\*\s+(tdw_\w+)\(", text, re.M)))


def test_library_exports_every_header_symbol():
    """libtdw.so (built by __graft_entry__.build) exports all C-ABI entry points."""
    names = {a or b for a, b in _header_functions()}
    assert len(names) >= 18
    so = _lib.LIB_PATH
    if not so.exists():
        from paper_2111_05205_b200 import build
        build.build()
    out = subprocess.run(["nm", "-D", "--defined-only", str(so)], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\bT (tdw_\w+)", out))
    assert names <= exported, names - exported
    assert set(_lib.EXPORTS) <= exported
    lib = _lib.load()   # loads without a GPU; no compute call is made here
    for n in names:
        assert hasattr(lib, n)


def test_library_refuses_to_run_without_gpu():
    """No CPU fallback: with no device visible the context cannot be created."""
    if _lib.load().tdw_device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(RuntimeError):
        _lib.Context(0)


def test_row_partition_rule():
    for ns in (320, 1280, 5120, 20480, 40960, 1000):
        for n in (1, 2, 4, 8):
            parts = distributed.row_partition(ns, n)
            assert parts[0][0] == 0 and parts[-1][1] == ns
            for (a, b), (c, d) in zip(parts, parts[1:]):
                assert b == c and (b - a) % 32 == 0 or b == ns
            assert max(b - a for a, b in parts) <= distributed.rows_per_rank(ns, n)


def test_vectorised_boundary_data_equals_per_step_calls():
    """PlanePulseData.sample_many (all Greville times at once, on a thread pool, with
    per-chunk callbacks) gives the per-step callable's values bit for bit, and
    sample_data's on_chunk covers every row exactly once for both callable kinds."""
    for cfg in (1, 2):
        spec = scenarios.build_spec(cfg)
        fn = spec.u_data if spec.u_data is not None else spec.q_data
        times = marching.greville_times(spec)
        ref = np.array([fn(float(t)) for t in times])
        out = np.empty_like(ref)
        seen = []
        marching.sample_data(fn, times, out, on_chunk=lambda a, b: seen.append((a, b)))
        np.testing.assert_array_equal(out, ref)
        assert sorted(seen)[0][0] == 0 and sum(b - a for a, b in seen) == len(times)
        plain = lambda t, f=fn: f(t)  # noqa: E731 -- no sample_many: the per-step loop
        seen = []
        out2 = np.empty_like(ref)
        marching.sample_data(plain, times, out2, on_chunk=lambda a, b: seen.append((a, b)))
        np.testing.assert_array_equal(out2, ref)
        assert seen == [(0, len(times))]


def test_time_history_sums_follow_the_reference():
    """TimeHistory.stock_sums / windowed_sums / tilde_sums / finalize_step
    (marching.py:205-242) on the reference's own config-0 history
    (tests/golden/march_cfg0.npz): stock sums reproduce its tau/sigma, the
    windowed sums truncate at the window bottom, the tilde sums drop the
    unknown w0 term, finalize_step promotes the solved density by phi."""
    g = golden("march_cfg0.npz")
    spec = scenarios.build_spec(0)
    h = marching.TimeHistory(spec.basis, spec.nt, spec.mesh.n_elements)
    h.u[:], h.q[:] = g["u"], g["q"]
    w, d = spec.basis.weights, spec.basis.d
    for beta in (0, 1, 2, 5, 40, spec.nt - 2):
        tau, sig = h.stock_sums(beta)
        np.testing.assert_allclose(tau, g["tau"][beta], rtol=0, atol=1e-13 * np.abs(g["tau"]).max())
        np.testing.assert_allclose(sig, g["sigma"][beta], rtol=0, atol=1e-13 * np.abs(g["sigma"]).max())
        for bstar in (beta - 1, beta - 2, beta - d - 1, beta - 10):
            tw, sw = h.windowed_sums(beta, bstar)
            kmax = min(d + 1, beta - bstar, beta)
            ref = sum(w[k] * h.q[beta - k] for k in range(kmax + 1))
            np.testing.assert_array_equal(tw, ref)
    uk, qk = marching.greville_samples(spec)
    beta = 7
    tt, st = h.tilde_sums(beta, spec.phi, uk[beta], qk[beta])
    tau, sig = h.stock_sums(beta)
    np.testing.assert_allclose(tt, tau - w[0] * h.q[beta] + w[0] * qk[beta] * spec.phi, atol=1e-12)
    np.testing.assert_allclose(st, sig - w[0] * h.u[beta] + w[0] * uk[beta] * (1 - spec.phi), atol=1e-12)
    x = g["u"][beta]
    h2 = marching.TimeHistory(spec.basis, spec.nt, spec.mesh.n_elements)
    h2.u[:beta], h2.q[:beta] = g["u"][:beta], g["q"][:beta]
    h2.finalize_step(beta, spec.phi, uk[beta], qk[beta], x)
    np.testing.assert_array_equal(h2.u[beta], x)            # phi = 1: u solved
    np.testing.assert_array_equal(h2.q[beta], qk[beta])     # q known
    np.testing.assert_allclose(h2.tau[beta], g["tau"][beta], atol=1e-13 * np.abs(g["tau"]).max())


def test_fmm_config_defaults_and_gpu_limits():
    """FmmConfig keeps the reference's defaults (ps = pt = 8, leaf capacity 100,
    fmm.py:35-41); the GPU fast solver implements ps = pt = 4 and raises
    ValueError naming that limit before any device work."""
    from paper_2111_05205_b200 import fmm, fmm_plan
    c = fmm_plan.FmmConfig()
    assert (c.ps, c.pt, c.leaf_capacity, c.mu) == (8, 8, 100, 8)
    spec = scenarios.build_spec(0)
    with pytest.raises(ValueError, match="ps = pt = 4"):
        fmm.fast_march(spec)
    with pytest.raises(ValueError, match="mu"):
        fmm_plan.FmmConfig(ps=4, pt=4, mu=9).check_gpu()
    b = fmm_plan.baseline_config()
    assert (b.ps, b.pt, b.leaf_capacity, b.mu) == (4, 4, 20, 8)
    b.check_gpu()


def _physics_spec(bc, bie, d, nt=64):
    """The reference's sphere scenario (tests/golden/make_golden.py physics_spec)."""
    import warnings
    from paper_2111_05205_b200.reference import IncidentPulse
    from paper_2111_05205_b200.tbasis import BSplineBasis
    mesh = icosphere(4, radius=0.5, centre=(0.5, 0.0, 0.0))
    v0, v1, v2 = mesh.element_vertices()
    dt = 0.5 * float(np.concatenate([np.linalg.norm(v1 - v0, axis=1), np.linalg.norm(v2 - v1, axis=1),
                                     np.linalg.norm(v0 - v2, axis=1)]).mean())
    pulse = IncidentPulse(0.5, 1.0)
    cen, nrm = mesh.centroids, mesh.normals
    phi = np.full(mesh.n_elements, 1.0 if bc == "neumann" else 0.0)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return marching.ProblemSpec(mesh, phi, bie, BSplineBasis(d, dt), 1.0, nt,
                                    u_data=(lambda t: -pulse.value(cen, t)) if bc == "dirichlet" else None,
                                    q_data=(lambda t: -pulse.normal_derivative(cen, nrm, t))
                                    if bc == "neumann" else None)


@pytest.mark.parametrize("bc,bie,d", [("neumann", "obie", 1), ("neumann", "bmbie", 2), ("dirichlet", "bmbie", 1)])
def test_sphere_reference_matches_the_reference(bc, bie, d):
    """reference_solution / arc_evaluation_indices / rel_l2_error (reference.py:124-254)
    reproduce the reference's own values on its sphere scenario
    (tests/golden/physics_sphere.npz)."""
    from paper_2111_05205_b200 import reference as R
    g = golden("physics_sphere.npz")
    key = f"{bc}_{bie}{d}"
    spec = _physics_spec(bc, bie, d)
    scen = R.SphereScenario(0.5, (0.5, 0.0, 0.0), bc, 0.5, 1.0)
    idx = R.arc_evaluation_indices(spec.mesh, scen)
    np.testing.assert_array_equal(idx, g[f"{key}_idx"])
    ref = R.reference_solution(scen, spec.mesh.centroids[idx], spec.nt, spec.basis.dt)
    gref = g[f"{key}_reference"]
    assert np.abs(ref - gref).max() <= 1e-10 * np.abs(gref).max()
    assert abs(R.rel_l2_error(g[f"{key}_numerical"], ref) - float(g[f"{key}_error"])) < 1e-9


def test_mesh_loaders_and_orientation(tmp_path):
    """load_mesh (Gmsh MSH 2 ASCII, Wavefront OBJ) and check_orientation
    (mesh.py:110-223): round trips, rejected element types, a flipped sphere."""
    from paper_2111_05205_b200.mesh import check_orientation, load_mesh
    obj = tmp_path / "tri.obj"
    obj.write_text("# one triangle\nv 0 0 0\nv 1 0 0\nv 0 1 0\nf 1/1 2/2 -1\n")
    m = load_mesh(obj)
    assert m.n_elements == 1
    np.testing.assert_allclose(m.normals[0], [0, 0, 1])
    quad = tmp_path / "quad.obj"
    quad.write_text("v 0 0 0\nv 1 0 0\nv 1 1 0\nv 0 1 0\nf 1 2 3 4\n")
    with pytest.raises(MeshError, match="non-triangle"):
        load_mesh(quad)
    msh = tmp_path / "tri.msh"
    msh.write_text("$MeshFormat\n2.2 0 8\n$EndMeshFormat\n$Nodes\n3\n7 0 0 0\n9 1 0 0\n8 0 1 0\n$EndNodes\n"
                   "$Elements\n2\n1 15 2 0 1 7\n2 2 2 0 1 7 9 8\n$EndElements\n")
    m = load_mesh(msh)
    assert m.n_elements == 1 and m.areas[0] == pytest.approx(0.5)
    np.testing.assert_array_equal(m.triangles[0], [0, 2, 1])   # nodes renumbered in id order
    bad = tmp_path / "quad.msh"
    bad.write_text("$MeshFormat\n2.2 0 8\n$EndMeshFormat\n$Nodes\n4\n1 0 0 0\n2 1 0 0\n3 1 1 0\n4 0 1 0\n"
                   "$EndNodes\n$Elements\n1\n1 3 2 0 1 1 2 3 4\n$EndElements\n")
    with pytest.raises(MeshError, match="non-triangle"):
        load_mesh(bad)
    with pytest.raises(MeshError, match="unsupported"):
        load_mesh(tmp_path / "x.stl")
    s = icosphere(4)
    check_orientation(s)
    with pytest.raises(MeshError):
        check_orientation(TriMesh(s.vertices, s.triangles[:, ::-1]))
