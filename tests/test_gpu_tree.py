"""The device-side octree and lists (csrc/tree.cu): bit-exact
against the reference's build_tree (tests/golden/tree_cfg{1,2,3,4}.npz,
uncorrected extra-pair rule) and against the host builder with the corrected
rule the fast solver uses."""
import time

import numpy as np
import pytest

from conftest import golden
from paper_2111_05205_b200 import fmm_tree, scenarios

pytestmark = pytest.mark.gpu


def _same_tree(t, u):
    assert t.leaf_level == u.leaf_level and t.root_half == u.root_half
    assert np.array_equal(t.root_centre, u.root_centre)
    for a, b in zip(t.levels, u.levels):
        assert np.array_equal(a.coords, b.coords) and np.array_equal(a.centres, b.centres)
        for f in ("parent", "il_obs", "il_src", "il_offsets"):
            x, y = getattr(a, f), getattr(b, f)
            assert (x is None and y is None) or np.array_equal(x, y), f
    for L in t.elem_cell:
        assert np.array_equal(t.elem_cell[L], u.elem_cell[L])
    assert all(np.array_equal(x, y) for x, y in zip(t.levels[t.leaf_level].cell_elems,
                                                    u.levels[u.leaf_level].cell_elems))
    assert np.array_equal(t.near_pairs[0], u.near_pairs[0]) and np.array_equal(t.near_pairs[1], u.near_pairs[1])
    assert sorted(t.extra_pairs) == sorted(u.extra_pairs)
    for L in t.extra_pairs:
        assert np.array_equal(t.extra_pairs[L][0], u.extra_pairs[L][0])
        assert np.array_equal(t.extra_pairs[L][1], u.extra_pairs[L][1])


@pytest.mark.parametrize("cfg", [1, 2, 3, 4])
def test_device_tree_is_the_reference_tree(cfg):
    g = golden(f"tree_cfg{cfg}.npz")
    spec = scenarios.build_spec(cfg)
    t0 = time.perf_counter()
    t = fmm_tree.build_tree_device(spec.mesh, spec.c, spec.basis.dt, int(g["leaf_capacity"]), 8, corrected=False)
    dt_dev = time.perf_counter() - t0
    assert t.leaf_level == int(g["leaf_level"])
    assert np.array_equal(t.root_centre, g["root_centre"]) and t.root_half == float(g["root_half"])
    for L, lev in enumerate(t.levels):
        assert np.array_equal(lev.coords, g[f"L{L}_coords"])
        if f"L{L}_il_obs" in g.files:
            assert np.array_equal(lev.il_obs, g[f"L{L}_il_obs"])
            assert np.array_equal(lev.il_src, g[f"L{L}_il_src"])
            assert np.array_equal(lev.il_offsets, g[f"L{L}_il_off"])
    assert np.array_equal(t.near_pairs[0], g["near_i"]) and np.array_equal(t.near_pairs[1], g["near_j"])
    ex = sorted(int(k[5:-2]) for k in g.files if k.startswith("extra") and k.endswith("_i"))
    assert sorted(t.extra_pairs) == ex
    for L in ex:
        assert np.array_equal(t.extra_pairs[L][0], g[f"extra{L}_i"])
        assert np.array_equal(t.extra_pairs[L][1], g[f"extra{L}_j"])
    print(f"cfg{cfg}: device tree {dt_dev:.3f} s (reference build_tree {float(g['t_build']):.1f} s)")


@pytest.mark.parametrize("cfg", [3, 4])
def test_device_tree_equals_host_corrected(cfg):
    spec = scenarios.build_spec(cfg)
    t = fmm_tree.build_tree_device(spec.mesh, spec.c, spec.basis.dt, 20, 8, corrected=True)
    u = fmm_tree.build_tree(spec.mesh, spec.c, spec.basis.dt, 20, 8, corrected=True)
    _same_tree(t, u)
