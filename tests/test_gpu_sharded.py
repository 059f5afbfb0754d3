"""The row-sharded (multi-GPU) code path, emulated on one B200.

tdw_march_emulated runs R shards (ranks) in one process on one device: each
shard assembles only its rows of the banded store and convolves them, reduces
its split partials into its block of b, the in-place all-gather is replaced by
device copies, and every shard runs the redundant cluster solve.  The NCCL
exchange itself runs through a one-rank communicator (tdw_comm_init with
nranks = 1): the same captured loop with the in-place ncclAllGather.  Results
must equal the single-rank march BIT FOR BIT: the convolution sums every row
in fixed tile groups whose partials are added in group order, independent of
the rank count (csrc/assemble.cu schedule), and the FMM's M2L columns do not
depend on which pairs share a work item (csrc/fmm.cu m2l_dmma_kernel).
"""
import ctypes as C

import numpy as np
import pytest

from paper_2111_05205_b200 import _lib, distributed, marching, scenarios

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfg,nranks", [(0, 2), (0, 3), (1, 2), (2, 2), (2, 4), (2, 8)])
def test_sharded_equals_single_rank(cfg, nranks):
    spec = scenarios.build_spec(cfg)
    ref = marching.march(spec)
    hs, infos = distributed.march_emulated(spec, nranks)
    rows = [(i["row_lo"], i["row_hi"]) for i in infos]
    assert rows[0][0] == 0 and max(hi for _, hi in rows) == spec.mesh.n_elements
    assert sum(i["n_pairs"] for i in infos) > 0
    x_ref = ref.u if spec.phi[0] == 1.0 else ref.q
    for h in hs:
        assert h.status == ref.status and h.n_steps == ref.n_steps
        x = h.u if spec.phi[0] == 1.0 else h.q
        np.testing.assert_array_equal(x, x_ref)
        np.testing.assert_array_equal(h.u, hs[0].u)
        np.testing.assert_array_equal(h.q, hs[0].q)


def test_shards_partition_the_band():
    """The shards' stores partition the single-rank store (same band entries)."""
    spec = scenarios.build_spec(0)
    full = marching.BandStore(spec).assemble().info()
    shards = [marching.BandStore(spec, nranks=3, rank=r, shard_only=True).assemble().info()
              for r in range(3)]
    assert sum(s["n_band"] for s in shards) == full["n_band"]
    assert sum(s["n_pairs"] for s in shards) == full["n_pairs"]


@pytest.mark.parametrize("cfg", [0, 2])
def test_one_rank_nccl_exchange_path(cfg):
    """The NCCL all-gather path (captured into the loop's CUDA graph) on a
    one-rank communicator gives the single-rank march bit for bit."""
    spec = scenarios.build_spec(cfg)
    ref = marching.march(spec)
    lib = _lib.load()
    ctx = _lib.Context(0)
    buf = C.create_string_buffer(128)
    _lib.check(lib.tdw_nccl_unique_id(buf), ctx.h, "tdw_nccl_unique_id")
    _lib.check(lib.tdw_comm_init(ctx.h, buf.raw, 1, 0), ctx.h, "tdw_comm_init")
    with pytest.raises(RuntimeError):
        _lib.check(lib.tdw_comm_init(ctx.h, buf.raw, 1, 0), ctx.h, "tdw_comm_init")
    store = marching.BandStore(spec, ctx=ctx).assemble()
    h1 = marching.march(spec, mats=store)
    h2 = marching.march(spec, mats=store)
    for h in (h1, h2):
        assert h.status == ref.status and h.n_steps == ref.n_steps
        np.testing.assert_array_equal(h.u, ref.u)
        np.testing.assert_array_equal(h.q, ref.q)
    store.close()
    ctx.close()


def _fmm_spec(bie, d, nt):
    import warnings
    base = scenarios.build_spec(1, nt=nt)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return marching.ProblemSpec(base.mesh, np.ones(1280), bie, type(base.basis)(d, base.basis.dt),
                                    1.0, nt, q_data=base.q_data)


@pytest.mark.parametrize("bie,d,Z,nt,nranks", [("obie", 1, 100, 64, 2), ("bmbie", 2, 20, 40, 3),
                                               ("bmbie", 2, 20, 40, 8)])
def test_fmm_target_cell_shards_equal_single_rank(bie, d, Z, nt, nranks):
    """Target-cell-sharded FMM, emulated on one GPU: every shard
    holds the single-rank history bit for bit, and the M2L work is split (each
    shard evaluates fewer interaction pairs than one GPU does)."""
    from paper_2111_05205_b200 import fmm, fmm_plan
    spec = _fmm_spec(bie, d, nt)
    cfg = fmm_plan.FmmConfig(ps=4, pt=4, leaf_capacity=Z)
    plan = fmm_plan.build_plan(spec, cfg)
    single = fmm.FmmStore(spec, cfg, plan=plan).assemble()
    ref = marching.march(spec, mats=single)
    pairs1 = single.info()["fmm_m2l_pairs"]
    single.close()
    hs, infos = distributed.fast_march_emulated(spec, nranks, cfg, plan=plan)
    for h in hs:
        assert h.status == ref.status and h.n_steps == ref.n_steps
        np.testing.assert_array_equal(h.u, ref.u)
        np.testing.assert_array_equal(h.u, hs[0].u)
    pairs = [i["fmm_m2l_pairs"] for i in infos]
    assert pairs1 > 0 and max(pairs) < pairs1 and sum(pairs) >= pairs1


def test_fmm_one_rank_nccl_exchange_path():
    """The FMM loop's in-place ncclAllGather of b on a one-rank communicator gives
    the communicator-free fast solver bit for bit."""
    from paper_2111_05205_b200 import fmm, fmm_plan
    spec = _fmm_spec("bmbie", 2, 40)
    cfg = fmm_plan.FmmConfig(ps=4, pt=4, leaf_capacity=20)
    ref = fmm.fast_march(spec, cfg)
    lib = _lib.load()
    ctx = _lib.Context(0)
    buf = C.create_string_buffer(128)
    _lib.check(lib.tdw_nccl_unique_id(buf), ctx.h, "tdw_nccl_unique_id")
    _lib.check(lib.tdw_comm_init(ctx.h, buf.raw, 1, 0), ctx.h, "tdw_comm_init")
    h = fmm.fast_march(spec, cfg, ctx=ctx, nranks=1, rank=0)
    assert h.status == ref.status and h.n_steps == ref.n_steps
    np.testing.assert_array_equal(h.u, ref.u)
    ctx.close()
