"""Row-sharded multi-GPU plumbing (one process per GPU).

The path shards by collocation rows: rank r assembles and
convolves only its rows of the banded store; once per time step the partial
right-hand sides are all-gathered over NVLink by NCCL inside libtdw
(csrc/march.cu, ncclAllGather on the library's stream, captured in the step
graph) and every rank solves the small lag-1 system redundantly.

torch.distributed is used only to bootstrap: rank 0 creates the NCCL unique id
through the C ABI (tdw_nccl_unique_id) and broadcasts its 128 bytes; the
library then owns its own communicator (tdw_comm_init).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib

TI = 32  # rows per I-block (csrc/tdw_impl.cuh TDW_TI)


def row_partition(ns: int, nranks: int) -> list[tuple[int, int]]:
    """Rows (internal order) owned by each rank: whole 32-row blocks, the same
    rule as tdw_problem_create (csrc/capi.cu)."""
    nblk = (ns + TI - 1) // TI
    per = (nblk + nranks - 1) // nranks
    rpr = per * TI
    return [(min(ns, r * rpr), min(ns, (r + 1) * rpr)) for r in range(nranks)]


def rows_per_rank(ns: int, nranks: int) -> int:
    nblk = (ns + TI - 1) // TI
    return ((nblk + nranks - 1) // nranks) * TI


def broadcast_unique_id(dist, id_bytes: bytes | None, device=None) -> bytes:
    """Broadcast the 128-byte NCCL id from rank 0 with torch.distributed."""
    import torch
    t = torch.zeros(128, dtype=torch.uint8, device=device or "cpu")
    if dist.get_rank() == 0:
        t.copy_(torch.frombuffer(bytearray(id_bytes), dtype=torch.uint8))
    dist.broadcast(t, src=0)
    return bytes(t.cpu().numpy().tobytes())


def init_comm(ctx: _lib.Context, dist) -> tuple[int, int]:
    """Create the library's NCCL communicator for this process group."""
    world, rank = dist.get_world_size(), dist.get_rank()
    if world == 1:
        return 1, 0
    lib = _lib.load()
    buf = C.create_string_buffer(128)
    if rank == 0:
        _lib.check(lib.tdw_nccl_unique_id(buf), ctx.h, "tdw_nccl_unique_id")
    import torch
    dev = torch.device("cuda", ctx.device) if dist.get_backend() == "nccl" else None
    uid = broadcast_unique_id(dist, buf.raw if rank == 0 else None, dev)
    _lib.check(lib.tdw_comm_init(ctx.h, uid, world, rank), ctx.h, "tdw_comm_init")
    return world, rank


def gather_rows(dist, own: np.ndarray, ns: int) -> np.ndarray:
    """Host-side mirror of the per-step exchange: every rank contributes its
    padded row block, the concatenation truncated to ns is the full vector."""
    import torch
    world = dist.get_world_size()
    rpr = rows_per_rank(ns, world)
    t = torch.zeros(rpr, dtype=torch.float64)
    t[: len(own)] = torch.from_numpy(np.asarray(own, dtype=np.float64))
    out = [torch.zeros(rpr, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(out, t)
    return torch.cat(out).numpy()[:ns]


def march_emulated(spec, nranks: int, window: bool = True, blowup_factor: float = 1e6):
    """Run the row-sharded march of `nranks` shards on ONE GPU (tdw_march_emulated):
    every shard assembles only its rows; the per-step all-gather is emulated by
    device copies.  Returns the TimeHistory of every shard (they solve the same
    system redundantly, so all of them hold the full history)."""
    import ctypes as C

    from . import marching
    shards = [marching.BandStore(spec, window=window, nranks=nranks, rank=r, shard_only=True).assemble()
              for r in range(nranks)]
    uk, qk = marching.greville_samples(spec)
    for sh in shards:
        sh.upload_known(uk, qk)
    arr = (C.c_void_p * nranks)(*[sh.h.value for sh in shards])
    thr = blowup_factor * max(spec.blowup_reference, 1e-30)
    _lib.check(_lib.load().tdw_march_emulated(arr, nranks, float(thr)), shards[0].ctx.h,
               "tdw_march_emulated")
    out = [sh.download() for sh in shards]
    infos = [sh.info() for sh in shards]
    for sh in shards:
        sh.close()
    return out, infos


def fast_march_emulated(spec, nranks: int, config=None, plan=None, blowup_factor: float = 1e6):
    """The target-cell-sharded FMM of `nranks` shards on ONE GPU
    (tdw_march_emulated on FMM shards): each shard assembles its rows' near
    field and evaluates M2L only into the leaf cells of its rows and their
    ancestors; b is exchanged by device copies every step.  Returns the shards'
    TimeHistory and info (fmm_m2l_pairs: the M2L pairs each shard evaluates)."""
    from . import fmm, fmm_plan, marching
    plan = plan or fmm_plan.build_plan(spec, config)
    shards = [fmm.FmmStore(spec, config, plan=plan, nranks=nranks, rank=r, shard_only=True).assemble()
              for r in range(nranks)]
    uk, qk = marching.greville_samples(spec)
    for sh in shards:
        sh.upload_known(uk, qk)
    arr = (C.c_void_p * nranks)(*[sh.h.value for sh in shards])
    thr = blowup_factor * max(spec.blowup_reference, 1e-30)
    _lib.check(_lib.load().tdw_march_emulated(arr, nranks, float(thr)), shards[0].ctx.h,
               "tdw_march_emulated (FMM)")
    out = [sh.download() for sh in shards]
    infos = [sh.info() for sh in shards]
    for sh in shards:
        sh.close()
    return out, infos
