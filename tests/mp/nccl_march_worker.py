"""Worker of tests/test_gpu_multiprocess.py (one process per GPU, torchrun).

Each rank: the row-sharded store of its rows (BandStore(nranks, rank)) and
march() over the library's NCCL communicator (grouped all-gather of b per
convolution pass), then a single-rank march of the same problem on a
communicator-free context.  The rank writes whether both histories are
bit-identical (and the FMM target-cell-sharded variant likewise)."""
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2111_05205_b200 import _lib, distributed, fmm, fmm_plan, marching, scenarios  # noqa: E402


def main():
    out = Path(sys.argv[1])
    cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    world, rank = dist.get_world_size(), dist.get_rank()
    ctx = _lib.Context(local)
    distributed.init_comm(ctx, dist)
    spec = scenarios.build_spec(cfg)
    store = marching.BandStore(spec, ctx=ctx, nranks=world, rank=rank).assemble()
    h = marching.march(spec, mats=store)
    store.close()
    solo = _lib.Context(local)   # no communicator: the single-GPU path
    ref = marching.march(spec, mats=marching.BandStore(spec, ctx=solo).assemble())
    res = {"rank": rank, "world": world, "direct_equal": bool(np.array_equal(h.u, ref.u) and np.array_equal(h.q, ref.q)),
           "status": h.status, "n_steps": h.n_steps}
    # FMM, target-cell sharded (1280 elements, BMBIE d = 2, 40 steps)
    fspec = scenarios.build_spec(1, nt=40)
    conf = fmm_plan.baseline_config()
    hf = fmm.fast_march(fspec, conf, ctx=ctx, nranks=world, rank=rank)
    rf = fmm.fast_march(fspec, conf, ctx=solo)
    res["fmm_equal"] = bool(np.array_equal(hf.u, rf.u))
    (out / f"rank{rank}.json").write_text(json.dumps(res))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
