"""Two processes, two GPUs, the real NCCL exchange.

Launches tests/mp/nccl_march_worker.py under torchrun with 2 ranks (one per
GPU, --master-addr 127.0.0.1): the row-sharded march with the grouped
in-place all-gather per convolution pass, and the target-cell-sharded FMM,
must give every rank the single-GPU history bit for bit.  Skipped when fewer
than two GPUs are visible (the emulated shards of test_gpu_sharded.py cover
the same code on one GPU)."""
import json
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _gpus():
    try:
        from paper_2111_05205_b200 import _lib
        return _lib.load().tdw_device_count()
    except Exception:
        return 0


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.skipif(_gpus() < 2, reason="needs two GPUs (one process per GPU)")
def test_two_rank_nccl_march_is_bit_identical(tmp_path):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           str(ROOT / "tests" / "mp" / "nccl_march_worker.py"), str(tmp_path), "2"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-4000:]
    for rank in range(2):
        res = json.loads((tmp_path / f"rank{rank}.json").read_text())
        assert res["direct_equal"] and res["fmm_equal"], res
        assert res["status"] == "stable" and res["n_steps"] == 255
