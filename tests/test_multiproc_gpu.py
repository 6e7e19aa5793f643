"""GPU: the solvers in a multi-process world (one process per rank, torchrun) against the oracle.

tests/nccl_parity.py runs NMF (MU/APG, float64 and the float32 tensor-core path), MDS, Cox
(float64, the fused float32 pass split over two calls, packed genotypes vs int8) and the
power-iteration sigma on column-sharded data, checking every rank's result against the CPU
oracle (ref solvers.py:144-450, comm.py:595-643).

* gloo+cuda, 2 ranks: runs on any box with one or more GPUs (ranks share a GPU; the
  collectives are staged through host memory) — the collective sequence and the padded
  uneven partitions of the multi-GPU solvers, end to end.
* nccl, 2 ranks: the production path (one GPU per rank, NCCL over NVLink); skipped on a
  single-GPU box.  Also exercises the solver-level C ABI loops (bs_*_run) over NCCL.
"""

import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(backend, nproc):
    env = dict(os.environ, BS_PARITY_BACKEND=backend)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(ROOT / "tests" / "nccl_parity.py")]
    res = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900, cwd=ROOT)
    out = res.stdout + res.stderr
    assert res.returncode == 0, out[-6000:]
    assert "FAIL" not in res.stdout, res.stdout[-6000:]
    return res.stdout


def test_two_ranks_gloo_on_one_gpu():
    out = _run("gloo+cuda", 2)
    assert out.count("OK") >= 20, out[-3000:]


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs for NCCL ranks")
def test_two_ranks_nccl():
    out = _run("nccl", 2)
    assert out.count("OK") >= 30, out[-3000:]
