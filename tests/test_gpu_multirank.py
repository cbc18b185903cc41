"""The row-slab solve across real GPUs: 2 (and, where present, 4 and 8)
processes, one per GPU, NCCL transport (hd_create_dist), against the
single-domain solve -- equal iterations and counts, history within 1e-10,
solution within 1e-8.  Needs as many GPUs as ranks (NCCL refuses two ranks
on one device); skipped on a one-GPU box (the one-process slab program with
virtual ranks covers the same code path there, tests/test_gpu_parity.py)."""
import json
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _ngpus():
    import torch
    return torch.cuda.device_count()


@pytest.mark.parametrize("nranks", [2, 4, 8])
def test_row_slabs_over_nccl_match_single_domain(nranks, tmp_path):
    if _ngpus() < nranks:
        pytest.skip(f"needs {nranks} GPUs, found {_ngpus()}")
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    out = tmp_path / "dist.json"
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nranks}",
                        "--master-addr=127.0.0.1", f"--master-port={port}", str(ROOT / "tests" / "dist_worker.py"),
                        str(out)], capture_output=True, text=True, timeout=900,
                       env=dict(__import__("os").environ, NCCL_DEBUG="INFO", NCCL_DEBUG_SUBSYS="INIT"))
    assert r.returncode == 0, r.stderr[-4000:]
    d = json.loads(out.read_text())
    assert len(d["bounds"]) == nranks + 1
    a, b = d["dist"], d["one"]
    assert (a["iterations"], a["converged"], a["counts"]) == (b["iterations"], b["converged"], b["counts"])
    assert max(abs(x - y) for x, y in zip(a["residuals"], b["residuals"])) <= 1e-10
    assert d["rel"] <= 1e-8
