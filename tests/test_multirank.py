"""bench.py's N > 1 plumbing on CPU (gloo, world_size 2): the max-over-ranks
timing / sum-over-ranks work reduction, and the reference arm's rank-0-only
rule.  The GPU path itself is exercised by tests/test_gpu_parity.py."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _reduce_rank(rank, ws, port, out):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    import bench
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        t, w = bench.rank_reduce(dist, 10.0 + 5.0 * rank, 7 + rank)
        np.save(os.path.join(out, f"r{rank}.npy"), np.array([t, w]))
    finally:
        dist.destroy_process_group()


def test_rank_reduce_max_time_sum_work(tmp_path):
    mp.spawn(_reduce_rank, args=(2, _port(), str(tmp_path)), nprocs=2, join=True)
    for r in range(2):
        t, w = np.load(tmp_path / f"r{r}.npy")
        assert t == 15.0 and w == 15.0  # max(10, 15); 7 + 8


def test_rank_reduce_single_process():
    sys.path.insert(0, ROOT)
    import bench
    assert bench.rank_reduce(None, 3.5, 4) == (3.5, 4.0)


def test_reference_arm_nonzero_rank_exits_quietly():
    env = dict(os.environ, WORLD_SIZE="2", RANK="1", LOCAL_RANK="1")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "1", "--warmup", "0", "--config", "C1"], env=env, capture_output=True, text=True,
                       timeout=300)
    assert p.returncode == 0 and p.stdout.strip() == ""


def test_reference_arm_rank0_prints_contract_line():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "2", "--warmup", "1", "--config", "C1"], env=env, capture_output=True, text=True,
                       timeout=300)
    assert p.returncode == 0, p.stderr
    line = json.loads(p.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["n_gpus"] == 2 and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "port"
