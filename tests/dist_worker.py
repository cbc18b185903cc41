"""One rank of a multi-GPU row-slab solve (launched by tests/test_gpu_multirank.py
under torch.distributed.run, one process per GPU): hd_create_dist over NCCL
with the ncclUniqueId broadcast through torch.distributed, the whole C3-sized
problem solved as nranks slabs; rank 0 also solves single-domain and writes
both results (iterations, counts, history, solution) to argv[1]."""
import json
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2010_10232_b200 as hd  # noqa: E402

rank, ws, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
BASE = dict(beta2="0.5", cycles=1, smoothing=1, omega=2.0 / 3.0)
ne, p, k = 320, 3, 200.0
s = hd.assemble(hd.point_source_2d(ne, p, k))
spec = hd.to_spec("DC_MG", p, k, **BASE)
uid = [hd.nccl_unique_id() if rank == 0 else None]
dist.broadcast_object_list(uid, src=0)
with hd.Solver(s, spec, dist=(rank, ws, uid[0], local)) as d:
    r = d.solve(hd.GmresOptions(100, 1e-7))
    bounds = d.slab_bounds
if rank == 0:
    with hd.Solver(s, spec, devices=[local]) as one:
        r1 = one.solve(hd.GmresOptions(100, 1e-7))
    out = dict(bounds=bounds,
               dist=dict(iterations=r.iterations, converged=r.converged, residuals=r.residuals,
                         counts=[r.counts.matvecs, r.counts.coarse_solves, r.counts.shift_solves, r.counts.vcycles]),
               one=dict(iterations=r1.iterations, converged=r1.converged, residuals=r1.residuals,
                        counts=[r1.counts.matvecs, r1.counts.coarse_solves, r1.counts.shift_solves,
                                r1.counts.vcycles]),
               rel=float(np.linalg.norm(r.solution - r1.solution) / np.linalg.norm(r1.solution)))
    Path(sys.argv[1]).write_text(json.dumps(out))
dist.barrier()
dist.destroy_process_group()
