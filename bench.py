#!/usr/bin/env python3
"""Benchmark of the deflated multigrid-CSLP GMRES solve (BASELINE.json metric:
preconditioned GMRES iterations/s & time-to-solution; achieved HBM GB/s).

One "step" = one complete solve (hd_solve_device: transformed rhs, start
vector, GMRES to tol 1e-7) of the workload.  Default workload: C5 = 2D point
source, k = 1000, p = 3, 1600 x 1600 elements (N = 2,563,201 complex
doubles), DC_MG^1 with beta2 = 0.5, omega = 2/3, nu = 1 -- the largest
BASELINE config and the one its roofline and scaling targets name.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--replicas]
  python bench.py --impl reference ...   # the reference algorithm on the host CPU (1 thread)

N > 1: one process per GPU.  Launched by torchrun (RANK / WORLD_SIZE set), or
by this script itself when --gpus N > 1 and WORLD_SIZE is unset (it re-runs
itself under torch.distributed.run on 127.0.0.1 and relays rank 0's line).
2D configs then run ONE solve as N row slabs over NCCL (hd_create_dist,
strong scaling); --replicas (and every 1D config) runs N
independent replicas instead (weak scaling).  NCCL_DEBUG=INFO is set for
N > 1 so the communicator lines show the rank count.
Timing: CUDA events on a dedicated torch stream that the library, the L2
flush and the events share; barrier + synchronize on both sides, max over
ranks; the L2 is flushed (256 MiB write) between steps, outside the events.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # name: (dim, p, elements, k, extra)   -- BASELINE.json configs[]
    "C1": (1, 2, 80, 50.0),
    "C2": (1, 4, 31623, 1000.0),
    "C3": (2, 2, 320, 200.0),
    "C4": (2, 3, 480, 150.0),   # three-layer wedge k0 = 150 (oracle extension)
    "C5": (2, 3, 1600, 1000.0),
}


def make_problem(mod, cfg):
    """The config's problem from `mod` (the device package or the oracle)."""
    dim, p, ne, k = CONFIGS[cfg]
    if cfg == "C4":
        return mod.wedge_2d(ne, p, k)
    return mod.point_source_2d(ne, p, k) if dim == 2 else mod.point_source_1d(ne, p, k)
SPEC = dict(tag="DC_MG", beta2="0.5", cycles=1, smoothing=1, omega=2.0 / 3.0)
TOL, MAXIT = 1e-7, 100


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def rank_reduce(dist, t_ms, work, device="cpu"):
    """Whole-job timing over ranks: the MAX of the per-rank timed regions and
    the SUM of the work units (bench contract).  Any backend (nccl on the GPU
    box, gloo in tests/test_multirank.py)."""
    if dist is None:
        return float(t_ms), float(work)
    import torch
    tt = torch.tensor([float(t_ms), float(work)], dtype=torch.float64, device=device)
    mx = tt.clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    sm = tt.clone()
    dist.all_reduce(sm, op=dist.ReduceOp.SUM)
    return float(mx[0]), float(sm[1])


def workload_name(cfg):
    dim, p, ne, k = CONFIGS[cfg]
    if cfg == "C4":
        return (f"C4: 2D IgA Helmholtz, three-layer wedge k0={k:g} (1.2/1.5/1.0), source (0.5, 1-h), p={p}, "
                f"{ne}^2 elements, DC_MG^1 (beta2=0.5, omega=2/3, nu=1), GMRES tol 1e-7")
    return f"{cfg}: {dim}D IgA Helmholtz point source, k={k:g}, p={p}, {ne}^{dim} elements, DC_MG^1 (beta2=0.5, omega=2/3, nu=1), GMRES tol 1e-7"


# ---------------------------------------------------------------------------
# CPU legs: the oracle restatement of the reference (test infrastructure)
# ---------------------------------------------------------------------------
def oracle_sample(cfg, iters, warm=0, threads=1):
    """Time `iters` GMRES iterations (after `warm` untimed ones) of the oracle
    on `threads` host threads (1: the reference is single-threaded per solve,
    README:262-263); returns (iterations/s, seconds, note, t_setup)."""
    from threadpoolctl import threadpool_limits
    from oracle import helmdef_oracle as O
    dim, p, ne, k = CONFIGS[cfg]
    with threadpool_limits(limits=threads):
        pb = make_problem(O, cfg)
        spec = O.to_spec(SPEC["tag"], p, k, beta2=SPEC["beta2"], cycles=SPEC["cycles"],
                         smoothing=SPEC["smoothing"], omega=SPEC["omega"])
        t0 = time.perf_counter()
        s = O.assemble(pb)
        big = dim == 2 and s.A.shape[0] > 300_000 and s.separable
        setup = O.compose(s, spec, galerkin="kron" if dim == 2 and s.separable else "sparse",
                          e_solver="fd" if big else "splu")
        t_setup = time.perf_counter() - t0
        gen = O.gmres_steps(setup.op, setup.rhs, setup.start, setup.monitor, O.GmresOptions(MAXIT, TOL))
        done = 0
        tic = time.perf_counter()
        for res in gen:
            done += 1
            if done == warm:
                tic = time.perf_counter()
            if done >= warm + iters or res.converged:
                break
        el = time.perf_counter() - tic
    n = max(done - warm, 1)
    note = (f"oracle port (scipy CSR SpMV + {'fast diagonalisation' if big else 'SuperLU'} E solve), "
            f"GMRES iterations {warm}..{warm + n - 1} of {cfg} on {threads} host thread(s), after "
            f"{t_setup:.1f}s untimed assembly + setup")
    return n / el, el, note, t_setup


def cpu_full_reference(cfg):
    """A committed full CPU time-to-solution of the config (profiles/r2_cpu_full_<cfg>.json), if any."""
    try:
        return json.loads((ROOT / "profiles" / f"r2_cpu_full_{cfg}.json").read_text())
    except Exception:
        return None


def cpu_threads():
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        return max([i.get("num_threads", 1) for i in info] + [1])
    except Exception:
        return os.cpu_count() or 1


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    rate, el, note, t_setup = oracle_sample(args.config, args.steps, warm=args.warmup, threads=1)
    line = {"metric": "preconditioned GMRES iterations/s", "value": rate, "unit": "iterations/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * el / max(args.steps, 1), "higher_is_better": True,
            "scaling": "strong" if (args.gpus > 1 and CONFIGS[args.config][0] == 2 and not args.replicas) else "weak",
            "vs_baseline": None, "dtype": "c128 (f64 complex)", "data": "synthetic (deterministic point source)",
            "config": {"workload": workload_name(args.config), "step": "one GMRES iteration (CPU sample)"},
            "impl": "reference",
            "cpu_baseline": {"value": rate, "unit": "iterations/s", "cores": 1, "kind": "port",
                             "sample": note, "full_solve": cpu_full_reference(args.config)},
            "e2e": {"value": rate, "unit": "iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# GPU leg
# ---------------------------------------------------------------------------
class ClockSampler:
    """Samples SM clocks and throttle reasons through NVML during the timed region."""

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.reasons = set()
        self._stop = threading.Event()
        self.ok = False
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {getattr(nv, k): k for k in dir(nv) if k.startswith("nvmlClocksThrottleReason") and
                 isinstance(getattr(nv, k), int)}
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for bit, name in names.items():
                    if bit and (r & bit) == bit and name not in ("nvmlClocksThrottleReasonNone",
                                                                  "nvmlClocksThrottleReasonAll",
                                                                  "nvmlClocksThrottleReasonGpuIdle",
                                                                  "nvmlClocksThrottleReasonApplicationsClocksSetting"):
                        self.reasons.add(name.replace("nvmlClocksThrottleReason", ""))
            except Exception:
                pass
            time.sleep(0.05)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons)}


def run_gpu(args):
    import torch
    import paper_2010_10232_b200 as hd

    ws, rank, local = dist_env()
    dim, p, ne, k = CONFIGS[args.config]
    slabs = ws > 1 and dim == 2 and not args.replicas
    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    t_asm0 = time.perf_counter()
    sys_ = hd.assemble(make_problem(hd, args.config))
    t_assemble = time.perf_counter() - t_asm0
    spec = hd.to_spec(SPEC["tag"], p, k, beta2=SPEC["beta2"], cycles=SPEC["cycles"], smoothing=SPEC["smoothing"],
                      omega=SPEC["omega"])
    opt = hd.GmresOptions(MAXIT, TOL)
    N = sys_.size
    if slabs:
        # row slabs, one per process, NCCL transport (hd_create_dist): strong scaling of one solve
        uid = [hd.nccl_unique_id() if rank == 0 else None]
        if dist:
            dist.broadcast_object_list(uid, src=0)
        solver = hd.Solver(sys_, spec, dist=(rank, ws, uid[0], local))
    else:
        solver = hd.Solver(sys_, spec, devices=[local])
    # setup of a second context in this process: hd_create without the one-time
    # CUDA / cuBLAS / cuSOLVER initialisation the first context pays
    t_setup_warm = None
    if not slabs:
        t_w0 = time.perf_counter()
        with hd.Solver(sys_, spec, devices=[local]):
            t_setup_warm = time.perf_counter() - t_w0
    # one dedicated stream for the library, the L2 flush and the timing events
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    solver.set_stream(stream.cuda_stream)
    rhs_d = torch.from_numpy(sys_.rhs.view(np.float64)).to(dev)
    x_d = torch.zeros(2 * N, dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def step():
        return solver.solve_device(rhs_d.data_ptr(), x_d.data_ptr(), opt)

    for _ in range(args.warmup):
        r = step()
    torch.cuda.synchronize()
    # --- timed region: K steps, per-step CUDA events, L2 flushed between steps
    #     (graph-resident GMRES loop; the per-kernel roofline comes from one
    #      extra profiled solve after the timed region)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    iters = 0
    launches = 0
    libcalls = 0
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.zero_()
            evs[i][0].record(stream)
            r = step()
            evs[i][1].record(stream)
            iters += r.iterations
            launches += r.kernel_launches
            libcalls += r.library_calls
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    times = [a.elapsed_time(b) for a, b in evs]
    t_ms = float(sum(times))
    # one profiled solve: every launch bracketed by CUDA events on the library stream
    solver.profile(True)
    flush.zero_()
    step()
    torch.cuda.synchronize()
    prof = solver.profile_read()
    solver.profile(False)
    t_max, iters_all = rank_reduce(dist, t_ms, iters, dev)
    if slabs:
        iters_all /= ws  # one distributed solve: every rank reports the same iterations
    value = iters_all / (t_max * 1e-3)

    # --- end to end through the public host-buffer API (pinned host memory)
    rhs_h = torch.from_numpy(sys_.rhs.view(np.float64).copy()).pin_memory()
    x_h = torch.zeros(2 * N, dtype=torch.float64).pin_memory()
    import ctypes as C
    from paper_2010_10232_b200 import HdGmres, HdReport, _check
    res_h = np.zeros(MAXIT + 1)
    e_iters = 0
    e_evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    lib = hd.load_library()
    o = HdGmres(opt.max_iterations, opt.tolerance)
    torch.cuda.synchronize()
    for i in range(args.steps):
        flush.zero_()
        rep = HdReport()
        e_evs[i][0].record(stream)
        _check(lib.hd_solve(solver._ctx, C.byref(o), C.cast(C.c_void_p(rhs_h.data_ptr()), C.POINTER(C.c_double)),
                            C.cast(C.c_void_p(x_h.data_ptr()), C.POINTER(C.c_double)),
                            res_h.ctypes.data_as(C.POINTER(C.c_double)), C.byref(rep)))
        e_evs[i][1].record(stream)
        e_iters += rep.iterations
    torch.cuda.synchronize()
    e_ms = float(sum(a.elapsed_time(b) for a, b in e_evs))
    e_ms, e_iters = rank_reduce(dist, e_ms, e_iters, dev)
    if slabs:
        e_iters /= ws
    e2e = {"value": e_iters / (e_ms * 1e-3), "unit": "iterations/s", "h2d_bytes_per_step": 16 * N,
           "d2h_bytes_per_step": 16 * N + 8 * (r.iterations), "ms_per_step": e_ms / args.steps}

    # --- roofline of the dominant kernel kind (live CUDA events, algorithmic bytes)
    peaks = {}
    try:
        peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)" if "hbm_gbs" in peaks else "fallback 6.65 TB/s"
    dom = max(((k_, v) for k_, v in prof.items() if k_ not in ("dgemm", "lib_gemm")), key=lambda kv: kv[1][1],
              default=None) if prof else None
    roof = None
    breakdown = {}
    tot_prof_ms = sum(v[1] for v in prof.values()) or 1.0
    for name, (n, ms, b) in sorted(prof.items(), key=lambda kv: -kv[1][1]):
        breakdown[name] = {"launches": n, "ms": round(ms, 3), "share": round(ms / tot_prof_ms, 4)}
        if name in ("dgemm", "lib_gemm"):  # FP64 GEMMs of the E solve: FLOPs, not bytes
            breakdown[name]["TFLOPs"] = round(b / (ms * 1e-3) / 1e12, 2) if ms > 0 and b > 0 else None
        else:
            breakdown[name]["GBps"] = round(b / (ms * 1e-3) / 1e9, 1) if ms > 0 and b > 0 else None
    if dom:
        name, (n, ms, b) = dom
        ach = b / (ms * 1e-3) / 1e9
        traffic, traffic_src = None, None
        try:  # per-launch DRAM bytes of the same kernels from the committed ncu capture
            tr_file = max((ROOT / "profiles").glob("r*_traffic.json"))  # the newest round's capture
            tr = json.loads(tr_file.read_text())
            if tr.get("kernel_kind") == name and args.config == "C5":
                traffic, traffic_src = tr["dram_bytes_per_launch"], tr["source"]
        except Exception:
            pass
        roof = {"bound": "hbm", "kernel": name, "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
                "frac": round(ach / peak, 4), "traffic": traffic, "traffic_source": traffic_src, "launches": n,
                "bytes_per_launch": b / n, "us_per_launch": 1e3 * ms / n, "peak_source": peak_src}
    # whole path: the algorithmic bytes of every own kernel of one solve (each
    # launch's compulsory vector passes: (2j+8) P for the Arnoldi passes of
    # iteration j, the fine / multigrid / projection passes, the monitor) over
    # the timed solve time.  Coarse multigrid levels are counted as HBM bytes
    # although they are L2-resident, so this is an upper bound on the DRAM
    # traffic the solve needs; the deflation GEMMs (compute) add none.
    all_b = sum(v[2] for k_, v in prof.items() if k_ not in ("lib_gemm", "dgemm"))
    t_solve_s = t_max / args.steps * 1e-3
    path = {"bytes_per_solve": all_b, "GBps": round(all_b / t_solve_s / 1e9, 1),
            "frac": round(all_b / t_solve_s / 1e9 / peak, 4),
            "note": "sum of the per-launch algorithmic bytes of one profiled solve (own kernels) over the "
                    "timed solve time; coarse levels counted as HBM bytes"}

    line = {"metric": "preconditioned GMRES iterations/s", "value": value, "unit": "iterations/s",
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_max / args.steps,
            "higher_is_better": True, "scaling": "strong" if slabs else "weak", "vs_baseline": None,
            "dtype": "c128 (f64 complex)",
            "data": "synthetic (deterministic point source, as the reference)",
            "config": {"workload": workload_name(args.config), "N": N, "iterations_per_solve": r.iterations,
                       "step": "one full solve (hd_solve_device)",
                       "parallelism": (f"row slabs x{ws} (NCCL)" if slabs else
                                       (f"replicas x{ws}" if ws > 1 else "single GPU")),
                       "l2": "flushed (256 MiB write) between steps, outside the timed events"},
            "time_to_solution_ms": t_max / args.steps, "t_setup_s": r.t_setup,
            "t_setup_warm_s": t_setup_warm, "t_assemble_s": t_assemble,
            "time_to_solution_with_setup_ms": ((t_assemble + t_setup_warm) * 1e3 + t_max / args.steps
                                               if t_setup_warm is not None else None),
            "e2e": e2e, "gpu_launches": launches, "library_calls": libcalls,
            "roofline": roof, "kernel_breakdown": breakdown,
            "roofline_note": "per-kernel CUDA events of one extra profiled solve (host-driven launch loop) "
                             "after the timed region; achieved = algorithmic bytes / event time",
            "path_roofline": path,
            "clocks": clk.summary()}
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        rate, el, note, _ = oracle_sample(args.config, args.cpu_iters, warm=args.cpu_warm, threads=1)
        line["cpu_baseline"] = {"value": rate, "unit": "iterations/s", "cores": 1, "kind": "port",
                                "sample": note, "full_solve": cpu_full_reference(args.config)}
    solver.close()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="C5")
    ap.add_argument("--cpu-iters", type=int, default=6, help="GMRES iterations timed by the cpu_baseline leg")
    ap.add_argument("--cpu-warm", type=int, default=2, help="untimed GMRES iterations before them")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: N independent replicas (weak scaling) instead of one solve as N row slabs")
    args = ap.parse_args()
    ws, _, _ = dist_env()
    if args.gpus > 1 and ws == 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


def spawn_ranks(args):
    """--gpus N without a launcher: re-run this script as N ranks under
    torch.distributed.run on 127.0.0.1 (one process per GPU); every rank's
    output is relayed, rank 0 prints the JSON line."""
    import socket
    import subprocess
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.call(cmd)


if __name__ == "__main__":
    sys.exit(main())
