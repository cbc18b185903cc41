"""helmdef-b200: B200-native deflated multigrid-CSLP GMRES for IgA Helmholtz.

Python mirror of the reference's solver surface for the hot path
(/root/reference/proj):

  reference (C++)                                   here
  ------------------------------------------------  ---------------------------------
  Problem factories  src/problems.cpp:34-74         point_source_1d/2d, layered_medium_2d
  assemble()         src/assembly.cpp:163-258       assemble()  -> DiscreteSystem (factored)
  PrecondSpec        inc/precond.hpp:122-130        PrecondSpec
  GmresOptions       inc/linalg.hpp:24-27           GmresOptions
  compose()+gmres()  src/precond.cpp:196, linalg:10 Solver(sys, spec).solve(opt)
  GmresResult        inc/linalg.hpp:29-34           GmresResult
  OperationCounts    inc/precond.hpp:114-119        OperationCounts
  to_spec/run_cell   src/harness.cpp:175-243        to_spec / run_cell

Everything below calls the C-ABI of include/helmdef_b200.h in the in-tree
``libhelmdef_b200.so`` (CUDA, sm_100a).  There is no CPU fallback: if the
library or a CUDA device is missing the calls raise.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import time
from dataclasses import dataclass, field
from pathlib import Path
from typing import List, Optional

import numpy as np

_PKG = Path(__file__).resolve().parent
# HD_LIBRARY: alternative build of the same library (A/B timing of kernel variants)
LIB_PATH = Path(os.environ["HD_LIBRARY"]) if os.environ.get("HD_LIBRARY") else _PKG / "libhelmdef_b200.so"

HD_FIELD_CONSTANT = 0
HD_FIELD_LAYERED = 1
HD_FIELD_WEDGE = 2
HD_APPLY_A, HD_APPLY_SHIFTED, HD_APPLY_MG, HD_APPLY_PROJECT, HD_APPLY_OP, HD_APPLY_Q = range(6)
# hd_status (include/helmdef_b200.h); HelmdefError.status carries one of these
HD_OK, HD_ERR_INVALID, HD_ERR_CUDA, HD_ERR_FACTOR, HD_ERR_NO_DEVICE, HD_ERR_NONFINITE = range(6)

# Every symbol include/helmdef_b200.h declares (checked by tests/test_capi.py).
EXPORTS = ["hd_problem_per_dim", "hd_assemble", "hd_assemble_field", "hd_create", "hd_solve", "hd_solve_device", "hd_size",
           "hd_levels", "hd_apply", "hd_debug_level", "hd_level_size", "hd_set_stream", "hd_profile",
           "hd_profile_read", "hd_destroy", "hd_last_error", "hd_create_slabs", "hd_slab_info",
           "hd_nccl_unique_id", "hd_create_dist", "hd_direct_solve", "hd_debug_check_guards"]
KERNEL_KINDS = ["op_fine", "op_coarse", "jacobi0", "transfer", "exact", "mgs", "iterate", "vec", "givens",
                "lib_gemm", "dgemm"]


class HdProblem(C.Structure):
    _fields_ = [("dim", C.c_int), ("order", C.c_int), ("elements", C.c_int), ("k", C.c_double),
                ("field_kind", C.c_int), ("multipliers", C.c_double * 16), ("lines", C.c_double * 4),
                ("point_source", C.c_int), ("source", C.c_double * 2)]


class HdSystem(C.Structure):
    _fields_ = [("dim", C.c_int), ("order", C.c_int), ("elements", C.c_int), ("per_dim", C.c_int),
                ("field_kind", C.c_int), ("k", C.c_double), ("multipliers", C.c_double * 16),
                ("stiffness_band", C.POINTER(C.c_double)), ("mass_band", C.POINTER(C.c_double)),
                ("interval_mass", C.POINTER(C.c_double)), ("corner_re", C.c_double), ("corner_im", C.c_double),
                ("shift_mass_2d", C.POINTER(C.c_double))]


class HdPrecond(C.Structure):
    _fields_ = [("deflate", C.c_int), ("drop", C.c_double), ("shift", C.c_int), ("beta2", C.c_double),
                ("cycles", C.c_int), ("smooth_steps", C.c_int), ("omega", C.c_double), ("coarsest", C.c_int)]


class HdGmres(C.Structure):
    _fields_ = [("max_iterations", C.c_int), ("tolerance", C.c_double)]


class HdReport(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int), ("matvecs", C.c_long),
                ("coarse_solves", C.c_long), ("shift_solves", C.c_long), ("vcycles", C.c_long),
                ("t_setup_s", C.c_double), ("t_solve_s", C.c_double), ("kernel_launches", C.c_int),
                ("library_calls", C.c_int)]


_lib = None


def load_library() -> C.CDLL:
    """Load the in-tree CUDA library; raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                           "(there is no CPU fallback)")
    lib = C.CDLL(str(LIB_PATH))
    dp = C.POINTER(C.c_double)
    lib.hd_problem_per_dim.argtypes = [C.POINTER(HdProblem)]
    lib.hd_problem_per_dim.restype = C.c_int
    lib.hd_assemble.argtypes = [C.POINTER(HdProblem), dp, dp, dp, dp]
    lib.hd_assemble.restype = C.c_int
    lib.hd_assemble_field.argtypes = [C.POINTER(HdProblem), dp]
    lib.hd_assemble_field.restype = C.c_int
    lib.hd_create.argtypes = [C.POINTER(HdSystem), C.POINTER(HdPrecond), C.POINTER(C.c_int), C.c_int,
                              C.POINTER(C.c_void_p)]
    lib.hd_create.restype = C.c_int
    lib.hd_create_slabs.argtypes = [C.POINTER(HdSystem), C.POINTER(HdPrecond), C.c_int, C.POINTER(C.c_void_p)]
    lib.hd_create_slabs.restype = C.c_int
    lib.hd_nccl_unique_id.argtypes = [C.c_char_p]
    lib.hd_nccl_unique_id.restype = C.c_int
    lib.hd_create_dist.argtypes = [C.POINTER(HdSystem), C.POINTER(HdPrecond), C.c_int, C.c_int, C.c_char_p, C.c_int,
                                   C.POINTER(C.c_void_p)]
    lib.hd_create_dist.restype = C.c_int
    lib.hd_slab_info.argtypes = [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int)]
    lib.hd_slab_info.restype = C.c_int
    lib.hd_solve.argtypes = [C.c_void_p, C.POINTER(HdGmres), dp, dp, dp, C.POINTER(HdReport)]
    lib.hd_solve.restype = C.c_int
    lib.hd_solve_device.argtypes = [C.c_void_p, C.POINTER(HdGmres), C.c_void_p, C.c_void_p, dp,
                                    C.POINTER(HdReport)]
    lib.hd_solve_device.restype = C.c_int
    lib.hd_size.argtypes = [C.c_void_p]
    lib.hd_size.restype = C.c_long
    lib.hd_levels.argtypes = [C.c_void_p]
    lib.hd_levels.restype = C.c_int
    lib.hd_apply.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
    lib.hd_apply.restype = C.c_int
    lib.hd_debug_level.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
    lib.hd_debug_level.restype = C.c_int
    lib.hd_level_size.argtypes = [C.c_void_p, C.c_int]
    lib.hd_level_size.restype = C.c_int
    lib.hd_set_stream.argtypes = [C.c_void_p, C.c_void_p]
    lib.hd_set_stream.restype = C.c_int
    lib.hd_profile.argtypes = [C.c_void_p, C.c_int]
    lib.hd_profile.restype = C.c_int
    lib.hd_profile_read.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_long), C.POINTER(C.c_double),
                                    C.POINTER(C.c_double)]
    lib.hd_profile_read.restype = C.c_int
    lib.hd_direct_solve.argtypes = [C.POINTER(HdSystem), dp, dp]
    lib.hd_direct_solve.restype = C.c_int
    lib.hd_debug_check_guards.argtypes = []
    lib.hd_debug_check_guards.restype = C.c_long
    lib.hd_destroy.argtypes = [C.c_void_p]
    lib.hd_destroy.restype = None
    lib.hd_last_error.argtypes = []
    lib.hd_last_error.restype = C.c_char_p
    _lib = lib
    return lib


class HelmdefError(RuntimeError):
    """Mirrors the reference's std::runtime_error on solver failures."""

    def __init__(self, status: int, msg: str):
        super().__init__(f"[hd_status {status}] {msg}")
        self.status = status


def _check(status: int):
    if status != 0:
        raise HelmdefError(status, load_library().hd_last_error().decode())


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


# ---------------------------------------------------------------------------
# problems and assembly (host side, native)
# ---------------------------------------------------------------------------
LAYERED_MULTIPLIERS = [1.00, 0.50, 1.25, 0.75, 1.50, 1.00, 0.50, 1.25,
                       0.75, 1.50, 1.00, 0.50, 1.25, 0.75, 1.50, 1.00]


@dataclass
class Problem:
    """helmdef::Problem (inc/problems.hpp:50-60), iteration-study subset."""

    name: str
    dim: int
    order: int
    elements: int
    k: float
    layered: bool = False
    multipliers: List[float] = field(default_factory=lambda: [1.0] * 16)
    wedge: bool = False
    wedge_lines: List[float] = field(default_factory=lambda: list(WEDGE_LINES))
    source_xy: Optional[List[float]] = None   # None: (1/2, 1/2), the reference's load


# BASELINE config 4 (an extension: the reference's WaveField cannot express it,
# SURVEY.md §0 C8): top iff y > 0.6 - 0.2x, middle iff y > 0.3 + 0.1x, else bottom.
WEDGE_LINES = [0.6, -0.2, 0.3, 0.1]
WEDGE_MULTIPLIERS = [1.2, 1.5, 1.0]


def point_source_1d(elements, order, k):
    return Problem("point_source_1d", 1, order, elements, float(k))


def point_source_2d(elements, order, k):
    return Problem("point_source_2d", 2, order, elements, float(k))


def layered_medium_2d(elements, order, k, multipliers=None):
    return Problem("layered_medium_2d", 2, order, elements, float(k), True,
                   list(multipliers or LAYERED_MULTIPLIERS))


def wedge_2d(elements, order, k0, multipliers=None, lines=None, source_xy=None):
    """BASELINE config 4: three-layer wedge k = k0 * (top, middle, bottom), point
    source at (0.5, 1 - h) by default (oracle/helmdef_oracle.py wedge_2d)."""
    src = list(source_xy) if source_xy is not None else [0.5, 1.0 - 1.0 / elements]
    return Problem("wedge_2d", 2, order, elements, float(k0), False,
                   list(multipliers or WEDGE_MULTIPLIERS) + [0.0] * 13, True, list(lines or WEDGE_LINES), src)


@dataclass
class DiscreteSystem:
    """DiscreteSystem (inc/assembly.hpp:43-52) in the factored form the device
    consumes: reduced 1D stiffness/mass bands + the load vector."""

    problem: Problem
    per_dim: int
    stiffness_band: np.ndarray     # per_dim x (2p+1)
    mass_band: np.ndarray
    rhs: np.ndarray                # complex128, per_dim**dim
    interval_mass: Optional[np.ndarray] = None
    shift_mass_2d: Optional[np.ndarray] = None   # wedge: K2 stencil, N x (2p+1)^2

    @property
    def dim(self):
        return self.problem.dim

    @property
    def size(self):
        return self.per_dim ** self.problem.dim


def _hd_problem(pb: Problem) -> HdProblem:
    h = HdProblem()
    h.dim, h.order, h.elements, h.k = pb.dim, pb.order, pb.elements, pb.k
    h.field_kind = HD_FIELD_WEDGE if pb.wedge else (HD_FIELD_LAYERED if pb.layered else HD_FIELD_CONSTANT)
    for i, m in enumerate(pb.multipliers):
        h.multipliers[i] = m
    for i, v in enumerate(pb.wedge_lines):
        h.lines[i] = v
    if pb.source_xy is not None:
        h.point_source = 1
        h.source[0], h.source[1] = pb.source_xy
    return h


def assemble(pb: Problem) -> DiscreteSystem:
    """assemble() (src/assembly.cpp:163-258) through the native host assembly."""
    lib = load_library()
    h = _hd_problem(pb)
    n = lib.hd_problem_per_dim(C.byref(h))
    nb = 2 * pb.order + 1
    S = np.zeros((n, nb))
    M = np.zeros((n, nb))
    IM = np.zeros((4, n, nb)) if pb.layered else None
    rhs = np.zeros(n ** pb.dim, dtype=np.complex128)
    _check(lib.hd_assemble(C.byref(h), _dp(S), _dp(M), _dp(IM) if IM is not None else None,
                           rhs.view(np.float64).ctypes.data_as(C.POINTER(C.c_double))))
    K2 = None
    if pb.wedge:
        K2 = np.zeros((n * n, nb * nb))
        _check(lib.hd_assemble_field(C.byref(h), _dp(K2)))
    return DiscreteSystem(pb, n, S, M, rhs, IM, K2)


# ---------------------------------------------------------------------------
# preconditioner / solver options
# ---------------------------------------------------------------------------
@dataclass
class PrecondSpec:
    """PrecondSpec (inc/precond.hpp:122-130)."""

    deflate: bool = False
    drop: float = 0.0
    shift: bool = False
    beta2: float = 1.0
    cycles: int = 0
    smooth_steps: int = 1
    omega: float = 0.6
    coarsest: int = 32  # MultigridOptions::coarsest (inc/precond.hpp:60)


@dataclass
class GmresOptions:
    """GmresOptions (inc/linalg.hpp:24-27)."""

    max_iterations: int = 100
    tolerance: float = 1e-7


@dataclass
class OperationCounts:
    matvecs: int = 0
    coarse_solves: int = 0
    shift_solves: int = 0
    vcycles: int = 0


@dataclass
class GmresResult:
    """GmresResult (inc/linalg.hpp:29-34) + counters and device timings."""

    solution: np.ndarray
    iterations: int = 0
    converged: bool = False
    residuals: List[float] = field(default_factory=list)
    counts: OperationCounts = field(default_factory=OperationCounts)
    t_setup: float = 0.0
    t_solve: float = 0.0
    kernel_launches: int = 0
    library_calls: int = 0


def resolve_beta2(expr, k):  # src/harness.cpp:143-147
    if expr == "1/k":
        return 1.0 / k
    if expr == "1/(3k)":
        return 1.0 / (3.0 * k)
    return float(expr)


def resolution_for(k, kh):  # src/problems.cpp:110-114
    return int(math.ceil(k / kh - 1e-12))


def derived_elements(k, kh, order):  # src/harness.cpp:149-152
    return max(resolution_for(k, kh) + 1 - order, 4)


def to_spec(tag, order, k, epsilon=0.1, beta2="1", cycles=1, smoothing=1, omega=0.6,
            smoothing_by_p=None, omega_by_p=None) -> PrecondSpec:
    """Tag -> PrecondSpec mapping of src/harness.cpp:175-205."""
    s = PrecondSpec()
    if tag == "D":
        s.deflate, s.drop = True, 0.0
    elif tag == "D_eps":
        s.deflate, s.drop = True, epsilon
    elif tag == "C_ex":
        s.shift, s.cycles = True, 0
    elif tag == "DC_MG":
        s.deflate, s.drop, s.shift, s.cycles = True, 0.0, True, cycles
    elif tag == "Deps_C_MG":
        s.deflate, s.drop, s.shift, s.cycles = True, epsilon, True, cycles
    elif tag != "none":
        raise ValueError("unknown preconditioner tag: " + tag)
    if s.shift:
        s.beta2 = resolve_beta2(str(beta2), k)
    s.smooth_steps = (smoothing_by_p or {}).get(order, smoothing)
    s.omega = (omega_by_p or {}).get(order, omega)
    return s


def nccl_unique_id() -> bytes:
    """128-byte ncclUniqueId for hd_create_dist (create on rank 0, broadcast to all)."""
    buf = C.create_string_buffer(128)
    _check(load_library().hd_nccl_unique_id(buf))
    return buf.raw


def system_from_bands(pb: Problem, S1: np.ndarray, M1: np.ndarray, rhs: np.ndarray) -> DiscreteSystem:
    """DiscreteSystem from given dense reduced 1D factors and load vector (a
    constant-k problem): the device solves exactly these inputs, e.g. the
    oracle's own assembly, so parity tests compare solvers on the same system."""
    n, b = S1.shape[0], pb.order
    def band(X):
        B = np.zeros((n, 2 * b + 1))
        for d in range(-b, b + 1):
            dg = np.diagonal(X, d)
            if d >= 0:
                B[:n - d, d + b] = dg
            else:
                B[-d:, d + b] = dg
        return B
    return DiscreteSystem(pb, n, band(np.asarray(S1)), band(np.asarray(M1)),
                          np.ascontiguousarray(rhs, dtype=np.complex128))


def _hd_system(sys_: DiscreteSystem):
    """hd_system view of a DiscreteSystem (+ the arrays it points into, to keep alive)."""
    pb = sys_.problem
    h = HdSystem()
    h.dim, h.order, h.elements, h.per_dim = pb.dim, pb.order, pb.elements, sys_.per_dim
    h.field_kind = HD_FIELD_WEDGE if pb.wedge else (HD_FIELD_LAYERED if pb.layered else HD_FIELD_CONSTANT)
    h.k = pb.k
    for i, m in enumerate(pb.multipliers):
        h.multipliers[i] = m
    keep = [np.ascontiguousarray(sys_.stiffness_band), np.ascontiguousarray(sys_.mass_band)]
    h.stiffness_band = _dp(keep[0])
    h.mass_band = _dp(keep[1])
    if sys_.interval_mass is not None:
        keep.append(np.ascontiguousarray(sys_.interval_mass))
        h.interval_mass = _dp(keep[-1])
    if sys_.shift_mass_2d is not None:
        keep.append(np.ascontiguousarray(sys_.shift_mass_2d))
        h.shift_mass_2d = _dp(keep[-1])
    return h, keep


def direct_solve(sys_: DiscreteSystem, rhs: Optional[np.ndarray] = None) -> np.ndarray:
    """x = A^-1 f by an exact device solve (hd_direct_solve): the reference's
    DirectSolver(sys.A).solve(sys.rhs) behind RunRecord::direct_gap
    (src/harness.cpp:234-238)."""
    lib = load_library()
    h, keep = _hd_system(sys_)
    b = np.ascontiguousarray(sys_.rhs if rhs is None else rhs, dtype=np.complex128)
    x = np.zeros_like(b)
    _check(lib.hd_direct_solve(C.byref(h), _dp(b.view(np.float64)), _dp(x.view(np.float64))))
    return x


def check_guards() -> int:
    """Changed guard zones over the live device allocations (HD_POISON=1 runs;
    the pool has no compute-sanitizer, see include/helmdef_b200.h)."""
    n = load_library().hd_debug_check_guards()
    if n < 0:
        raise HelmdefError(2, load_library().hd_last_error().decode())
    return int(n)


class Solver:
    """compose(sys, spec) on the device; .solve() is gmres(op, rhs, start, monitor)."""

    def __init__(self, sys_: DiscreteSystem, spec: PrecondSpec, devices=None, slabs: int = 0, dist=None):
        """slabs > 0: the row-slab decomposition on this GPU (hd_create_slabs);
        dist = (rank, nranks, nccl_id, device): one slab per process over NCCL (hd_create_dist)."""
        lib = load_library()
        self._lib = lib
        self.sys = sys_
        self.spec = spec
        h, self._keep = _hd_system(sys_)
        p = HdPrecond(int(spec.deflate), spec.drop, int(spec.shift), spec.beta2, spec.cycles,
                      spec.smooth_steps, spec.omega, spec.coarsest)
        ctx = C.c_void_p()
        if devices:
            arr = (C.c_int * len(devices))(*devices)
            _check(lib.hd_create(C.byref(h), C.byref(p), arr, len(devices), C.byref(ctx)))
        elif dist is not None:
            rank, nranks, uid, dev = dist
            _check(lib.hd_create_dist(C.byref(h), C.byref(p), int(rank), int(nranks), bytes(uid), int(dev),
                                      C.byref(ctx)))
            slabs = int(nranks)
        elif slabs:
            _check(lib.hd_create_slabs(C.byref(h), C.byref(p), int(slabs), C.byref(ctx)))
        else:
            _check(lib.hd_create(C.byref(h), C.byref(p), None, 0, C.byref(ctx)))
        self._ctx = ctx
        self.size = lib.hd_size(ctx)
        self.levels = lib.hd_levels(ctx)
        gl = C.c_int(0)
        bnd = (C.c_int * 65)()
        self.slabs = lib.hd_slab_info(ctx, C.byref(gl), bnd) if slabs else 0
        self.slab_gather_level = gl.value if self.slabs else None
        self.slab_bounds = [bnd[i] for i in range(self.slabs + 1)] if self.slabs else None

    def close(self):
        if getattr(self, "_ctx", None):
            self._lib.hd_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _result(self, rep: HdReport, x, res):
        return GmresResult(x, rep.iterations, bool(rep.converged), list(res[:max(rep.iterations, 1)])
                           if rep.iterations or rep.converged else [],
                           OperationCounts(rep.matvecs, rep.coarse_solves, rep.shift_solves, rep.vcycles),
                           rep.t_setup_s, rep.t_solve_s, rep.kernel_launches, rep.library_calls)

    def solve(self, opt: GmresOptions = GmresOptions(), rhs: Optional[np.ndarray] = None) -> GmresResult:
        """Host buffers in/out (hd_solve)."""
        b = np.ascontiguousarray(self.sys.rhs if rhs is None else rhs, dtype=np.complex128)
        x = np.zeros(self.size, dtype=np.complex128)
        res = np.zeros(opt.max_iterations + 1)
        rep = HdReport()
        o = HdGmres(opt.max_iterations, opt.tolerance)
        _check(self._lib.hd_solve(self._ctx, C.byref(o), _dp(b.view(np.float64)), _dp(x.view(np.float64)),
                                  _dp(res), C.byref(rep)))
        return self._result(rep, x, res)

    def solve_device(self, d_rhs_ptr: int, d_x_ptr: int, opt: GmresOptions = GmresOptions()) -> GmresResult:
        """Device-resident rhs / x (hd_solve_device); pointers are raw CUDA addresses."""
        res = np.zeros(opt.max_iterations + 1)
        rep = HdReport()
        o = HdGmres(opt.max_iterations, opt.tolerance)
        _check(self._lib.hd_solve_device(self._ctx, C.byref(o), C.c_void_p(d_rhs_ptr), C.c_void_p(d_x_ptr),
                                         _dp(res), C.byref(rep)))
        return self._result(rep, None, res)

    def set_stream(self, stream_handle: int):
        """Run on an external cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream); 0 = own stream."""
        _check(self._lib.hd_set_stream(self._ctx, C.c_void_p(stream_handle or None)))

    def profile(self, enable: bool = True):
        """Enable per-launch CUDA-event timing of subsequent solves (clears old records)."""
        _check(self._lib.hd_profile(self._ctx, int(enable)))

    def profile_read(self) -> dict:
        """{kind: (launches, ms, algorithmic_bytes)} of the profiled solves."""
        out = {}
        for i, name in enumerate(KERNEL_KINDS):
            n, ms, b = C.c_long(), C.c_double(), C.c_double()
            _check(self._lib.hd_profile_read(self._ctx, i, C.byref(n), C.byref(ms), C.byref(b)))
            if n.value:
                out[name] = (n.value, ms.value, b.value)
        return out

    def debug_level(self, which: int, level: int, d_x_ptr: int, d_y_ptr: int):
        """Test hook on one multigrid level (see hd_debug_level in include/helmdef_b200.h)."""
        _check(self._lib.hd_debug_level(self._ctx, which, level, C.c_void_p(d_x_ptr), C.c_void_p(d_y_ptr)))

    def level_size(self, level: int) -> int:
        return self._lib.hd_level_size(self._ctx, level)

    def apply(self, which: int, d_x_ptr: int, d_y_ptr: int):
        """Test hook: y = A x | M x | MG^-1 x | P x | op(x) | Q x on device pointers."""
        _check(self._lib.hd_apply(self._ctx, which, C.c_void_p(d_x_ptr), C.c_void_p(d_y_ptr)))


def run_cell(problem: str, tag: str, order: int, k: float, elements: int, opt: GmresOptions = GmresOptions(),
             **spec_kw):
    """run_cell (src/harness.cpp:207-243): assemble -> compose -> gmres -> record."""
    t0 = time.perf_counter()
    factories = {"point_source_1d": point_source_1d, "point_source_2d": point_source_2d,
                 "layered_medium_2d": layered_medium_2d}
    sys_ = assemble(factories[problem](elements, order, k))
    spec = to_spec(tag, order, k, **spec_kw)
    with Solver(sys_, spec) as s:
        r = s.solve(opt)
    cyc = spec_kw.get("cycles", 1)
    rec = dict(problem=problem, tag=f"{tag}^{cyc}" if tag in ("DC_MG", "Deps_C_MG") else tag, k=k, p=order,
               elements=elements, dofs=sys_.size, iterations=r.iterations, converged=r.converged,
               residual=r.residuals[-1] if r.residuals else 0.0, matvecs=r.counts.matvecs,
               shift_solves=r.counts.shift_solves, vcycles=r.counts.vcycles, coarse_solves=r.counts.coarse_solves,
               seconds=time.perf_counter() - t0)
    return rec, r, sys_
