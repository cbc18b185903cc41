"""GPU diagnostics: component-wise and end-to-end parity against the oracle,
printed rather than asserted (one gpurun call gives the whole picture)."""
import sys
import time
import traceback
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2010_10232_b200 as hd  # noqa: E402
from oracle import helmdef_oracle as O  # noqa: E402


def dev(v):
    return torch.from_numpy(np.ascontiguousarray(v)).to("cuda")


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def components(dim, p, ne, k, tag="DC_MG", beta2="0.5", omega=2 / 3, cycles=1, smoothing=1, eps=0.1):
    pb = hd.point_source_2d(ne, p, k) if dim == 2 else hd.point_source_1d(ne, p, k)
    sysg = hd.assemble(pb)
    spec = hd.to_spec(tag, p, k, epsilon=eps, beta2=beta2, cycles=cycles, smoothing=smoothing, omega=omega)
    so = O.assemble(O.point_source_2d(ne, p, k) if dim == 2 else O.point_source_1d(ne, p, k))
    ospec = O.to_spec(tag, p, k, epsilon=eps, beta2=beta2, cycles=cycles, smoothing=smoothing, omega=omega)
    gal, es = ("kron", "fd") if dim == 2 else ("sparse", "splu")
    st = O.compose(so, ospec, galerkin=gal, e_solver=es)
    rng = np.random.default_rng(12345)
    N = sysg.size
    v = rng.uniform(-1, 1, N) + 1j * rng.uniform(-1, 1, N)
    out = {}
    with hd.Solver(sysg, spec) as s:
        xd = dev(v)
        yd = torch.zeros_like(xd)
        checks = [("A", hd.HD_APPLY_A, lambda: so.A @ v),
                  ("shifted", hd.HD_APPLY_SHIFTED, lambda: O.shifted_operator(so, ospec.beta2) @ v)]
        if spec.shift:
            checks.append(("MG", hd.HD_APPLY_MG, lambda: st.multigrid.solve(v, ospec.cycles)))
        if spec.deflate:
            checks.append(("Q", hd.HD_APPLY_Q, lambda: st.deflation.apply_Q(v)))
            checks.append(("project", hd.HD_APPLY_PROJECT, lambda: st.deflation.project(v)))
        checks.append(("op", hd.HD_APPLY_OP, lambda: st.op(v)))
        for name, which, ref in checks:
            s.apply(which, xd.data_ptr(), yd.data_ptr())
            torch.cuda.synchronize()
            out[name] = rel(yd.cpu().numpy(), ref())
        print(f"  levels gpu={s.levels} oracle={st.multigrid.levels() if st.multigrid else 0}")
    return out


def solve(dim, p, ne, k, tag="DC_MG", beta2="0.5", omega=2 / 3, cycles=1, smoothing=1, eps=0.1, oracle=True,
          maxit=100):
    pb = hd.point_source_2d(ne, p, k) if dim == 2 else hd.point_source_1d(ne, p, k)
    sysg = hd.assemble(pb)
    spec = hd.to_spec(tag, p, k, epsilon=eps, beta2=beta2, cycles=cycles, smoothing=smoothing, omega=omega)
    opt = hd.GmresOptions(maxit, 1e-7)
    with hd.Solver(sysg, spec) as s:
        r = s.solve(opt)
        r2 = s.solve(opt)
    line = (f"  gpu: it={r.iterations} conv={r.converged} t_setup={r.t_setup:.3f}s t_solve={r.t_solve*1e3:.2f}ms "
            f"(2nd {r2.t_solve*1e3:.2f}ms) launches={r.kernel_launches} counts={r.counts}")
    print(line)
    if oracle:
        so = O.assemble(O.point_source_2d(ne, p, k) if dim == 2 else O.point_source_1d(ne, p, k))
        ospec = O.to_spec(tag, p, k, epsilon=eps, beta2=beta2, cycles=cycles, smoothing=smoothing, omega=omega)
        gal, es = ("kron", "fd") if dim == 2 else ("sparse", "splu")
        t = time.perf_counter()
        st = O.compose(so, ospec, galerkin=gal, e_solver=es)
        g = O.gmres(st.op, st.rhs, st.start, st.monitor, O.GmresOptions(maxit, 1e-7))
        t = time.perf_counter() - t
        m = min(len(g.residuals), len(r.residuals))
        dres = np.abs(np.array(g.residuals[:m]) - np.array(r.residuals[:m]))
        print(f"  oracle: it={g.iterations} conv={g.converged} ({t:.2f}s) counts={st.counts}")
        print(f"  |d res| max={dres.max():.3e} first>1e-10 at {int(np.argmax(dres > 1e-10)) if (dres > 1e-10).any() else -1}"
              f" rel L2(x)={rel(r.solution, g.solution):.3e}  rerun-identical={np.array_equal(r.solution, r2.solution)}")
        print("  gpu res:", ["%.6e" % x for x in r.residuals])
        print("  ora res:", ["%.6e" % x for x in g.residuals])


def main():
    torch.cuda.init()
    print(torch.cuda.get_device_name(0))
    cases = [
        ("C1 1D p2 k50 80el", (1, 2, 80, 50), {}),
        ("1D p4 k200", (1, 4, 317, 200), {}),
        ("2D p2 k20 40el", (2, 2, 40, 20), {}),
        ("2D p3 k40 64el", (2, 3, 64, 40), {}),
        ("2D p2 k40 64el nu2 cycles2 eps", (2, 2, 64, 40), dict(tag="Deps_C_MG", cycles=2, smoothing=2)),
    ]
    for name, a, kw in cases:
        print(name)
        try:
            print("  components:", {k: f"{v:.2e}" for k, v in components(*a, **kw).items()})
            solve(*a, **kw)
        except Exception:
            traceback.print_exc()
    for name, a, kw in [("C3 2D p2 k200 320el", (2, 2, 320, 200), {}),
                        ("C2 1D p4 k1000 31623el", (1, 4, 31623, 1000), {}),
                        ("table4 1D DC_MG^1 p3 k1000", (1, 3, O.derived_elements(1000, 0.625, 3), 1000),
                         dict(beta2="1", omega=0.6))]:
        print(name)
        try:
            solve(*a, **kw)
        except Exception:
            traceback.print_exc()
    print("C5 2D p3 k1000 1600el (no oracle)")
    try:
        solve(2, 3, 1600, 1000, oracle=False)
    except Exception:
        traceback.print_exc()




def mg_debug(dim, p, ne, k, beta2="0.5", omega=2 / 3):
    pb = hd.point_source_2d(ne, p, k) if dim == 2 else hd.point_source_1d(ne, p, k)
    sysg = hd.assemble(pb)
    spec = hd.to_spec("DC_MG", p, k, beta2=beta2, omega=omega)
    so = O.assemble(O.point_source_2d(ne, p, k) if dim == 2 else O.point_source_1d(ne, p, k))
    ospec = O.to_spec("DC_MG", p, k, beta2=beta2, omega=omega)
    st = O.compose(so, ospec, galerkin="kron" if dim == 2 else "sparse", e_solver="fd" if dim == 2 else "splu")
    mg = st.multigrid
    rng = np.random.default_rng(7)
    with hd.Solver(sysg, spec) as s:
        for l in range(s.levels):
            n = s.level_size(l)
            NL = n ** dim
            v = rng.uniform(-1, 1, NL) + 1j * rng.uniform(-1, 1, NL)
            xd = dev(v)
            M = mg.mats[l]
            dinv = mg.inv_diag[l]
            refs = {0: M @ v, 1: omega * dinv * v, 2: v + omega * dinv * (v - M @ v), 3: v - M @ v}
            if l + 1 < s.levels:
                refs[4] = mg.transT[l] @ v
            if l == s.levels - 1:
                refs[6] = mg.coarse.solve(v)
            res = {}
            for which, ref in refs.items():
                yd = torch.zeros(len(ref), dtype=torch.complex128, device="cuda")
                s.debug_level(which, l, xd.data_ptr(), yd.data_ptr())
                res[which] = rel(yd.cpu().numpy(), ref)
            if l + 1 < s.levels:
                nc = s.level_size(l + 1) ** dim
                e = rng.uniform(-1, 1, nc) + 1j * rng.uniform(-1, 1, nc)
                yd = torch.zeros(NL, dtype=torch.complex128, device="cuda")
                s.debug_level(5, l, dev(e).data_ptr(), yd.data_ptr())
                res[5] = rel(yd.cpu().numpy(), mg.trans[l] @ e)
            print(f"  level {l} n={n}:", {k: f"{v:.2e}" for k, v in sorted(res.items())})


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "mg":
        for a in [(2, 2, 40, 20), (2, 3, 64, 40), (1, 2, 80, 50)]:
            print("mg_debug", a)
            try:
                mg_debug(*a)
            except Exception:
                traceback.print_exc()
    else:
        main()
