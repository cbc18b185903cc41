"""Sensitivity envelope of the C5 residual history (run from the repo root).

Runs the oracle's C5 solve a second time with the Arnoldi orthogonalisation in
its one-reduction inverse-compact-WY form (algebraically identical to MGS,
different rounding) and records |r_mgs(j) - r_icwy(j)| per iteration.  This is
the rounding sensitivity of the method itself: two exact CPU implementations
disagree by this much, so the device may too.  Writes C5_envelope.json.
"""
import json
import math
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import helmdef_oracle as O  # noqa: E402


def gmres_icwy(op, rhs, start, monitor, maxit=100, tol=1e-7):
    x0 = start.copy()
    r0 = monitor(x0)
    if r0 <= tol:
        return [r0]
    r = rhs - op(x0)
    beta = np.linalg.norm(r)
    U, sig = [r], [1 / beta]
    H = np.zeros((maxit + 1, maxit), complex)
    g = np.zeros(maxit + 1, complex)
    g[0] = beta
    cs = np.zeros(maxit, complex)
    sn = np.zeros(maxit, complex)
    L = np.zeros((maxit + 1, maxit + 1), complex)
    res = []
    for j in range(maxit):
        wraw = op(U[j])
        s = np.array([np.vdot(U[i], wraw) for i in range(j + 1)]) * np.array(sig[:j + 1]) * sig[j]
        for l in range(j):
            L[j, l] = np.vdot(U[j], U[l]) * sig[j] * sig[l]
        h = np.zeros(j + 1, complex)
        for i in range(j + 1):
            h[i] = s[i] - sum(L[i, l] * h[l] for l in range(i))
        w = sig[j] * wraw
        for i in range(j + 1):
            w = w - (h[i] * sig[i]) * U[i]
        hnew = np.linalg.norm(w)
        H[:j + 1, j] = h
        H[j + 1, j] = hnew
        for i in range(j):
            t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
            H[i + 1, j] = -np.conj(sn[i]) * H[i, j] + np.conj(cs[i]) * H[i + 1, j]
            H[i, j] = t
        d = math.sqrt(abs(H[j, j]) ** 2 + abs(H[j + 1, j]) ** 2)
        cs[j], sn[j] = np.conj(H[j, j]) / d, np.conj(H[j + 1, j]) / d
        H[j, j] = cs[j] * H[j, j] + sn[j] * H[j + 1, j]
        H[j + 1, j] = 0
        g[j + 1] = -np.conj(sn[j]) * g[j]
        g[j] = cs[j] * g[j]
        m = j + 1
        y = np.zeros(m, complex)
        for i in range(m - 1, -1, -1):
            y[i] = (g[i] - sum(H[i, l] * y[l] for l in range(i + 1, m))) / H[i, i]
        x = x0 + sum((y[i] * sig[i]) * U[i] for i in range(m))
        rr = monitor(x)
        res.append(rr)
        print(j, rr, flush=True)
        if rr <= tol:
            break
        U.append(w)
        sig.append(1 / hnew)
    return res


if __name__ == "__main__":
    ref = json.loads((Path(__file__).resolve().parent / "C5_oracle.json").read_text())
    p, ne, k = 3, 1600, 1000.0
    spec = O.to_spec("DC_MG", p, k, beta2="0.5", cycles=1, smoothing=1, omega=2.0 / 3.0)
    s = O.assemble(O.point_source_2d(ne, p, k))
    st = O.compose(s, spec, galerkin="kron", e_solver="fd")
    res = gmres_icwy(st.op, st.rhs, st.start, st.monitor)
    m = min(len(res), len(ref["residuals"]))
    env = [abs(a - b) for a, b in zip(res[:m], ref["residuals"][:m])]
    out = dict(config="C5", residuals_icwy=res, iterations_icwy=len(res), envelope=env,
               note="|r_MGS(j) - r_ICWY(j)| of two exact CPU implementations (oracle)")
    (Path(__file__).resolve().parent / "C5_envelope.json").write_text(json.dumps(out, indent=1))
    print("iterations", len(res), "max env", max(env))
