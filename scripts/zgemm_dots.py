"""Bandwidth of the Arnoldi pass-1 shape as a cuBLAS ZGEMM: U^H [w, u_j] with U = N x (j+1)."""
import torch
N = 2563201
for j in (10, 40, 77):
    U = torch.randn(j + 1, N, dtype=torch.complex128, device="cuda")  # rows = basis vectors (contiguous)
    W = torch.randn(2, N, dtype=torch.complex128, device="cuda")
    for _ in range(3):
        R = torch.matmul(U.conj(), W.T)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        R = torch.matmul(U.conj(), W.T)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    gb = (j + 3) * N * 16 / 1e9
    print(f"j={j}: {ms*1e3:.1f} us, {gb/ms*1e3/1e3:.2f} TB/s ({gb:.2f} GB)")
