import torch, time
for n, m, k in [(8192, 8192, 8192), (800, 1600, 800), (1600, 1600, 1600)]:
    a = torch.randn(n, k, dtype=torch.float64, device="cuda")
    b = torch.randn(k, m, dtype=torch.float64, device="cuda")
    for _ in range(3):
        c = a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5 if n > 4000 else 50
    e0.record()
    for _ in range(reps):
        c = a @ b
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps * 1e-3
    print(f"DGEMM {n}x{m}x{k}: {2*n*m*k/t/1e12:.1f} TFLOP/s ({t*1e6:.1f} us)")
