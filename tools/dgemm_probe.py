import torch, time
for n, k in ((93312, 540), (25920, 540), (31104*3, 1080)):
    A = torch.randn(n, n, dtype=torch.float64, device="cuda") if n*n*8 < 80e9 else None
    X = torch.randn(n, k, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    for _ in range(2): Y = A @ X
    torch.cuda.synchronize()
    t = time.time(); reps = 5
    for _ in range(reps): Y = A @ X
    torch.cuda.synchronize()
    dt = (time.time() - t) / reps
    print(n, k, "%.1f ms  %.1f TFLOP/s" % (dt * 1e3, 2 * n * n * k / dt / 1e12), flush=True)
    del A, X, Y
    torch.cuda.empty_cache()
