"""cuBLAS DGEMM (torch float64 matmul / bmm) at the Schur-update shapes of the top levels,
for comparison with large_update_kernel<1> (which does the lower triangle only)."""
import torch
def t(f, reps=10):
    for _ in range(3): f()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best
for (b, n, k) in [(128, 1535, 256), (64, 2047, 512), (32, 3071, 512), (16, 4095, 256), (16, 4095, 1024),
                  (8, 5120, 256), (4, 4097, 256), (1, 4096, 256), (1, 8192, 256)]:
    a = torch.randn(b, n, k, dtype=torch.float64, device="cuda")
    c = torch.randn(b, n, n, dtype=torch.float64, device="cuda")
    at = a.transpose(1, 2)
    ms = t(lambda: torch.baddbmm(c, a, at, alpha=-1.0, out=c))
    print(f"batch {b:4d} n {n:5d} k {k:5d}: {ms:8.3f} ms  {2*b*n*n*k/ms/1e9:6.2f} TF/s (full)  "
          f"syrk-equivalent time {ms/2:.3f} ms")
