"""Time cuFFT (via torch.fft, fp64) 3D real transforms for candidate mid-grid sizes.
Prints ms per forward+inverse pair; used to pick FFT-friendly sizes in the plan rule."""
import sys, time, torch

def timeit(f, n=5):
    for _ in range(2): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n

shapes = [(1200, 600, 600), (1152, 576, 576), (1200, 576, 576), (1024, 600, 600), (1024, 640, 640), (1280, 640, 640),
          (1250, 625, 625), (1296, 648, 648), (1120, 560, 560), (1176, 588, 588), (1200, 640, 640), (1152, 600, 600),
          (1344, 672, 672), (1024, 576, 576), (1000, 600, 600), (1152, 640, 640), (1280, 600, 600), (1200, 608, 608)]
for s in shapes:
    x = torch.randn(s, dtype=torch.float64, device="cuda")
    X = torch.fft.rfftn(x)
    tf = timeit(lambda: torch.fft.rfftn(x))
    ti = timeit(lambda: torch.fft.irfftn(X, s=s))
    pts = s[0] * s[1] * s[2]
    print(f"{s}: fwd {tf:7.2f} ms inv {ti:7.2f} ms  ns/pt {1e6*(tf+ti)/pts:.3f}", flush=True)
    del x, X
    torch.cuda.empty_cache()
# 2D-per-plane + 1D-z split with only the nonzero planes transformed in 2D
for (Z, X_, Y, nz) in [(1200, 600, 600, 620)]:
    x = torch.zeros((Z, X_, Y), dtype=torch.float64, device="cuda")
    x[:nz].normal_()
    def split():
        a = torch.fft.rfft2(x[:nz])                     # (nz, X, Y/2+1)
        b = torch.zeros((Z,) + a.shape[1:], dtype=a.dtype, device="cuda")
        b[:nz] = a
        return torch.fft.fft(b, dim=0)
    print("split 2D+1D (torch, incl. copies):", timeit(split), "ms")
