import torch, time
M = 640 * 321
for L in (1250, 1260, 1280, 1296, 1344, 1350, 1372, 1400):
    x = torch.randn(M, L, dtype=torch.complex128, device="cuda")
    for _ in range(3): y = torch.fft.fft(x, dim=1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): y = torch.fft.fft(x, dim=1)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(L, "%.3f ms" % ms, "%.3f ns/pt" % (ms * 1e6 / (M * L)))
    del x, y
