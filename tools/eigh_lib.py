"""Library context for the PSD projection: torch.linalg.eigh (cuSOLVER syevd) on the same FP64 block sizes."""
import sys
import torch

for N in [int(x) for x in (sys.argv[1:] or ["861", "325", "285", "231"])]:
    g = torch.Generator(device="cuda").manual_seed(N)
    G = torch.randn(N, N, dtype=torch.float64, device="cuda", generator=g)
    A = G + G.T
    for _ in range(3):
        w, V = torch.linalg.eigh(A)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    e0.record()
    for _ in range(reps):
        w, V = torch.linalg.eigh(A)
        P = (V * w.clamp(min=0)) @ V.T
    e1.record()
    torch.cuda.synchronize()
    print(f"N={N}: torch.linalg.eigh + reconstruction {e0.elapsed_time(e1) / reps:.3f} ms per projection")
