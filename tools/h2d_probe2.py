"""Raw pinned H2D bandwidth for the C3 log-likelihoods (5.84 GB): chunk size x copy streams."""
import torch, time
T, B, P = 500, 512, 5700
h = torch.empty((T, B, P), dtype=torch.float32, pin_memory=True)
d = torch.empty((100, B, P), dtype=torch.float32, device='cuda')
for ch in (10, 25, 50):
    for ns in (1, 2, 4):
        ss = [torch.cuda.Stream() for _ in range(ns)]
        best = 0
        for rep in range(3):
            torch.cuda.synchronize(); a = time.perf_counter()
            for k, t0 in enumerate(range(0, T, ch)):
                with torch.cuda.stream(ss[k % ns]):
                    o = (k % (100 // ch)) * ch
                    d[o:o + ch].copy_(h[t0:t0 + ch], non_blocking=True)
            torch.cuda.synchronize(); b = time.perf_counter()
            best = max(best, h.numel() * 4 / (b - a) / 1e9)
        print(f"chunk {ch} frames ({ch*B*P*4/1e6:.0f} MB), {ns} stream(s): {best:.1f} GB/s", flush=True)
