"""C5: per-call split of wfst_get_partial_paths into GPU time (events bracketing the call after a
sync, so only the partial kernel + its D2H are inside) and host time of the Python wrapper."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1910_10032_b200 import wfst_gpu as W

wl = bench.make_workload(sys.argv[1] if len(sys.argv) > 1 else "c5", "clean")
T, B = wl["T"], wl["B"]
G = W.Graph.from_arrays(wl["graph"])
D = W.Decoder(G, B, wl["beam"], wl["alpha"])
ll = bench.device_loglikes(W, torch, wl, "cuda:0")
E = lambda: torch.cuda.Event(enable_timing=True)
for rep in range(2):
    D.reset()
    tot_gpu, tot_wall = 0.0, 0.0
    for t0 in range(0, T, 50):
        D.decode_frames(ll[t0:t0 + 50])
        torch.cuda.synchronize()
        e1, e2 = E(), E()
        e1.record()
        h0 = time.perf_counter()
        pp = D.partial_paths()
        tot_wall += time.perf_counter() - h0
        e2.record()
        torch.cuda.synchronize()
        tot_gpu += e1.elapsed_time(e2)
    print(f"rep {rep}: partial calls (10): events {tot_gpu:.1f} ms, wall {tot_wall*1e3:.1f} ms", flush=True)
