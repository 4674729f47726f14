"""Time wfst_get_partial_paths on C5 (4096 streams) after each 50-frame chunk."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1910_10032_b200 import wfst_gpu as W

wl = bench.make_workload("c5", "clean")
T, B = wl["T"], wl["B"]
G = W.Graph.from_arrays(wl["graph"])
D = W.Decoder(G, B, wl["beam"], wl["alpha"])
ll = bench.device_loglikes(W, torch, wl, "cuda:0")
D.reset()
for cap in (2064, 512, 64):
    D.reset()
    tot_dec, tot_pp, n_arcs, settled = 0.0, 0.0, 0, None
    for t0 in range(0, T, 50):
        torch.cuda.synchronize(); a = time.perf_counter()
        D.decode_frames(ll[t0:t0 + 50]); torch.cuda.synchronize(); b = time.perf_counter()
        pp = D.partial_paths(cap=cap); c = time.perf_counter()
        tot_dec += b - a; tot_pp += c - b
        n_arcs += sum(len(x) for x in pp["arcs"]); settled = pp["settled_frames"]
    print(f"cap {cap}: decode {tot_dec*1e3:.1f} ms, partial {tot_pp*1e3:.1f} ms over 10 calls, "
          f"arcs/stream {n_arcs/B:.1f}, settled frames min/median {settled.min()}/{int(sorted(settled)[B//2])} of {T}")
