"""C5 (4096 streams, 50-frame chunks): split the cost of settled partial results per chunk into
the partial kernel's GPU time, the host's share of the call, and the GPU idle gap it leaves."""
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
    torch.cuda.synchronize()
    dec, part, host, wall = 0.0, 0.0, 0.0, 0.0
    w0 = time.perf_counter()
    for t0 in range(0, T, 50):
        e0, e1, e2 = E(), E(), E()
        e0.record()
        D.decode_frames(ll[t0:t0 + 50])
        e1.record()
        h0 = time.perf_counter()
        pp = D.partial_paths()
        host += time.perf_counter() - h0
        e2.record()
        torch.cuda.synchronize()
        dec += e0.elapsed_time(e1)
        part += e1.elapsed_time(e2)
    wall = time.perf_counter() - w0
    # the same without partial results
    D.reset()
    torch.cuda.synchronize()
    f0, f1 = E(), E()
    f0.record()
    for t0 in range(0, T, 50):
        D.decode_frames(ll[t0:t0 + 50])
    f1.record()
    torch.cuda.synchronize()
    print(f"rep {rep}: decode {dec:.1f} ms + partial (GPU, e1->e2) {part:.1f} ms (host in the call {host*1e3:.1f} ms); "
          f"wall {wall*1e3:.1f} ms; decode-only run {f0.elapsed_time(f1):.1f} ms", flush=True)
