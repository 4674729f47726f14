"""Per-frame claim / survivor distribution of C3 on the GPU (diagnostic)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import bench
from paper_1910_10032_b200 import build, wfst_gpu as W
build.build()
cfg, preset = (sys.argv[1] if len(sys.argv) > 1 else "c3"), (sys.argv[2] if len(sys.argv) > 2 else "clean")
wl = bench.make_workload(cfg, preset)
G = W.Graph.from_arrays(wl["graph"])
D = W.Decoder(G, wl["B"], wl["beam"], wl["alpha"])
ll = bench.device_loglikes(W, torch, wl, "cuda:0")
D.reset(); D.decode_frames(ll); torch.cuda.synchronize()
cl, sv, arcs, alpha = [], [], [], []
for b in range(0, wl["B"], max(1, wl["B"] // 16)):
    fs, fc = D.frame_stats(b)
    cl.append(fc[:, 0]); sv.append(fc[:, 2]); arcs.append(fc[:, 3]); alpha.append(np.isfinite(fs[:, 2]))
cl, sv, arcs, alpha = map(np.concatenate, (cl, sv, arcs, alpha))
q = [50, 90, 99, 99.9, 100]
print("claims pct", dict(zip(q, np.percentile(cl, q).round())))
print("claims in alpha frames pct", dict(zip(q, np.percentile(cl[alpha], q).round())) if alpha.any() else None)
print("survivors pct", dict(zip(q, np.percentile(sv, q).round())))
print("arcs pct", dict(zip(q, np.percentile(arcs, q).round())))
print("frac frames claims>12000", float((cl > 12000).mean()), "alpha frames", float(alpha.mean()))
print("stats", D.stats())
