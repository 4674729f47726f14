"""How far the settled prefix trails the newest frame (row f2), per 50-frame chunk, on C5's graph
with `--preset`: settled frames min/median/max, and the records each stream must keep (unsettled
window) -- the quantity traceback reclamation bounds.  Usage: settle_probe.py <preset> <streams>"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1910_10032_b200 import wfst_gpu as W  # noqa: E402

preset = sys.argv[1] if len(sys.argv) > 1 else "other"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 256
wl = bench.make_workload("c5", preset, 0, 1, None, None)
T = wl["T"]
G = W.Graph.from_arrays(wl["graph"])
D = W.Decoder(G, B, wl["beam"], wl["alpha"], reclaim=1, records_per_stream=6_000_000, max_frames=1024)
ll = bench.device_loglikes(W, torch, wl, "cuda:0")[:, :B].contiguous()
D.reset()
for t0 in range(0, T, 50):
    D.decode_frames(ll[t0:t0 + 50].contiguous())
    pp = D.partial_paths(cap=4096)
    s = np.asarray(pp["settled_frames"])
    lag = (t0 + 50) - s
    print(f"after {t0 + 50:3d} frames: settled min/med/max {s.min()}/{int(np.median(s))}/{s.max()}  "
          f"lag med/max {int(np.median(lag))}/{lag.max()}  records_used_max {D.stats()['records_used_max']}", flush=True)
