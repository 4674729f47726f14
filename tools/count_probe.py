"""Instrumented run (library built with -DWFST_COUNT): per stream-frame averages of arcs,
claims, survivors, and the share of frame cycles spent in frames where max-active binds."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1910_10032_b200 import wfst_gpu as W

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
preset = sys.argv[2] if len(sys.argv) > 2 else "clean"
wl = bench.make_workload(cfg, preset, 0, 1, None, None)
G = W.Graph.from_arrays(wl["graph"])
D = W.Decoder(G, wl["B"], wl["beam"], wl["alpha"])
ll = bench.device_loglikes(W, torch, wl, "cuda:0")
D.reset(); D.decode_frames(ll); torch.cuda.synchronize()
st = D.stats()
f = st["frames"]
ph = st["phase_cycles"]
print(json.dumps({"config": cfg, "preset": preset, "frames": f,
                  "arcs": st["emit_arcs"] / f, "alpha_frame_claims_above_kalpha_le2": ph["map_build"] / max(1, st["alpha_frames"]),
                  "alpha_frame_claims_above_kalpha_gt2": ph["eps_backptr"] / max(1, st["alpha_frames"]),
                  "claims": st["candidates"] / f, "survivors": st["survivors"] / f,
                  "ovf": st["overflow_inserts"] / f, "alpha_frames": st["alpha_frames"] / f}))
