"""Per-frame SM cycles vs frame shape (library built with -DWFST_FRAMECYC; diagnostic only).
Prints the share of frame cycles and frames by claim-count bucket, alpha-bound or not."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1910_10032_b200 import wfst_gpu as W  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
preset = sys.argv[2] if len(sys.argv) > 2 else "clean"
wl = bench.make_workload(cfg, preset, 0, 1, None, None)
G = W.Graph.from_arrays(wl["graph"])
D = W.Decoder(G, wl["B"], wl["beam"], wl["alpha"])
ll = bench.device_loglikes(W, torch, wl, "cuda:0")
for _ in range(2):
    D.reset(); D.decode_frames(ll); torch.cuda.synchronize()
rows = []
for b in range(0, wl["B"], max(1, wl["B"] // 64)):
    fs, fc = D.frame_stats(b)
    te = fc[:, 1].astype(np.uint64)
    rows.append(np.column_stack([fc[:, 0], fc[:, 2], fc[:, 3], np.isfinite(fs[:, 2]), fc[:, 4],
                                 (te & np.uint64(0xFFFFFFFF)).astype(np.float64), (te >> np.uint64(32)).astype(np.float64)]))
R = np.concatenate(rows).astype(np.float64)
cl, sv, arcs, al, cyc, t_exp, t_eps = R.T
tot = cyc.sum()
print(f"frames {len(cyc)}  mean cycles {cyc.mean():.0f}  alpha frames {al.mean():.3f} share {cyc[al > 0].sum() / tot:.3f}")
edges = [0, 300, 1000, 2000, 4000, 7000, 10000, 13000, 20000, 1e9]
print("claims bucket | frames | cycle share | mean cycles | to end of expansion | expansion end -> closure end | rest | mean surv | mean arcs | alpha frac")
for lo, hi in zip(edges[:-1], edges[1:]):
    m = (cl >= lo) & (cl < hi)
    if m.any():
        print(f"[{lo:.0f},{hi:.0f}) | {m.mean():.3f} | {cyc[m].sum() / tot:.3f} | {cyc[m].mean():.0f} | "
              f"{t_exp[m].mean():.0f} | {(t_eps - t_exp)[m].mean():.0f} | {(cyc - t_eps)[m].mean():.0f} | "
              f"{sv[m].mean():.0f} | {arcs[m].mean():.0f} | {al[m].mean():.2f}")
        if lo == 0:   # the tiny frames: with / without the unigram hub's arcs
            for name, mm in (("  tiny, hub expanded", m & (arcs >= 15000)), ("  tiny, no hub", m & (arcs < 15000))):
                if mm.any():
                    print(f"{name} | {mm.mean():.3f} | {cyc[mm].sum() / tot:.3f} | {cyc[mm].mean():.0f} | "
                          f"{t_exp[mm].mean():.0f} | {(t_eps - t_exp)[mm].mean():.0f} | {(cyc - t_eps)[mm].mean():.0f} | "
                          f"{sv[mm].mean():.0f} | {arcs[mm].mean():.0f} |")
# cycles per claim / per arc fit (least squares, all frames)
A = np.column_stack([np.ones_like(cl), cl, arcs, sv])
coef = np.linalg.lstsq(A, cyc, rcond=None)[0]
print("fit cycles = %.0f + %.2f*claims + %.3f*arcs + %.2f*survivors" % tuple(coef))
