"""Small decodes for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
C1 (20 states, infinite beam), a 20k-state C2-shaped graph with max-active binding, the lattice
and partial-result kernels, and an epsilon-general (permuted, backward epsilon arcs) graph.
Run: compute-sanitizer --tool <t> python tools/sanitize_driver.py"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1910_10032_b200 import inputs as I  # noqa: E402
from paper_1910_10032_b200 import wfst_gpu as W  # noqa: E402


def run(g, T, B, P, beam, alpha, preset="clean", **opts):
    pl = I.planted_walks(g, B, T, seed=3)
    ll = torch.from_numpy(I.loglikes(4, range(B), T, P, pl, **I.preset(preset))).cuda()
    G = W.Graph.from_arrays(g)
    D = W.Decoder(G, B, beam, alpha, **opts)
    D.reset()
    D.decode_frames(ll[: T // 2].contiguous())
    if opts.get("reclaim") or not opts.get("lattice"):
        D.partial_paths()
    D.decode_frames(ll[T // 2:].contiguous())
    res = D.best_paths(cap=4 * T + 64, raise_on_error=False)
    if opts.get("lattice"):
        D.lattice(0)
    D.sync()
    print("ok", g.n_states, B, T, int(res["rc"]), flush=True)


def run_chunks(g, T, B, P, beam, alpha, chunk, **opts):   # partial results after every chunk
    pl = I.planted_walks(g, B, T, seed=5)
    ll = torch.from_numpy(I.loglikes(6, range(B), T, P, pl, **I.preset("clean"))).cuda()
    D = W.Decoder(W.Graph.from_arrays(g), B, beam, alpha, **opts)
    D.reset()
    for t0 in range(0, T, chunk):
        D.decode_frames(ll[t0:t0 + chunk].contiguous())
        D.partial_paths(cap=8)   # small cap: the over-capacity path too
    D.sync()
    print("ok chunks", g.n_states, B, T, flush=True)


which = sys.argv[1] if len(sys.argv) > 1 else "all"
c1 = I.c1_graph()
c2s = I.hclg_graph(20000, 6.0, 400, seed=2)
if which in ("all", "c1"):
    run(c1, 30, 1, 10, float("inf"), 0, preset=dict(sigma=1.5, boost=2.0))
if which in ("all", "c2"):
    run(c2s, 12, 6, 400, 10.0, 300, preset="other")
    run(c2s, 12, 4, 400, 10.0, 300, threads=256, ctas_per_sm=2, table_slots=512, overflow_slots=4096)
if which in ("all", "lat"):
    run(c2s, 8, 3, 400, 10.0, 300, lattice=1, lattice_beam=6.0)
if which in ("all", "gc"):   # traceback GC (gc_kernel) with partial results and reclaim
    run(c2s, 12, 4, 400, 10.0, 300, gc_frames=3)
    run(c2s, 12, 3, 400, 10.0, 300, gc_frames=4, reclaim=1)
if which in ("all", "partial"):
    run_chunks(c2s, 24, 5, 400, 10.0, 300, 4)
    run_chunks(c2s, 24, 3, 400, 10.0, 300, 5, reclaim=1)
if which in ("all", "eps") and hasattr(I, "hclg_graph_eps"):
    run(I.hclg_graph_eps(20000, 5.0, 400, seed=6), 12, 4, 400, 10.0, 300)
print("done", flush=True)
