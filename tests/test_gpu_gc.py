"""Traceback GC by live-set compaction (opts.gc_frames; csrc/gc_kernel.cuh).

Collection only drops records that no current survivor's traceback reaches, so every result must
equal the oracle's (and the same decoder's without GC) bit for bit, while a stream's record
high-water mark stays at its live tree plus gc_frames frames of new records."""
import numpy as np
import pytest

from paper_1910_10032_b200 import inputs as I

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def W():
    from paper_1910_10032_b200 import build, wfst_gpu
    build.build()
    return wfst_gpu


@pytest.fixture(scope="module")
def torch():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch


def _check(res, og, ll, beam, alpha, B, tails=None):
    for b in range(B):
        r = og.decode(ll[:, b, :], beam, alpha)
        arcs = list(res["arcs"][b, :res["n_arcs"][b]])
        if tails is not None:
            arcs = tails[b] + arcs
        assert arcs == list(r.arcs), b
        assert res["cost"][b] == r.cost32 and res["reached_final"][b] == r.reached_final, b


@pytest.mark.parametrize("gc,preset,graph", [(1, "clean", "hclg"), (7, "other", "hclg"), (16, "clean", "eps"),
                                             (5, "other", "eps")])
def test_gc_results_unchanged(W, torch, oracle_mod, gc, preset, graph):
    P = 400
    g = (I.hclg_graph(20_000, 6.0, P, seed=3) if graph == "hclg"
         else I.hclg_graph_eps(20_000, 5.0, P, seed=6))
    og = oracle_mod.OracleGraph(g)
    T, B, beam, alpha = 90, 6, 10.0, 300
    pl = I.planted_walks(g, B, T, seed=5)
    ll = I.loglikes(12, range(B), T, P, pl, **I.preset(preset))
    G = W.Graph.from_arrays(g)
    t = torch.from_numpy(ll).cuda()
    D = W.Decoder(G, B, beam, alpha, gc_frames=gc)
    D.reset()
    for t0 in range(0, T, 30):           # several decode calls, each split into gc_frames launches
        D.decode_frames(t[t0:t0 + 30].contiguous())
    res = D.best_paths(cap=4 * T + 64)
    _check(res, og, ll, beam, alpha, B)
    D0 = W.Decoder(G, B, beam, alpha)
    D0.reset()
    D0.decode_frames(t)
    assert D.stats()["records_used_max"] < D0.stats()["records_used_max"]
    # per-frame statistics are untouched by collection
    for b in range(B):
        assert np.array_equal(D.frame_stats(b)[0].view(np.uint32), D0.frame_stats(b)[0].view(np.uint32))


def test_gc_long_stream_small_arena(W, torch, oracle_mod):
    """600 frames with a record arena of 8000 records (~27 frames at the max-active bound of 300):
    with GC every 16 frames the stream fits and its path equals the oracle's; without GC it runs
    out (CAPACITY)."""
    g = I.hclg_graph(3000, 6, 200, seed=4)
    og = oracle_mod.OracleGraph(g)
    T, B, P, beam, alpha = 600, 4, 200, 10.0, 300
    pl = I.planted_walks(g, B, T, seed=9)
    ll = I.loglikes(77, range(B), T, P, pl, 1.0, 4.0)
    G = W.Graph.from_arrays(g)
    t = torch.from_numpy(ll).cuda()
    opts = dict(max_frames=1024, records_per_stream=8000)
    D = W.Decoder(G, B, beam, alpha, gc_frames=16, **opts)
    D.reset()
    D.decode_frames(t)
    res = D.best_paths(cap=4 * T + 64)
    assert res["rc"] == 0
    _check(res, og, ll, beam, alpha, B)
    D2 = W.Decoder(G, B, beam, alpha, **opts)
    D2.reset()
    D2.decode_frames(t)
    assert D2.best_paths(cap=4 * T + 64, raise_on_error=False)["rc"] == 6   # CAPACITY


def test_gc_with_partial_results_and_reclaim(W, torch, oracle_mod):
    """GC between partial-result calls (the settle point's record is remapped by compaction):
    the partial outputs followed by the final tail equal the oracle's path, with and without
    reclaim, on an epsilon-general graph and the host-input path."""
    g = I.hclg_graph_eps(8000, 5.0, 300, seed=2)
    og = oracle_mod.OracleGraph(g)
    T, B, P, beam, alpha = 240, 5, 300, 10.0, 400
    pl = I.planted_walks(g, B, T, seed=3)
    ll = I.loglikes(41, range(B), T, P, pl, 1.0, 4.0)
    G = W.Graph.from_arrays(g)
    for reclaim in (0, 1):
        D = W.Decoder(G, B, beam, alpha, gc_frames=9, reclaim=reclaim, max_frames=512)
        D.reset()
        acc = [[] for _ in range(B)]
        for t0 in range(0, T, 20):
            D.decode_frames_host(np.ascontiguousarray(ll[t0:t0 + 20]), chunk_frames=6)
            pp = D.partial_paths(cap=4 * T)
            for b in range(B):
                acc[b] += pp["arcs"][b].tolist()
        res = D.best_paths(cap=4 * T + 64)
        assert res["rc"] == 0
        if reclaim:
            _check(res, og, ll, beam, alpha, B, tails=acc)
        else:
            _check(res, og, ll, beam, alpha, B)
            for b in range(B):   # the settled prefix is a prefix of the final path
                r = og.decode(ll[:, b, :], beam, alpha)
                assert list(r.arcs)[:len(acc[b])] == acc[b], b


def test_gc_excludes_lattice(W):
    g = I.hclg_graph(2000, 3, 50, seed=1)
    G = W.Graph.from_arrays(g)
    with pytest.raises(W.WfstError):
        W.Decoder(G, 2, 10.0, 100, gc_frames=8, lattice=1, lattice_beam=8.0)
    with pytest.raises(W.WfstError):
        W.Decoder(G, 2, 10.0, 100, gc_frames=-1)


def test_c5_other_full_size_with_gc(W, torch, oracle_mod):
    """C5 "other" on ONE GPU (4096 streams, 500 frames, 50-frame chunks, flat posteriors with
    max-active binding every frame): without traceback GC its records do not fit (some streams
    never settle); with partial results + reclaim + GC after every chunk it runs
    to completion, and sampled streams' partial outputs + final tails equal the oracle's paths."""
    import bench
    wl = bench.make_workload("c5", "other")
    T, B, P = wl["T"], wl["B"], wl["P"]
    G = W.Graph.from_arrays(wl["graph"])
    D = W.Decoder(G, B, wl["beam"], wl["alpha"], reclaim=1, gc_frames=50)
    ll = bench.device_loglikes(W, torch, wl, "cuda:0")
    og = oracle_mod.OracleGraph(wl["graph"])
    c = wl["c"]
    sample = (1, 1777, 4094)
    D.reset()
    acc = {b: [] for b in range(B)}
    for t0 in range(0, T, c["chunk"]):
        D.decode_frames(ll[t0:t0 + c["chunk"]])
        pp = D.partial_paths(cap=4 * T + 64)
        for b in sample:
            acc[b] += pp["arcs"][b].tolist()
    res = D.best_paths(cap=4 * T + 64)
    assert res["rc"] == 0
    st = D.stats()
    assert st["records_used_max"] < st["records_per_stream"]
    for b in sample:
        llh = I.loglikes_stream(c["ll_seed"], b, T, P, wl["planted"][:, b], **wl["preset"])
        r = og.decode(llh, wl["beam"], wl["alpha"])
        tail = list(res["arcs"][b, :res["n_arcs"][b]])
        assert acc[b] + tail == list(r.arcs), b
        assert res["cost"][b] == r.cost32, b
