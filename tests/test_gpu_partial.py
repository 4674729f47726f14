"""Row f2 (NEXT): settled partial results on the GPU vs the oracle's settled prefix (reading
R15), and SPEC's prefix consistency of mid-utterance best paths: after k frames
the best path equals the oracle's decode of the k-frame prefix."""
import math

import numpy as np
import pytest

import bruteforce as BF
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


@pytest.mark.parametrize("chunk,beam,alpha,cap", [(10, 10.0, 300, 224), (7, 12.0, 2000, 3), (1, 10.0, 50, 224)])
def test_partial_paths_match_oracle(W, torch, oracle_mod, chunk, beam, alpha, cap):
    """(cap 3: streams whose new arcs do not fit keep their settle point and are fetched again)"""
    g = I.hclg_graph(3000, 6, 200, seed=4)
    og = oracle_mod.OracleGraph(g)
    emit = g.ilabel[BF.canonical_order(g)] != 0
    T, B, P = 40, 6, 200
    pl = I.planted_walks(g, B, T, seed=9)
    ll = I.loglikes(77, range(B), T, P, pl, 1.0, 4.0)
    G = W.Graph.from_arrays(g)
    D = W.Decoder(G, B, beam, alpha)
    D.reset()
    t = torch.from_numpy(ll).cuda()
    acc = [[] for _ in range(B)]
    olab = [[] for _ in range(B)]
    grew = 0
    for t0 in range(0, T, chunk):
        D.decode_frames(t[t0:t0 + chunk].contiguous())
        pp = D.partial_paths(cap=cap)
        bp = D.best_paths(cap=4 * T + 64)
        for b in range(B):
            acc[b] += pp["arcs"][b].tolist()
            olab[b] += pp["olabels"][b].tolist()
            grew += len(pp["arcs"][b]) > 0
            L = min(t0 + chunk, T)
            want = og.settled_prefix(ll[:L, b, :], beam, alpha)
            assert acc[b] == want.tolist(), (b, L)
            assert pp["settled_frames"][b] == int(emit[want].sum()), (b, L)
            # SPEC prefix consistency: the mid-utterance best path is the prefix decode's
            r = og.decode(ll[:L, b, :], beam, alpha)
            n = bp["n_arcs"][b]
            assert list(bp["arcs"][b, :n]) == list(r.arcs) and bp["cost"][b] == r.cost32, (b, L)
            assert acc[b] == list(bp["arcs"][b, :len(acc[b])])
    assert grew > B
    olc = g.olabel[BF.canonical_order(g)]
    for b in range(B):
        assert olab[b] == [int(x) for x in olc[acc[b]] if x != 0]


def test_partial_paths_reset_restarts(W, torch):
    g = I.hclg_graph(2000, 3, 50, seed=3)
    G = W.Graph.from_arrays(g)
    D = W.Decoder(G, 2, 10.0, 100)
    pl = I.planted_walks(g, 2, 20, seed=2)
    ll = torch.from_numpy(I.loglikes(5, range(2), 20, 50, pl, 1.0, 4.0)).cuda()
    D.reset()
    D.decode_frames(ll)
    first = D.partial_paths()
    assert D.partial_paths()["arcs"][0].size == 0          # nothing new since the last call
    D.reset()
    D.decode_frames(ll)
    again = D.partial_paths()
    for b in range(2):
        assert np.array_equal(first["arcs"][b], again["arcs"][b])


def test_reclaim_unbounded_stream(W, torch, oracle_mod):
    """Traceback GC (second half of row f2): 600 frames through a 64-layer index ring and a
    record ring of ~60 frames, partial results every 20 frames.  The partial outputs followed by
    the final best path (which then starts at the settle point) equal the oracle's one-best
    path; the same decoder without reclaim runs out of layers."""
    g = I.hclg_graph(3000, 6, 200, seed=4)
    og = oracle_mod.OracleGraph(g)
    T, B, P, beam, alpha = 600, 4, 200, 10.0, 300
    pl = I.planted_walks(g, B, T, seed=9)
    ll = I.loglikes(77, range(B), T, P, pl, 1.0, 4.0)
    G = W.Graph.from_arrays(g)
    t = torch.from_numpy(ll).cuda()
    opts = dict(max_frames=64, records_per_stream=60 * 1200)
    D = W.Decoder(G, B, beam, alpha, reclaim=1, **opts)
    D.reset()
    acc = [[] for _ in range(B)]
    for t0 in range(0, T, 20):
        D.decode_frames(t[t0:t0 + 20].contiguous())
        pp = D.partial_paths(cap=4 * T)
        for b in range(B):
            acc[b] += pp["arcs"][b].tolist()
    res = D.best_paths(cap=4 * T + 64)
    assert res["rc"] == 0
    for b in range(B):
        r = og.decode(ll[:, b, :], beam, alpha)
        tail = list(res["arcs"][b, :res["n_arcs"][b]])
        assert acc[b] + tail == list(r.arcs), b
        assert res["cost"][b] == r.cost32 and len(tail) < len(r.arcs) // 4
    D2 = W.Decoder(G, B, beam, alpha, **opts)
    D2.reset()
    for t0 in range(0, T, 20):
        D2.decode_frames(t[t0:t0 + 20].contiguous())
    assert D2.best_paths(cap=4 * T + 64, raise_on_error=False)["rc"] == 6   # CAPACITY


def test_reclaim_excludes_lattice(W):
    g = I.hclg_graph(2000, 3, 50, seed=1)
    G = W.Graph.from_arrays(g)
    with pytest.raises(W.WfstError):
        W.Decoder(G, 2, 10.0, 100, reclaim=1, lattice=1, lattice_beam=8.0)


def test_partial_and_lattice_before_any_frame(W, torch, oracle_mod):
    """Edge case T = 0: right after reset nothing is settled, the lattice is layer 0 alone (the
    initial epsilon closure, reading R3) and equals the oracle's."""
    g = I.hclg_graph(3000, 6, 200, seed=4)
    G = W.Graph.from_arrays(g)
    D = W.Decoder(G, 2, 10.0, 300)
    D.reset()
    pp = D.partial_paths()
    assert all(a.size == 0 for a in pp["arcs"]) and list(pp["settled_frames"]) == [0, 0]
    DL = W.Decoder(G, 1, 10.0, 300, lattice=1, lattice_beam=8.0)
    DL.reset()
    L = DL.lattice(0)
    og = oracle_mod.OracleGraph(g)
    r = og.lattice(np.zeros((0, 200), np.float32), 10.0, 300, 8.0)
    assert L["n_layers"] == 1 == len(r.segments)
    st = DL.debug_layer(0, 0)[0]
    got = sorted((int(a), int(st[j])) for a, j in zip(L["segments"][0][0], L["segments"][0][2]))
    want = sorted((int(a), int(r.layers[0][0][j])) for a, j in zip(r.segments[0][0], r.segments[0][2]))
    assert got == want


def test_reclaim_long_streams_c3_graph(W, torch, oracle_mod):
    """Traceback GC at C3's scale: 64 streams x 3000 frames (30 s of audio each) on the 5M-state
    graph through a 256-layer ring and ~100 frames' worth of records per stream, settled results
    every 50 frames; sampled streams equal the oracle's one-best path end to end."""
    c = I.CONFIGS["c3"]
    g = I.config_graph("c3")
    T, B, P, chunk = 3000, 64, c["n_pdfs"], 50
    G = W.Graph.from_arrays(g)
    D = W.Decoder(G, B, c["beam"], c["max_active"], reclaim=1, max_frames=256, records_per_stream=100 * 12000)
    pl = I.planted_walks(g, B, T, seed=123)
    ids = torch.arange(0, B, dtype=torch.int32, device="cuda")
    plt = torch.from_numpy(np.ascontiguousarray(pl)).cuda()
    D.reset()
    acc = [[] for _ in range(B)]
    for t0 in range(0, T, chunk):
        x = torch.empty((chunk, B, P), dtype=torch.float32, device="cuda")
        W.synth_loglikes(x, ids, t0, 60006, plt[t0:t0 + chunk].contiguous(), **I.preset("clean"))
        D.decode_frames(x)
        pp = D.partial_paths()
        for b in range(B):
            acc[b] += pp["arcs"][b].tolist()
    res = D.best_paths(cap=4 * T + 64)
    assert res["rc"] == 0
    og = oracle_mod.OracleGraph(g)
    for b in (0, 37):
        ll = I.loglikes_stream(60006, b, T, P, pl[:, b], **I.preset("clean"))
        r = og.decode(ll, c["beam"], c["max_active"])
        tail = list(res["arcs"][b, :res["n_arcs"][b]])
        assert acc[b] + tail == list(r.arcs), b
        assert res["cost"][b] == r.cost32


def test_row_and_packed_apis_agree(W, torch):
    """wfst_get_partial_paths_ex (rows [n][cap]) and wfst_get_partial_paths_packed (ranges at
    offsets) return the same arcs, olabels, counts and settle points on two decoders fed the same
    chunks; the packed ranges do not overlap and *total is their sum."""
    import ctypes as C
    g = I.hclg_graph(3000, 6, 200, seed=4)
    T, B, P, cap = 40, 9, 200, 64
    pl = I.planted_walks(g, B, T, seed=2)
    t = torch.from_numpy(I.loglikes(5, range(B), T, P, pl, 1.0, 4.0)).cuda()
    G = W.Graph.from_arrays(g)
    D1, D2 = W.Decoder(G, B, 10.0, 300), W.Decoder(G, B, 10.0, 300)
    D1.reset()
    D2.reset()
    L = W.lib()
    p = lambda a: a.ctypes.data_as(C.c_void_p)
    for t0 in range(0, T, 8):
        D1.decode_frames(t[t0:t0 + 8])
        D2.decode_frames(t[t0:t0 + 8])
        ids = np.arange(B, dtype=np.int32)
        ra, ro = np.full((B, cap), -7, np.int32), np.full((B, cap), -7, np.int32)
        rn, rno, rf, rs = (np.zeros(B, np.int32) for _ in range(4))
        assert L.wfst_get_partial_paths_ex(D1.h, p(ids), B, p(ra), p(ro), cap, p(rn), p(rno), p(rf), p(rs)) == 0
        pa, po = np.full(B * cap, -7, np.int32), np.full(B * cap, -7, np.int32)
        off, tot = np.zeros(B, np.int64), np.zeros(1, np.int64)
        pn, pno, pf, ps = (np.zeros(B, np.int32) for _ in range(4))
        assert L.wfst_get_partial_paths_packed(D2.h, p(ids), B, p(pa), p(po), C.c_int64(B * cap), cap, p(off), p(tot),
                                               p(pn), p(pno), p(pf), p(ps)) == 0
        assert (rn == pn).all() and (rno == pno).all() and (rf == pf).all() and (rs == ps).all()
        assert int(tot[0]) == int(pn.sum())
        spans = sorted((int(off[i]), int(off[i]) + int(pn[i])) for i in range(B) if pn[i])
        assert all(a[1] <= b[0] for a, b in zip(spans, spans[1:]))
        for i in range(B):
            assert list(ra[i, :rn[i]]) == list(pa[off[i]:off[i] + pn[i]])
            assert list(ro[i, :rno[i]]) == list(po[off[i]:off[i] + pno[i]])
    # total_cap below n * cap is rejected before any work
    rc = L.wfst_get_partial_paths_packed(D2.h, p(ids), B, p(pa), p(po), C.c_int64(B * cap - 1), cap, p(off), p(tot),
                                         p(pn), p(pno), p(pf), p(ps))
    assert rc == 1
