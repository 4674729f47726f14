"""CUDA path (libwfst_gpu.so through the C ABI) vs the CPU oracle, element by element.

Bar (north_star): identical olabel sequences and arc-id traceback, identical
reached-final flag, best cost within 1e-4 relative -- and since both sides follow the same
fp32 operation order (R1) and tie rule (R9), we assert the cost BIT-EXACT as well.
"""
import math

import numpy as np
import pytest

import bruteforce as BF
from paper_1910_10032_b200 import inputs as I

pytestmark = pytest.mark.gpu
INF = math.inf


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


def _gpu_run(W, torch, g, ll, beam, alpha, streams=None, splits=None, G=None, **opts):
    G = G or W.Graph.from_arrays(g)
    T, B, P = ll.shape
    D = W.Decoder(G, B, beam, alpha, **opts)
    D.reset()
    t = torch.from_numpy(np.ascontiguousarray(ll)).cuda()
    if splits:
        t0 = 0
        for n in splits:
            D.decode_frames(t[t0:t0 + n].contiguous(), streams=streams)
            t0 += n
        assert t0 == T
    else:
        D.decode_frames(t, streams=streams)
    torch.cuda.synchronize()
    return D, D.best_paths(cap=4 * T + 64, raise_on_error=False)


def _compare(og, ll, beam, alpha, res, b, lane=None):
    lane = b if lane is None else lane
    r = og.decode(ll[:, b, :], beam, alpha)
    n = res["n_arcs"][lane]
    assert res["reached_final"][lane] == r.reached_final, (b, lane)
    assert list(res["arcs"][lane, :n]) == list(r.arcs), (b, lane)
    assert list(res["olabels"][lane, :res["n_olabels"][lane]]) == list(r.olabels)
    assert abs(float(res["cost"][lane]) - r.cost) <= 1e-4 * max(1.0, abs(r.cost))
    assert res["cost"][lane] == r.cost32, (b, float(res["cost"][lane]), r.cost)
    return r


def test_synth_loglikes_bit_identical(W, torch):
    for (T, B, P, seed, t0, boost) in [(3, 4, 37, 5, 0, 4.0), (2, 3, 5700, 30003, 17, 0.0)]:
        ids = np.array([0, 7, 123456, 9][:B], np.int32)
        pl = np.random.default_rng(0).integers(0, P, (T, B)).astype(np.int32)
        out = torch.empty((T, B, P), dtype=torch.float32, device="cuda")
        W.synth_loglikes(out, torch.from_numpy(ids).cuda(), t0, seed, torch.from_numpy(pl).cuda(), 1.0, boost)
        host = np.stack([I.loglikes_stream(seed, int(s), t0 + T, P, np.concatenate(
            [np.zeros(t0, np.int32), pl[:, j]]), 1.0, boost)[t0:] for j, s in enumerate(ids)], axis=1)
        assert np.array_equal(out.cpu().numpy().view(np.uint32), host.view(np.uint32))


def test_spec_example(W, torch, oracle_mod):
    """SPEC S:493 through the text loader: words [1, 2], cost -2.2."""
    import os
    G = W.Graph.load(os.path.join(os.path.dirname(__file__), "golden", "spec_example.txt"))
    info = G.info()
    assert (info.n_states, info.n_arcs, info.n_emitting, info.eq1_bytes) == (3, 3, 2, 68)
    D = W.Decoder(G, 1, INF, 0)
    D.reset()
    D.decode_frames(torch.tensor([[[2.0, 0.0]], [[0.0, 1.0]]], device="cuda"))
    r = D.best_path(0)
    assert list(r["olabels"]) == [1, 2] and r["reached_final"] == 1
    assert r["cost32"] == np.float32(np.float32(np.float32(0.5) - np.float32(2.0)) + np.float32(0.3)) - np.float32(1.0)


def test_empty_utterance_and_errors(W, torch):
    g = I._mk(2, 0, [0], [1], [1], [0], [1.0], [0.0, np.inf])
    G = W.Graph.from_arrays(g)
    D = W.Decoder(G, 2, 10.0, 100)
    with pytest.raises(W.WfstError) as e:             # decode before reset
        D.decode_frames(torch.zeros((1, 2, 1), device="cuda"))
    assert e.value.status == "STATE"
    D.reset()
    r = D.best_path(1)                                # T = 0: start state final 0
    assert r["cost"] == 0.0 and r["reached_final"] == 1 and len(r["arcs"]) == 0
    with pytest.raises(W.WfstError) as e:             # P <= max pdf
        D.decode_frames(torch.zeros((1, 2, 0), device="cuda"))
    assert e.value.status in ("PDF_RANGE", "INVALID_ARG")
    D.decode_frames(torch.zeros((1, 2, 1), device="cuda"))
    D.decode_frames(torch.zeros((1, 2, 1), device="cuda"))   # state 1 has no arcs -> NO_SURVIVOR
    with pytest.raises(W.WfstError) as e:
        D.sync()
    assert e.value.status == "NO_SURVIVOR"
    assert D.status(0) == "NO_SURVIVOR"


def test_tiny_random_graphs(W, torch, oracle_mod):
    """Random <=6-state graphs, infinite and finite beams, vs oracle (and brute force)."""
    n = 0
    for seed in range(60):
        g = I.random_tiny_graph(seed)
        rng = np.random.default_rng(seed + 7)
        T = int(rng.integers(1, 6))
        ll = rng.uniform(-3, 0, (T, 1, 4)).astype(np.float32)
        og = oracle_mod.OracleGraph(g)
        for beam, alpha in ((INF, 0), (1.0, 2)):
            try:
                og.decode(ll[:, 0, :], beam, alpha)
            except oracle_mod.OracleError:
                continue
            D, res = _gpu_run(W, torch, g, ll, beam, alpha)
            _compare(og, ll, beam, alpha, res, 0)
            n += 1
    assert n > 60


def test_c1_parity(W, torch, oracle_mod):
    """C1: 200 log-likelihood seeds decoded as 200 concurrent streams, infinite beam; also
    equal to the fp64 trellis on tie-free seeds."""
    g = I.c1_graph()
    B, T, P = 200, 30, 10
    pl = np.stack([I.planted_walks(g, 1, T, seed=s)[:, 0] for s in range(1, B + 1)], axis=1)
    ll = np.stack([I.loglikes_stream(s, 0, T, P, pl[:, s - 1], 1.5, 2.0) for s in range(1, B + 1)], axis=1)
    og = oracle_mod.OracleGraph(g)
    D, res = _gpu_run(W, torch, g, ll, INF, 0)
    canon = BF.canonical_order(g)
    for b in range(B):
        r = _compare(og, ll, INF, 0, res, b)
        kb = BF.trellis_kbest(g, ll[:, b, :], k=1)
        assert [int(canon[a]) for a in r.arcs] == kb[0][1] or abs(kb[0][0] - r.cost) < 1e-4


def _hclg_case(n_states, degree, P, B, T, seed, preset="clean"):
    g = I.hclg_graph(n_states, degree, P, seed=seed)
    pl = I.planted_walks(g, B, T, seed=seed + 1)
    ll = I.loglikes(seed + 1, range(B), T, P, pl, **I.preset(preset))
    return g, ll


def test_c2_parity_all_streams(W, torch, oracle_mod):
    """C2 (BASELINE configs[1]): 50k states / 300k arcs / 2k pdfs, 100 streams x 500 frames,
    beam 10, max-active 10k -- every stream."""
    c = I.CONFIGS["c2"]
    g = I.config_graph("c2")
    T, B, P = c["frames"], c["streams"], c["n_pdfs"]
    pl = I.planted_walks(g, B, T, seed=c["ll_seed"])
    ll = I.loglikes(c["ll_seed"], range(B), T, P, pl, **I.preset(c["preset"]))
    og = oracle_mod.OracleGraph(g)
    D, res = _gpu_run(W, torch, g, ll, c["beam"], c["max_active"])
    assert res["rc"] == 0
    for b in range(B):
        _compare(og, ll, c["beam"], c["max_active"], res, b)
    # per-frame cutoffs bit-exact on a few streams
    for b in (0, 37, 99):
        r = og.decode(ll[:, b, :], c["beam"], c["max_active"])
        fs, fc = D.frame_stats(b)
        assert np.array_equal(fs[:, :2].view(np.uint32), r.frame_stats[:, :2].view(np.uint32))
        assert np.array_equal(fc[:, 2], r.frame_counts[:, 2])       # survivors per frame
        assert np.array_equal(fc[:, 3], r.frame_counts[:, 3])       # emitting arcs expanded
        assert np.array_equal(fc[:, 4], r.frame_counts[:, 4])       # eps out-degree of survivors
        both = np.isfinite(fs[:, 2]) & np.isfinite(r.frame_stats[:, 2])
        assert np.array_equal(fs[both, 2], r.frame_stats[both, 2])


def test_alpha_bound_other_preset_survivor_sets(W, torch, oracle_mod):
    """Flat ("other") posteriors: max-active binds every frame.  Survivor sets per layer equal."""
    g, ll = _hclg_case(20_000, 3.0, 500, 6, 60, seed=12, preset="other")
    og = oracle_mod.OracleGraph(g)
    for alpha in (300, 2000):
        D, res = _gpu_run(W, torch, g, ll, 15.0, alpha, debug_costs=1)
        for b in range(6):
            r = og.decode(ll[:, b, :], 15.0, alpha, survivors=True)
            _compare(og, ll, 15.0, alpha, res, b)
            for k in (0, 1, 7, 30, 60):
                st, ar, co = D.debug_layer(b, k)
                o = np.argsort(st)
                ost, oar, oco = r.layers[k]
                assert np.array_equal(st[o], ost) and np.array_equal(ar[o], oar)
                assert np.array_equal(co[o].view(np.uint32), oco.view(np.uint32))


def test_overflow_table_path(W, torch, oracle_mod):
    """A tiny on-chip table forces the global overflow table: results must not change; an
    overflow table that is also too small must raise CAPACITY (never silently drop)."""
    g, ll = _hclg_case(20_000, 3.0, 500, 4, 40, seed=13, preset="other")
    og = oracle_mod.OracleGraph(g)
    D, res = _gpu_run(W, torch, g, ll, 15.0, 1000, table_slots=256, overflow_slots=32768)
    st = D.stats()
    assert st["overflow_inserts"] > 0
    for b in range(4):
        _compare(og, ll, 15.0, 1000, res, b)
    D, res = _gpu_run(W, torch, g, ll, 15.0, 5000, table_slots=256, overflow_slots=256)
    assert res["rc"] == 6 or any(D.status(b) == "CAPACITY" for b in range(4))


def test_lane_order_subset_and_chunk_invariance(W, torch, oracle_mod):
    """S:249/S:266 lane independence: a stream decoded in a permuted lane order, in frame
    chunks across calls, gives the same result."""
    g, ll = _hclg_case(20_000, 3.0, 500, 8, 50, seed=14)
    og = oracle_mod.OracleGraph(g)
    D, base = _gpu_run(W, torch, g, ll, 12.0, 800)
    perm = np.array([5, 2, 7, 0, 1, 6, 3, 4], np.int32)
    D2, res = _gpu_run(W, torch, g, ll, 12.0, 800, streams=perm, splits=[7, 20, 23])
    for b in range(8):
        lane = int(perm[b])
        assert res["cost"][lane] == base["cost"][b]
        assert np.array_equal(res["arcs"][lane, :res["n_arcs"][lane]], base["arcs"][b, :base["n_arcs"][b]])
        _compare(og, ll, 12.0, 800, base, b)
    # many frames per work item vs one: forces lane migration between CTAs
    D3, res3 = _gpu_run(W, torch, g, ll, 12.0, 800, frames_per_item=1, max_ctas=3)
    assert np.array_equal(res3["cost"].view(np.uint32), base["cost"].view(np.uint32))


def test_host_input_path_and_determinism(W, torch, oracle_mod):
    g, ll = _hclg_case(20_000, 3.0, 500, 6, 40, seed=15)
    G = W.Graph.from_arrays(g)
    D = W.Decoder(G, 6, 15.0, 1000)
    D.reset()
    D.decode_frames_host(np.ascontiguousarray(ll), chunk_frames=7)
    D.sync()
    a = D.best_paths(cap=256)
    _, b = _gpu_run(W, torch, g, ll, 15.0, 1000, G=G)
    _, c = _gpu_run(W, torch, g, ll, 15.0, 1000, G=G)
    assert np.array_equal(a["cost"].view(np.uint32), b["cost"].view(np.uint32))
    assert np.array_equal(b["cost"].view(np.uint32), c["cost"].view(np.uint32))
    for k in range(6):
        n = b["n_arcs"][k]
        assert a["n_arcs"][k] == n == c["n_arcs"][k]
        assert np.array_equal(a["arcs"][k, :n], b["arcs"][k, :n]) and np.array_equal(b["arcs"][k, :n], c["arcs"][k, :n])


def _all_streams_vs_oracle(og, gen_ll, streams, beam, alpha, res, lane_of=None, batch=48):
    """Every stream of a full-size run against the oracle: host log-likelihoods regenerated by
    inputs.py (never copied from the device) in batches, decoded by the oracle's threaded batch
    driver on all host cores, compared element by element (path, olabel-bearing arcs, flag, cost
    bits)."""
    import concurrent.futures as cf
    import os
    cores = os.cpu_count() or 1
    streams = list(streams)
    cap = res["arcs"].shape[1]
    n = 0
    for k in range(0, len(streams), batch):
        ids = streams[k:k + batch]
        with cf.ThreadPoolExecutor(cores) as ex:
            rows = list(ex.map(gen_ll, ids))
        ll = np.ascontiguousarray(np.stack(rows, axis=1))
        cost, reached, rc, _, arcs, n_arcs = og.decode_batch(ll, beam, alpha, cores, arcs_cap=cap)
        for j, b in enumerate(ids):
            lane = b if lane_of is None else lane_of(b)
            assert rc[j] == 0, (b, rc[j])
            m = res["n_arcs"][lane]
            assert m == n_arcs[j] and np.array_equal(res["arcs"][lane, :m], arcs[j, :m]), b
            assert res["reached_final"][lane] == reached[j], b
            assert res["cost"][lane].view(np.uint32) == cost[j].view(np.uint32), b
            n += 1
    return n


@pytest.mark.slow
@pytest.mark.parametrize("preset", ["clean", "other"])
def test_c3_full_size_all_streams(W, torch, oracle_mod, preset):
    """C3 (the bench workload) at full size in bench.py's launch configuration: 512 streams x
    500 frames, 5M-state graph, beam 15, max-active 10k, device-generated log-likelihoods --
    EVERY stream against the oracle, for the clean preset and the alpha-saturated "other"."""
    import bench
    res, ctx = bench.run_gpu_once("c3", preset, with_paths=True)
    assert res["rc"] == 0
    og = oracle_mod.OracleGraph(ctx["graph"])
    c = I.CONFIGS["c3"]
    gen = lambda b: I.loglikes_stream(c["ll_seed"], b, c["frames"], c["n_pdfs"], ctx["planted"][:, b],
                                      **I.preset(preset))
    assert _all_streams_vs_oracle(og, gen, range(c["streams"]), c["beam"], c["max_active"], res) == 512


def test_eps_general_permuted_c2_all_streams(W, torch, oracle_mod):
    """C2's shape (50k states, degree 6, 2k pdfs, 100 streams x 500 frames, beam 10, max-active
    10k) on the epsilon-general generator: random state ids, back-off chains of 5 epsilon arcs,
    heavier skip arcs (re-relaxation), positive epsilon 2-cycles -- every stream, plus the
    survivor sets of a few layers on the alpha-saturated preset."""
    c = I.CONFIGS["c2"]
    g = I.hclg_graph_eps(50_000, 6.0, 2000, seed=2)
    T, B, P = c["frames"], c["streams"], c["n_pdfs"]
    pl = I.planted_walks(g, B, T, seed=c["ll_seed"])
    og = oracle_mod.OracleGraph(g)
    G = W.Graph.from_arrays(g)
    ll = I.loglikes(c["ll_seed"], range(B), T, P, pl, **I.preset(c["preset"]))
    D, res = _gpu_run(W, torch, g, ll, c["beam"], c["max_active"], G=G)
    assert res["rc"] == 0
    gen = lambda b: np.ascontiguousarray(ll[:, b, :])
    assert _all_streams_vs_oracle(og, gen, range(B), c["beam"], c["max_active"], res) == B
    st = D.stats()
    assert st["eps_relax"] > st["eps_arcs"] > 0      # epsilon work happened (incl. re-relaxations)
    llo = I.loglikes(c["ll_seed"] + 1, range(4), 40, P, pl[:40, :4], **I.preset("other"))
    D, res = _gpu_run(W, torch, g, llo, c["beam"], 600, G=G, debug_costs=1)
    for b in range(4):
        r = og.decode(llo[:, b, :], c["beam"], 600, survivors=True)
        _compare(og, llo, c["beam"], 600, res, b)
        for k in (0, 1, 13, 40):
            st_, ar, co = D.debug_layer(b, k)
            o = np.argsort(st_)
            ost, oar, oco = r.layers[k]
            assert np.array_equal(st_[o], ost) and np.array_equal(ar[o], oar)
            assert np.array_equal(co[o].view(np.uint32), oco.view(np.uint32))


@pytest.mark.parametrize("threads,ctas", [(256, 1), (256, 2), (512, 2), (256, 3), (256, 4), (1024, 1)])
def test_kernel_variants_parity(W, torch, oracle_mod, threads, ctas):
    """Every (CTA size, CTAs per SM) variant of the frame kernel gives the oracle's answer,
    including when its smaller on-chip table spills to the overflow table."""
    g, ll = _hclg_case(20_000, 3.0, 500, 12, 60, seed=16, preset="other")
    og = oracle_mod.OracleGraph(g)
    D, res = _gpu_run(W, torch, g, ll, 15.0, 3000, threads=threads, ctas_per_sm=ctas)
    assert res["rc"] == 0
    for b in range(12):
        _compare(og, ll, 15.0, 3000, res, b)


def test_tie_heavy_dyadic(W, torch, oracle_mod):
    """Integer-valued weights and log-likelihoods make exact fp32 cost ties common: the GPU's
    winner words must reproduce the oracle's (cost, canonical arc id) tie-break (R9) exactly,
    including ties between candidates from different source tokens and between emitting and
    epsilon arcs."""
    g = I.hclg_graph(20_000, 3.0, 40, seed=17)
    g.weight = np.round(g.weight).astype(np.float32)
    g.final = np.where(np.isfinite(g.final), np.round(g.final), np.inf).astype(np.float32)
    B, T, P = 8, 40, 40
    rng = np.random.default_rng(5)
    ll = rng.integers(-3, 1, (T, B, P)).astype(np.float32)
    og = oracle_mod.OracleGraph(g)
    for beam, alpha in ((6.0, 300), (4.0, 50), (INF, 2000)):
        D, res = _gpu_run(W, torch, g, ll, beam, alpha)
        for b in range(B):
            _compare(og, ll, beam, alpha, res, b)


@pytest.mark.slow
@pytest.mark.slow
def test_c4_full_size_all_streams(W, torch, oracle_mod):
    """C4 (BASELINE configs[3]) at its bench size and launch configuration: 1024 streams x 500
    frames on the ~50M-state / ~150M-arc graph, decoded in 50-frame chunks -- the final paths of
    EVERY stream against the oracle, element by element."""
    import bench
    wl = bench.make_workload("c4", "clean")
    T, B = wl["T"], wl["B"]
    c = wl["c"]
    G = W.Graph.from_arrays(wl["graph"])
    D = W.Decoder(G, B, wl["beam"], wl["alpha"])
    ll = bench.device_loglikes(W, torch, wl, "cuda:0")
    D.reset()
    for t0 in range(0, T, c["chunk"]):
        D.decode_frames(ll[t0:t0 + c["chunk"]])
    res = D.best_paths(cap=4 * T + 64)
    assert res["rc"] == 0
    del ll
    og = oracle_mod.OracleGraph(wl["graph"])
    gen = lambda b: I.loglikes_stream(c["ll_seed"], b, T, wl["P"], wl["planted"][:, b], **wl["preset"])
    assert _all_streams_vs_oracle(og, gen, range(B), wl["beam"], wl["alpha"], res) == 1024


def test_c4_large_graph_memory_and_chunks(W, torch, oracle_mod):
    """C4 (BASELINE configs[3]): a large-LM-shaped graph (~50M states / ~150M arcs) and 1024
    streams decoded in 50-frame chunks.  Checks the device footprint against Eq. 1
    and sampled streams against the oracle."""
    c = I.CONFIGS["c4"]
    g = I.config_graph("c4")
    T, B, P = 100, c["streams"], c["n_pdfs"]
    G = W.Graph.from_arrays(g)
    info = G.info()
    assert info.n_states == g.n_states and info.n_arcs == g.n_arcs
    # device layout: 16 B per state + 16 B per arc + 4 B olabel per arc, vs Eq. 1's 12|Q|+8|E|+4|E_E|
    assert info.device_bytes == 16 * info.n_states + 20 * info.n_arcs
    assert info.eq1_bytes == 12 * info.n_states + 8 * info.n_arcs + 4 * info.n_emitting
    pl = I.planted_walks(g, 8, T, seed=c["ll_seed"])
    D = W.Decoder(G, B, c["beam"], c["max_active"], records_per_stream=T * 12000)
    ll = torch.empty((T, B, P), dtype=torch.float32, device="cuda")
    ids = torch.arange(0, B, dtype=torch.int32, device="cuda")
    plb = np.zeros((T, B), np.int32)
    plb[:, :8] = pl
    W.synth_loglikes(ll, ids, 0, c["ll_seed"], torch.from_numpy(plb).cuda(), **I.preset(c["preset"]))
    D.reset()
    for t0 in range(0, T, c["chunk"]):
        D.decode_frames(ll[t0:t0 + c["chunk"]])
    res = D.best_paths(cap=4 * T + 64)
    assert res["rc"] == 0
    st = D.stats()
    assert st["frames"] == T * B and st["device_bytes"] > 0
    og = oracle_mod.OracleGraph(g)
    for b in (0, 3, 7):
        llh = I.loglikes_stream(c["ll_seed"], b, T, P, pl[:, b], **I.preset(c["preset"]))
        r = og.decode(llh, c["beam"], c["max_active"])
        n = res["n_arcs"][b]
        assert res["reached_final"][b] == r.reached_final
        assert list(res["arcs"][b, :n]) == list(r.arcs)
        assert res["cost"][b] == r.cost32


def test_c3_other_full_size_sampled(W, torch, oracle_mod):
    """C3's alpha-saturated "other" preset (max-active binds every frame, 10k survivors) at full
    size in the bench's launch configuration; sampled streams against the oracle, including the
    per-frame cutoffs."""
    import bench
    res, ctx = bench.run_gpu_once("c3", "other", with_paths=True)
    og = oracle_mod.OracleGraph(ctx["graph"])
    c = I.CONFIGS["c3"]
    for b in (3, 300):
        ll = I.loglikes_stream(c["ll_seed"], b, c["frames"], c["n_pdfs"], ctx["planted"][:, b], **I.preset("other"))
        r = og.decode(ll, c["beam"], c["max_active"])
        n = res["n_arcs"][b]
        assert list(res["arcs"][b, :n]) == list(r.arcs)
        assert res["cost"][b] == r.cost32 and res["reached_final"][b] == r.reached_final


def test_c5_online_chunks_full_size(W, torch, oracle_mod):
    """C5 (BASELINE configs[4]) on one GPU: 4096 concurrent streams on C3's graph, 500 frames in
    50-frame chunks, settled partial results fetched after every chunk (row f2); sampled streams
    checked against the oracle (final path, and the settled prefix after each chunk)."""
    import bench
    wl = bench.make_workload("c5", "clean")
    T, B, P = wl["T"], wl["B"], wl["P"]
    G = W.Graph.from_arrays(wl["graph"])
    D = W.Decoder(G, B, wl["beam"], wl["alpha"])
    ll = bench.device_loglikes(W, torch, wl, "cuda:0")
    og = oracle_mod.OracleGraph(wl["graph"])
    c = wl["c"]
    sample = (0, 2047, 4095)
    llh = {b: I.loglikes_stream(c["ll_seed"], b, T, P, wl["planted"][:, b], **wl["preset"]) for b in sample}
    D.reset()
    acc = {b: [] for b in sample}
    for t0 in range(0, T, c["chunk"]):
        D.decode_frames(ll[t0:t0 + c["chunk"]])
        pp = D.partial_paths(streams=list(sample), cap=4 * T + 64)
        for i, b in enumerate(sample):
            acc[b] += pp["arcs"][i].tolist()
            if t0 in (0, 200, 450):
                want = og.settled_prefix(llh[b][:t0 + c["chunk"]], wl["beam"], wl["alpha"])
                assert acc[b] == want.tolist(), (b, t0)
    res = D.best_paths(cap=4 * T + 64)
    assert res["rc"] == 0
    for b in sample:
        r = og.decode(llh[b], wl["beam"], wl["alpha"])
        n = res["n_arcs"][b]
        assert list(res["arcs"][b, :n]) == list(r.arcs) and res["cost"][b] == r.cost32
        assert acc[b] == list(r.arcs[:len(acc[b])]) and len(acc[b]) > 100
    # final paths of EVERY one of the 4096 streams against the oracle
    gen = lambda b: I.loglikes_stream(c["ll_seed"], b, T, P, wl["planted"][:, b], **wl["preset"])
    assert _all_streams_vs_oracle(og, gen, range(B), wl["beam"], wl["alpha"], res) == 4096


def test_graph_replicate(W, torch, oracle_mod):
    """Row e: a graph replica (device-to-device copy; onto every visible device) decodes like the
    original."""
    g = I.hclg_graph(3000, 6, 200, seed=4)
    G = W.Graph.from_arrays(g)
    T, B = 20, 4
    pl = I.planted_walks(g, B, T, seed=9)
    ll = I.loglikes(77, range(B), T, 200, pl, 1.0, 4.0)
    outs = []
    for dev in range(torch.cuda.device_count()):
        Gr = G.replicate(dev)
        info, info0 = Gr.info(), G.info()
        assert (info.n_states, info.n_arcs, info.device) == (info0.n_states, info0.n_arcs, dev)
        with torch.cuda.device(dev):
            D = W.Decoder(Gr, B, 10.0, 300)
            D.reset()
            D.decode_frames(torch.from_numpy(ll).to(f"cuda:{dev}"))
            outs.append(D.best_paths(cap=4 * T + 64))
    og = oracle_mod.OracleGraph(g)
    for b in range(B):
        r = og.decode(ll[:, b, :], 10.0, 300)
        for res in outs:
            n = res["n_arcs"][b]
            assert list(res["arcs"][b, :n]) == list(r.arcs) and res["cost"][b] == r.cost32


@pytest.mark.parametrize("order,cap", [(0, 0), (1, 0), (2, 0), (2, 16)])
def test_insert_order_never_changes_results(W, torch, oracle_mod, order, cap):
    """Bin-ordered insertion (opts.insert_order) changes only the order in which
    a frame's candidates enter the token table -- arrival order, bin order after alpha-bound
    frames (default), always bin order, and bin order with tiny bin buffers (most candidates
    take the direct-insert fallback): survivors, cutoffs and paths equal the oracle's."""
    g, ll = _hclg_case(20_000, 3.0, 500, 6, 50, seed=18, preset="other")
    og = oracle_mod.OracleGraph(g)
    opts = dict(insert_order=order, debug_costs=1)
    if cap:
        opts["bin_capacity"] = cap
    for alpha in (300, 2500):
        D, res = _gpu_run(W, torch, g, ll, 15.0, alpha, **opts)
        assert res["rc"] == 0
        for b in range(6):
            r = og.decode(ll[:, b, :], 15.0, alpha, survivors=True)
            _compare(og, ll, 15.0, alpha, res, b)
            fs, fc = D.frame_stats(b)
            assert np.array_equal(fs[:, :2].view(np.uint32), r.frame_stats[:, :2].view(np.uint32))
            # k_alpha: equal where both sides used it; the GPU may skip the selection (+inf) when its
            # table held <= alpha candidates (early-rejected ones are above k_alpha), the survivors
            # are the same either way (checked below)
            both = np.isfinite(fs[:, 2]) & np.isfinite(r.frame_stats[:, 2])
            assert np.array_equal(fs[both, 2].view(np.uint32), r.frame_stats[both, 2].view(np.uint32))
            assert np.all(fc[np.isfinite(r.frame_stats[:, 2]) & ~both, 2] >= alpha)
            for k in (1, 25, 50):
                st, ar, co = D.debug_layer(b, k)
                o = np.argsort(st)
                ost, oar, oco = r.layers[k]
                assert np.array_equal(st[o], ost) and np.array_equal(ar[o], oar)
                assert np.array_equal(co[o].view(np.uint32), oco.view(np.uint32))
