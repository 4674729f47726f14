"""Row f1 (NEXT): lattice segments and the end-of-utterance backward sweep on the GPU vs the CPU
oracle (oracle_lattice / oracle_lattice_finalize, readings R13-R14), element by element.

Token indices differ (the GPU's layers are in cost-bucketed order, the oracle's sorted by state),
so entries are compared through the states they name: per segment k the set of
(arc, src state, dst state, slack bits), per arc the path slack bits, per (layer, state) gamma.
Both sides do the same fp32 operations (R1), so everything is compared bit-exact.  The GPU's
CSR layout is checked as such: destination token indices non-decreasing, arc ids ascending
inside a group.
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


def _bits(x):
    return int(np.float32(x).view(np.uint32)) if not (np.float32(x) == 0) else 0   # +0 == -0


def _gpu_lattice(W, torch, g, ll, beam, alpha, lb, splits=None, G=None):
    G = G or W.Graph.from_arrays(g)
    T, B, P = ll.shape
    D = W.Decoder(G, B, beam, alpha, lattice=1, lattice_beam=lb)
    D.reset()
    t = torch.from_numpy(np.ascontiguousarray(ll)).cuda()
    t0 = 0
    for n in (splits or [T]):
        if n:
            D.decode_frames(t[t0:t0 + n].contiguous())
        t0 += n
    torch.cuda.synchronize()
    return D


def _check_stream(D, og, ll_b, beam, alpha, lb, b, emit):
    r = og.lattice(ll_b, beam, alpha, lb)
    L = D.lattice(b)
    T = ll_b.shape[0]
    assert L["n_layers"] == T + 1 == len(r.layers)
    assert L["reached_final"] == r.reached_final
    assert _bits(L["best"]) == _bits(r.lattice_best), (b, float(L["best"]), r.lattice_best)
    gl = [D.debug_layer(b, k)[0] for k in range(T + 1)]
    off = np.concatenate([[0], np.cumsum([len(x) for x in gl])])
    n_arcs = 0
    for k in range(T + 1):
        st_g, st_o = gl[k], r.layers[k][0]
        assert sorted(st_g.tolist()) == st_o.tolist(), (b, k)
        arc, src, dst, sl = L["segments"][k]
        ps = L["pslack"][k]
        n_arcs += len(arc)
        # CSR by destination token, arc ascending inside a group
        if len(dst) > 1:
            d = np.diff(dst)
            assert np.all(d >= 0), (b, k)
            same = d == 0
            assert np.all(np.diff(arc)[same] > 0), (b, k)
        prev_g = gl[k - 1] if k > 0 else None
        got, got_ps = set(), {}
        for a, i, j, s, p in zip(arc, src, dst, sl, ps):
            emitting = i >= 0 and k > 0 and int(a) in emit
            sst = prev_g[i] if emitting else st_g[i]
            got.add((int(a), int(sst), int(st_g[j]), _bits(s)))
            got_ps[int(a)] = _bits(p)
        oa, osrc, odst, osl = r.segments[k]
        prev_o = r.layers[k - 1][0] if k > 0 else None
        want, want_ps = set(), {}
        for a, i, j, s, p in zip(oa, osrc, odst, osl, r.pslack[k]):
            emitting = k > 0 and int(a) in emit
            sst = prev_o[i] if emitting else st_o[i]
            want.add((int(a), int(sst), int(st_o[j]), _bits(s)))
            want_ps[int(a)] = _bits(p)
        assert got == want, (b, k, sorted(got ^ want)[:6])
        assert got_ps == want_ps, (b, k)
        # gamma per state
        gg = dict(zip(st_g.tolist(), (_bits(x) for x in L["gamma"][off[k]:off[k + 1]])))
        go = dict(zip(st_o.tolist(), (_bits(x) for x in r.gamma[k])))
        assert gg == go, (b, k)
    return n_arcs


def _emit_set(g):
    """canonical ids of the emitting arcs"""
    return set(np.nonzero(g.ilabel[BF.canonical_order(g)] != 0)[0].tolist())


def _dyadic(seed, Q=6, E=16, T=4, P=4):
    rng = np.random.default_rng(seed)
    g = I.random_tiny_graph(seed, n_states=Q, n_arcs=E, n_pdfs=P)
    g.weight = (np.round(g.weight * 8) / 8).astype(np.float32)
    g.final = np.where(np.isfinite(g.final), np.round(g.final * 8) / 8, np.inf).astype(np.float32)
    ll = (rng.integers(-24, 1, (T, P)) / 8.0).astype(np.float32)
    return g, ll


@pytest.mark.parametrize("lb", [0.0, 1.25, 8.0, INF])
def test_lattice_tiny_infinite_beam(W, torch, oracle_mod, lb):
    """Tiny dyadic instances (the ones the oracle is pinned on by path enumeration)."""
    n = 0
    for seed in range(40):
        g, ll = _dyadic(seed)
        og = oracle_mod.OracleGraph(g)
        try:
            og.decode(ll, INF, 0)
        except oracle_mod.OracleError:
            continue
        D = _gpu_lattice(W, torch, g, ll[:, None, :], INF, 0, lb)
        _check_stream(D, og, ll, INF, 0, lb, 0, _emit_set(g))
        n += 1
    assert n > 25


def test_lattice_c2_shaped_finite_beam(W, torch, oracle_mod):
    """HCLG-shaped graph, finite beam and max-active, 8 streams, two decode calls (the segment
    arena and layer index across calls), lattice-beam 6."""
    g = I.hclg_graph(3000, 6, 200, seed=4)
    og = oracle_mod.OracleGraph(g)
    emit = _emit_set(g)
    T, B = 30, 8
    pl = I.planted_walks(g, B, T, seed=9)
    ll = I.loglikes(77, range(B), T, 200, pl, 1.0, 4.0)
    D = _gpu_lattice(W, torch, g, ll, 10.0, 300, 6.0, splits=[13, 17])
    total = 0
    for b in range(B):
        total += _check_stream(D, og, ll[:, b, :], 10.0, 300, 6.0, b, emit)
    assert total > 1000


def test_lattice_c2_graph_alpha_binding(W, torch, oracle_mod):
    """C2's 50k-state graph, flat posteriors (max-active binds), lattice-beam 8."""
    g = I.hclg_graph(50_000, 6, 2000, seed=2)
    og = oracle_mod.OracleGraph(g)
    emit = _emit_set(g)
    T, B = 12, 3
    pl = I.planted_walks(g, B, T, seed=3)
    ll = I.loglikes(20002, range(B), T, 2000, pl, 1.0, 0.0)
    D = _gpu_lattice(W, torch, g, ll, 10.0, 2000, 8.0)
    for b in range(B):
        _check_stream(D, og, ll[:, b, :], 10.0, 2000, 8.0, b, emit)


def test_lattice_requires_option(W, torch):
    g = I.hclg_graph(2000, 3, 50, seed=1)
    G = W.Graph.from_arrays(g)
    D = W.Decoder(G, 2, 10.0, 100)
    D.reset()
    with pytest.raises(W.WfstError):
        D.lattice(0)


def test_lattice_with_stream_subsets(W, torch, oracle_mod):
    """Decode calls on changing subsets of the streams (row f3) with lattices on: each call's
    segments land in the right streams' arenas and layers."""
    g = I.hclg_graph(3000, 6, 200, seed=4)
    og = oracle_mod.OracleGraph(g)
    emit = _emit_set(g)
    T, B = 24, 4
    pl = I.planted_walks(g, B, T, seed=9)
    ll = I.loglikes(77, range(B), T, 200, pl, 1.0, 4.0)
    G = W.Graph.from_arrays(g)
    D = W.Decoder(G, B, 10.0, 300, lattice=1, lattice_beam=6.0)
    D.reset()
    t = torch.from_numpy(ll).cuda()
    pos = [0] * B
    schedule = [([0, 1], 5), ([2, 3], 7), ([3, 0], 6), ([1], 9), ([2], 10), ([0, 1, 3], 8), ([3, 2, 1, 0], 2), ([2], 7),
                ([0], 5), ([1], 10), ([3], 10)]
    for ids, n in schedule:
        n = min(n, *(T - pos[b] for b in ids))
        if n <= 0:
            continue
        x = torch.stack([t[pos[b]:pos[b] + n, b] for b in ids], dim=1).contiguous()
        D.decode_frames(x, streams=np.array(ids, np.int32))
        for b in ids:
            pos[b] += n
    assert pos == [T] * B
    torch.cuda.synchronize()
    for b in range(B):
        _check_stream(D, og, ll[:, b, :], 10.0, 300, 6.0, b, emit)
