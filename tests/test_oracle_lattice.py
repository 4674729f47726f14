"""Pins of the oracle's lattice step (row f1, readings R13-R14): exhaustive path enumeration on
tiny graphs with exact (dyadic) arithmetic, the SPEC worked example of grouping,
the lattice-beam = 0 special case (the one-best path) and invariants that hold at any size."""
import math
import os
import sys

import numpy as np
import pytest

from paper_1910_10032_b200 import inputs as I

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import bruteforce as BF  # noqa: E402

INF = float("inf")


def _dyadic_instance(seed, Q=6, E=16, T=4, P=4):
    rng = np.random.default_rng(seed)
    g = I.random_tiny_graph(seed, n_states=Q, n_arcs=E, n_pdfs=P)
    g.weight = (np.round(g.weight * 8) / 8).astype(np.float32)
    g.final = np.where(np.isfinite(g.final), np.round(g.final * 8) / 8, np.inf).astype(np.float32)
    ll = (rng.integers(-24, 1, (T, P)) / 8.0).astype(np.float32)
    return g, ll


def _brute_lattice(g, ll):
    """fp64 enumeration: per (segment k, canonical arc) and per (layer k, state), the minimum
    slack (cost - best) of the complete paths through it (R10 pool: final paths if any)."""
    paths = BF.enumerate_paths(g, ll)
    pool, fin = BF.best_of_enumeration(paths)
    if not pool:
        return None
    best = pool[0][0]
    canon = BF.canonical_order(g)
    inv = np.empty_like(canon)
    inv[canon] = np.arange(len(canon))
    arc_slack, tok_slack = {}, {}
    for cost, arcs, _ in pool:
        s = cost - best
        k, q = 0, g.start
        toks = [(0, q)]
        keys = []
        for a in arcs:
            if g.ilabel[a] != 0:
                k += 1
            keys.append((k, int(inv[a])))
            q = int(g.dst[a])
            toks.append((k, q))
        for key in keys:
            arc_slack[key] = min(arc_slack.get(key, INF), s)
        for key in toks:
            tok_slack[key] = min(tok_slack.get(key, INF), s)
    return best, fin, arc_slack, tok_slack


def _kept(r, lb):
    """(segment, arc) -> path slack of the oracle's final lattice (pslack <= lb)."""
    out = {}
    for k, (arc, _src, _dst, _sl) in enumerate(r.segments):
        for a, ps in zip(arc, r.pslack[k]):
            if ps <= lb:
                out[(k, int(a))] = float(ps)
    return out


@pytest.mark.parametrize("lb", [0.0, 0.5, 1.25, 3.0, 8.0])
def test_lattice_equals_path_enumeration(oracle_mod, lb):
    """Infinite beam, exact arithmetic: the final lattice holds exactly the arcs that lie on a
    complete path with slack <= lattice_beam, each with the slack of the best such path, and
    gamma of every token is the best complete-path slack through it."""
    n = 0
    for seed in range(120):
        g, ll = _dyadic_instance(seed)
        bf = _brute_lattice(g, ll)
        og = oracle_mod.OracleGraph(g)
        if bf is None:
            continue
        best, fin, arc_slack, tok_slack = bf
        r = og.lattice(ll, INF, 0, lb)
        assert r.lattice_best == best == r.cost, seed
        want = {key: s for key, s in arc_slack.items() if s <= lb}
        assert _kept(r, lb) == want, seed
        for k, L in enumerate(r.layers):
            for j, q in enumerate(L[0]):
                bfs = tok_slack.get((k, int(q)), INF)
                if bfs <= lb:   # gamma is exact for tokens that a kept arc reaches
                    assert r.gamma[k][j] == bfs, (seed, k, int(q))
                else:
                    assert r.gamma[k][j] > lb, (seed, k, int(q))
        n += 1
    assert n > 80


def test_lattice_beam_zero_is_the_one_best_path(oracle_mod):
    """Tie-free instances: with lattice_beam = 0 the final lattice is exactly the best path."""
    n = 0
    for seed in range(200):
        g, ll = _dyadic_instance(seed + 1000)
        paths = BF.enumerate_paths(g, ll)
        pool, _ = BF.best_of_enumeration(paths)
        if len(pool) < 2 or pool[1][0] - pool[0][0] < 0.125:
            continue
        og = oracle_mod.OracleGraph(g)
        r = og.lattice(ll, INF, 0, 0.0)
        canon = BF.canonical_order(g)
        k, want = 0, set()
        for a in r.arcs:
            if g.ilabel[canon[a]] != 0:
                k += 1
            want.add((k, int(a)))
        assert set(_kept(r, 0.0)) == want, seed
        n += 1
    assert n > 50


def test_spec_grouping_example(oracle_mod):
    """tokens (state 2, 1.0), (state 2, 1.4), (state 5, 1.2) -> two groups, state 2's
    representative is the 1.0 token, all kept at lattice-beam 8; at 0.3 the 1.4 token (slack
    0.4) is dropped."""
    g = I.Wfst(n_states=6, start=0,
               src=np.array([0, 0, 0], np.int32), dst=np.array([2, 2, 5], np.int32),
               ilabel=np.array([1, 1, 1], np.int32), olabel=np.zeros(3, np.int32),
               weight=np.array([1.0, 1.4, 1.2], np.float32),
               final=np.array([INF, INF, 0, INF, INF, 0], np.float32))
    og = oracle_mod.OracleGraph(g)
    ll = np.zeros((1, 1), np.float32)
    r = og.lattice(ll, INF, 0, 8.0)
    arc, src, dst, sl = r.segments[1]
    states = r.layers[1][0]
    groups = {}
    for a, j, s in zip(arc, dst, sl):
        groups.setdefault(int(states[j]), []).append((int(a), float(s)))
    assert sorted(groups) == [2, 5]
    assert groups[2][0] == (0, 0.0) and groups[2][1][0] == 1
    assert abs(groups[2][1][1] - 0.4) < 1e-6 and groups[5] == [(2, 0.0)]
    assert r.layers[1][1][list(states).index(2)] == 0          # representative = the 1.0 arc
    r = og.lattice(ll, INF, 0, 0.3)
    assert sorted(int(a) for a in r.segments[1][0]) == [0, 2]


def test_segments_complete_at_infinite_beams(oracle_mod):
    """beam = lattice_beam = inf: segment k holds every emitting arc of layer k-1 and every
    epsilon arc of layer k (all of them reach a kept token), each token's winner arc with slack
    0, and no slack is negative."""
    for seed in range(60):
        g, ll = _dyadic_instance(seed + 5000, Q=7, E=20, T=5)
        og = oracle_mod.OracleGraph(g)
        try:
            r = og.lattice(ll, INF, 0, INF)
        except oracle_mod.OracleError:
            continue
        canon = BF.canonical_order(g)
        src_c, il_c = g.src[canon], g.ilabel[canon]
        emit_deg = np.bincount(src_c[il_c != 0], minlength=g.n_states)
        eps_deg = np.bincount(src_c[il_c == 0], minlength=g.n_states)
        for k, (arc, src, dst, sl) in enumerate(r.segments):
            n_want = int(eps_deg[r.layers[k][0]].sum())
            if k > 0:
                n_want += int(emit_deg[r.layers[k - 1][0]].sum())
            assert len(arc) == n_want, (seed, k)
            assert np.all(sl >= 0)
            pairs = set(zip(arc.tolist(), dst.tolist()))
            for j, a in enumerate(r.layers[k][1]):
                if a >= 0:
                    assert (int(a), j) in pairs
                    assert sl[(arc == a) & (dst == j)][0] == 0.0


def test_finite_beam_segment_invariants(oracle_mod):
    """C2-shaped graph, beam 10 / alpha 300: every segment arc passes its frame's cutoff,
    joins the right tokens (src(arc), dst(arc)), has 0 <= slack <= lattice_beam, recomputes to
    the same fp32 slack, and the final lattice contains the one-best path at path slack 0."""
    g = I.hclg_graph(3000, 6, 200, seed=4)
    og = oracle_mod.OracleGraph(g)
    canon = BF.canonical_order(g)
    src_c, dst_c, il_c, w_c = g.src[canon], g.dst[canon], g.ilabel[canon], g.weight[canon]
    pl = I.planted_walks(g, 1, 25, seed=9)
    ll = I.loglikes_stream(77, 0, 25, 200, pl[:, 0], 1.0, 4.0)
    lb = 6.0
    r = og.lattice(ll, 10.0, 300, lb)
    for k, (arc, src, dst, sl) in enumerate(r.segments):
        cut_b = np.float32(10.0) if k == 0 else r.frame_stats[k - 1, 1]
        cut_a = np.float32(INF) if k == 0 else r.frame_stats[k - 1, 2]
        st_k, _, co_k = r.layers[k]
        for a, i, j, s in zip(arc, src, dst, sl):
            emitting = il_c[a] != 0
            st_s, _, co_s = r.layers[k - 1] if emitting else r.layers[k]
            assert st_s[i] == src_c[a] and st_k[j] == dst_c[a]
            c = np.float32(co_s[i] + w_c[a])
            if emitting:
                c = np.float32(c - ll[k - 1, il_c[a] - 1])
            assert c < cut_b and c <= cut_a
            assert np.float32(c - co_k[j]) == s and 0 <= s <= lb
    kb = 0
    for a in r.arcs:
        if il_c[a] != 0:
            kb += 1
        arc_k, _, _, _ = r.segments[kb]
        assert r.pslack[kb][list(arc_k).index(a)] == 0.0
    assert not math.isinf(r.lattice_best)
