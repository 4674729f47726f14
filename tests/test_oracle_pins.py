"""Pins for the CPU oracle (oracle/wfst_oracle.c) against things other than itself:
SPEC worked examples, the fp64 frame-unrolled shortest path and exhaustive path
enumeration (tests/bruteforce.py), exact dyadic arithmetic, and invariants of
beam search that hold at any size.  CPU only."""
import math

import numpy as np
import pytest

import bruteforce as BF
from paper_1910_10032_b200 import inputs as I

INF = math.inf


def _g(n, arcs, finals, start=0):
    src, dst, il, ol, w = zip(*arcs) if arcs else ([], [], [], [], [])
    fin = np.full(n, np.inf)
    for q, f in finals.items():
        fin[q] = f
    return I._mk(n, start, src, dst, il, ol, w, fin)


SPEC_G = lambda: _g(3, [(0, 1, 1, 1, 0.5), (0, 2, 0, 0, 1.0), (1, 2, 2, 2, 0.3)], {2: 0.0})


def test_spec_serial_example(oracle_mod):
    """loglike(ilabel 1)=2.0 at t=0, loglike(ilabel 2)=1.0 at t=1 -> words [1, 2],
    cost (0.5-2.0)+(0.3-1.0) = -2.2 (+ final 0)."""
    og = oracle_mod.OracleGraph(SPEC_G())
    ll = np.array([[2.0, 0.0], [0.0, 1.0]], np.float32)
    r = og.decode(ll, INF, 0)
    assert list(r.olabels) == [1, 2] and r.reached_final == 1
    expect = np.float32(np.float32(np.float32(0.5) - np.float32(2.0)) + np.float32(0.3)) - np.float32(1.0)
    assert r.cost32 == np.float32(expect) and abs(r.cost - (-2.2)) < 1e-6


def test_spec_expand_arithmetic(oracle_mod):
    """start token cost 0, arc weight 0.5, loglike 2.0 -> candidate cost -1.5."""
    og = oracle_mod.OracleGraph(SPEC_G())
    r = og.decode(np.array([[2.0, 0.0]], np.float32), INF, 0, survivors=True)
    assert r.frame_stats[0, 0] == np.float32(-1.5)
    st, ar, co = r.layers[1]
    assert list(st) == [1] and list(co) == [np.float32(-1.5)]


def test_spec_eps_relaxation(oracle_mod):
    """token at 0 (cost 0), epsilon arc 0->2 weight 1.0 -> token at 2 cost 1.0."""
    og = oracle_mod.OracleGraph(SPEC_G())
    r = og.decode(np.zeros((0, 2), np.float32), INF, 0, survivors=True)
    st, ar, co = r.layers[0]
    assert dict(zip(st.tolist(), co.tolist())) == {0: 0.0, 2: 1.0}


def test_spec_eps_chain(oracle_mod):
    """epsilon chain 0->1->2->3, weights 0.1 -> costs 0.1, 0.2, 0.3."""
    g = _g(4, [(0, 1, 0, 0, 0.1), (1, 2, 0, 0, 0.1), (2, 3, 0, 0, 0.1), (3, 3, 1, 0, 1.0)], {3: 0.0})
    r = oracle_mod.OracleGraph(g).decode(np.zeros((0, 1), np.float32), INF, 0, survivors=True)
    st, ar, co = r.layers[0]
    d = dict(zip(st.tolist(), co.tolist()))
    assert all(abs(d[q] - 0.1 * q) < 1e-6 for q in (1, 2, 3))
    assert r.cost32 == co[st.tolist().index(3)] and r.reached_final == 1
    assert len(r.arcs) == 3


def test_empty_utterance(oracle_mod):
    """no frames, start state final cost 0 -> cost 0, empty word sequence;
    a non-final start falls back to reached_final = 0 (reading R10)."""
    r = oracle_mod.OracleGraph(_g(1, [], {0: 0.0})).decode(np.zeros((0, 1), np.float32), INF, 0)
    assert r.cost == 0.0 and r.reached_final == 1 and len(r.olabels) == 0 and len(r.arcs) == 0
    r = oracle_mod.OracleGraph(_g(2, [(0, 1, 1, 0, 1.0)], {1: 0.0})).decode(np.zeros((0, 1), np.float32), INF, 0)
    assert r.cost == 0.0 and r.reached_final == 0


def test_errors(oracle_mod):
    og = oracle_mod.OracleGraph(_g(2, [(0, 1, 1, 0, 1.0)], {1: 0.0}))   # state 1 has no arcs
    with pytest.raises(oracle_mod.OracleError) as e:
        og.decode(np.zeros((2, 1), np.float32), INF, 0)
    assert e.value.rc == 7                                              # NO_SURVIVOR
    og = oracle_mod.OracleGraph(_g(2, [(0, 1, 3, 0, 1.0)], {1: 0.0}))
    with pytest.raises(oracle_mod.OracleError) as e:
        og.decode(np.zeros((1, 2), np.float32), INF, 0)                 # pdf 2 needs P >= 3
    assert e.value.rc == 5


def _tiny_instance(seed):
    g = I.random_tiny_graph(seed)
    rng = np.random.default_rng(seed + 7)
    T = int(rng.integers(1, 6))
    ll = rng.uniform(-3, 0, (T, 4)).astype(np.float32)
    return g, ll


def test_infinite_beam_equals_bruteforce_tiny(oracle_mod):
    """with beam = +inf the oracle is the exact frame-unrolled shortest path:
    compare with DFS enumeration and fp64 trellis 2-best on 300 random <=6-state graphs."""
    n_checked = n_path = 0
    for seed in range(300):
        g, ll = _tiny_instance(seed)
        paths = BF.enumerate_paths(g, ll)
        og = oracle_mod.OracleGraph(g)
        try:
            r = og.decode(ll, INF, 0)
        except oracle_mod.OracleError as e:
            assert e.rc == 7 and not paths, seed
            continue
        pool, fin = BF.best_of_enumeration(paths)
        kb = BF.trellis_kbest(g, ll)
        assert bool(r.reached_final) == fin
        assert abs(r.cost - pool[0][0]) <= 1e-4 * max(1.0, abs(pool[0][0])), seed
        assert abs(kb[0][0] - pool[0][0]) < 1e-9
        n_checked += 1
        gap = pool[1][0] - pool[0][0] if len(pool) > 1 else INF
        if gap > 1e-4:
            canon = BF.canonical_order(g)
            assert [int(canon[a]) for a in r.arcs] == pool[0][1] == kb[0][1], seed
            n_path += 1
    assert n_checked > 250 and n_path > 200


def test_c1_infinite_beam_equals_trellis(oracle_mod):
    """C1 (BASELINE configs[0]): 20 states / 60 arcs / 10 pdfs / 30 frames, infinite beam,
    200 log-likelihood seeds vs the fp64 trellis; tie-free seeds must give the same path."""
    g = I.c1_graph()
    og = oracle_mod.OracleGraph(g)
    canon = BF.canonical_order(g)
    n_tie_free = 0
    for seed in range(1, 201):
        pl = I.planted_walks(g, 1, 30, seed=seed)
        ll = I.loglikes_stream(seed, 0, 30, 10, pl[:, 0], 1.5, 2.0)
        r = og.decode(ll, INF, 0)
        kb = BF.trellis_kbest(g, ll, k=2)
        assert bool(r.reached_final) == kb[0][2]
        assert abs(r.cost - kb[0][0]) <= 1e-4 * max(1.0, abs(kb[0][0]))
        if len(kb) > 1 and kb[1][0] - kb[0][0] > 1e-5 * max(1.0, abs(kb[0][0])):
            assert [int(canon[a]) for a in r.arcs] == kb[0][1]
            n_tie_free += 1
    assert n_tie_free >= 150


def _dyadic_instance(seed, Q=7, E=18, T=6, P=4):
    rng = np.random.default_rng(seed)
    g = I.random_tiny_graph(seed, n_states=Q, n_arcs=E, n_pdfs=P)
    g.weight = (np.round(g.weight * 8) / 8).astype(np.float32)
    g.final = np.where(np.isfinite(g.final), np.round(g.final * 8) / 8, np.inf).astype(np.float32)
    ll = (rng.integers(-24, 1, (T, P)) / 8.0).astype(np.float32)
    return g, ll


def test_dyadic_exact_equals_fp64(oracle_mod):
    """All weights/log-likelihoods multiples of 1/8: fp32 sums are exact, so the oracle's cost
    must equal the fp64 shortest path EXACTLY (a dropped term or wrong sign cannot hide)."""
    n = 0
    for seed in range(200):
        g, ll = _dyadic_instance(seed)
        try:
            r = oracle_mod.OracleGraph(g).decode(ll, INF, 0)
        except oracle_mod.OracleError:
            continue
        kb = BF.trellis_kbest(g, ll, k=1)
        assert r.cost == kb[0][0], seed
        n += 1
    assert n > 100


def _c2_small(seed=2):
    return I.hclg_graph(5000, 6.0, 300, seed=seed)


def _stream_ll(g, seed, s, T, P, preset="clean"):
    pl = I.planted_walks(g, s + 1, T, seed=seed)
    return I.loglikes_stream(seed, s, T, P, pl[:, s], **I.preset(preset))


def test_maxactive_and_cutoff_invariants(oracle_mod):
    """R5/R6: every survivor is under the cutoff; emitting-arc
    survivors strictly below k_alpha number < alpha; when alpha binds, >= alpha tokens survive."""
    g = _c2_small()
    og = oracle_mod.OracleGraph(g)
    for s, (beam, alpha) in enumerate([(10.0, 50), (6.0, 20), (14.0, 200), (INF, 100)]):
        ll = _stream_ll(g, 11, s, 40, 300, "other")
        r = og.decode(ll, beam, alpha, survivors=True)
        used = 0
        for t in range(40):
            best, cut, ka = r.frame_stats[t]
            st, ar, co = r.layers[t + 1]
            assert np.all(co < cut) and np.all(co <= ka)
            if np.isfinite(ka):
                used += 1
                emit = np.array([g.ilabel[BF.canonical_order(g)[a]] != 0 for a in ar])
                assert np.sum(emit & (co < ka)) < alpha
                assert len(st) >= alpha
            assert r.frame_counts[t, 2] == len(st)
        if beam < INF or alpha < 1000:
            assert used > 0 or s == 2


def test_certificate_pruned_equals_exact(oracle_mod):
    """If every token of the exact best path survives pruning, the pruned search returns that
    path (the beam only removes tokens; SURVEY §8.4 pin (iii))."""
    g = _c2_small(5)
    og = oracle_mod.OracleGraph(g)
    canon = BF.canonical_order(g)
    certified = 0
    for s in range(12):
        ll = _stream_ll(g, 21, s, 25, 300, "clean")
        ex = og.decode(ll, INF, 0)
        pr = og.decode(ll, 8.0, 60, survivors=True)
        # tokens (layer, state) along the exact path
        layer, q, ok = 0, g.start, True
        toks = [(0, q)]
        for a in ex.arcs:
            ia = canon[a]
            if g.ilabel[ia] != 0:
                layer += 1
            q = int(g.dst[ia])
            toks.append((layer, q))
        for (k, q) in toks:
            if q not in set(pr.layers[k][0].tolist()):
                ok = False
                break
        if pr.reached_final and ex.reached_final:   # fallback costs (R10) are not comparable
            assert pr.cost >= ex.cost - 1e-3 * max(1, abs(ex.cost))
        if ok:
            certified += 1
            assert np.array_equal(pr.arcs, ex.arcs) and pr.cost32 == ex.cost32
    assert certified >= 3


def test_pruned_path_is_a_real_path(oracle_mod):
    """At any beam / alpha the reported arcs form a connected path from the start consuming
    every frame, ending where the flag says, whose fp64 cost matches the reported fp32 cost."""
    g = _c2_small(7)
    og = oracle_mod.OracleGraph(g)
    canon = BF.canonical_order(g)
    for s, (beam, alpha) in enumerate([(10.0, 10000), (5.0, 30), (12.0, 500)]):
        T = 60
        ll = _stream_ll(g, 31, s, T, 300, "clean")
        r = og.decode(ll, beam, alpha)
        arcs_in = [int(canon[a]) for a in r.arcs]
        cost, end, frames = BF.path_cost_fp64(g, ll, arcs_in)
        assert frames == T
        assert bool(np.isfinite(g.final[end])) == bool(r.reached_final)
        assert abs(cost - r.cost) <= 1e-4 * max(1.0, abs(cost))
        assert [int(g.olabel[a]) for a in arcs_in if g.olabel[a] != 0] == list(r.olabels)


def test_shift_invariance_dyadic(oracle_mod):
    """Adding a constant to every log-likelihood of a frame shifts every candidate of that
    frame equally: with exact (dyadic) arithmetic the pruned path is unchanged and the cost
    moves by exactly -sum(shifts)."""
    for seed in range(60):
        g, ll = _dyadic_instance(seed, Q=8, E=24, T=7, P=4)
        og = oracle_mod.OracleGraph(g)
        shifts = (np.random.default_rng(seed).integers(-8, 9, ll.shape[0]) / 4.0).astype(np.float32)
        try:
            a = og.decode(ll, 1.5, 3)
        except oracle_mod.OracleError:
            continue
        b = og.decode(ll + shifts[:, None], 1.5, 3)
        assert np.array_equal(a.arcs, b.arcs)
        assert b.cost == a.cost - float(shifts.sum())


def test_arc_order_invariance(oracle_mod):
    """Permuting the input arc order changes canonical ids but not the decoded path (as input
    arcs) on tie-free inputs ("independent of arc input order")."""
    g = _c2_small(9)
    rng = np.random.default_rng(0)
    perm = rng.permutation(g.n_arcs)
    h = I._mk(g.n_states, g.start, g.src[perm], g.dst[perm], g.ilabel[perm], g.olabel[perm], g.weight[perm], g.final)
    og, oh = oracle_mod.OracleGraph(g), oracle_mod.OracleGraph(h)
    cg, ch = BF.canonical_order(g), BF.canonical_order(h)
    for s in range(4):
        ll = _stream_ll(g, 41, s, 30, 300, "clean")
        a, b = og.decode(ll, 10.0, 100), oh.decode(ll, 10.0, 100)
        assert [int(cg[x]) for x in a.arcs] == [int(perm[ch[x]]) for x in b.arcs]
        assert a.cost32 == b.cost32


def test_infinite_beam_survivors_are_reachable_set(oracle_mod):
    """With beam = +inf every state reachable in exactly t frames survives at layer t."""
    for seed in range(40):
        g, ll = _tiny_instance(seed)
        try:
            r = oracle_mod.OracleGraph(g).decode(ll, INF, 0, survivors=True)
        except oracle_mod.OracleError:
            continue
        reach = {g.start}
        def eclose(S):
            S = set(S)
            while True:
                n = {int(g.dst[i]) for i in range(g.n_arcs) if g.ilabel[i] == 0 and int(g.src[i]) in S} - S
                if not n:
                    return S
                S |= n
        reach = eclose(reach)
        assert set(r.layers[0][0].tolist()) == reach
        for t in range(ll.shape[0]):
            reach = eclose({int(g.dst[i]) for i in range(g.n_arcs) if g.ilabel[i] != 0 and int(g.src[i]) in reach})
            assert set(r.layers[t + 1][0].tolist()) == reach


def test_batch_driver_matches_single(oracle_mod):
    g = _c2_small(3)
    og = oracle_mod.OracleGraph(g)
    T, B, P = 20, 5, 300
    pl = I.planted_walks(g, B, T, seed=3)
    ll = I.loglikes(3, range(B), T, P, pl, 1.0, 4.0)
    cost, reached, rc, cnt, arcs, n_arcs = og.decode_batch(ll, 10.0, 200, 3, arcs_cap=128)
    for b in range(B):
        r = og.decode(ll[:, b, :], 10.0, 200)
        assert rc[b] == 0 and cost[b] == r.cost32 and list(arcs[b, :n_arcs[b]]) == list(r.arcs)
        assert cnt[b] == int(r.frame_counts[:, 3].sum() + r.frame_counts[:, 4].sum())


def test_eps_general_infinite_beam_equals_bruteforce(oracle_mod):
    """Epsilon arcs in both directions with positive-weight epsilon cycles (inputs
    random_tiny_graph(eps_back=True)): with beam = +inf the oracle's cost equals the exhaustive
    minimum over complete paths (DFS enumeration, fp64), and its path when the best is unique."""
    n_checked = n_path = n_cyc = 0
    for seed in range(200):
        g = I.random_tiny_graph(seed, n_states=5, n_arcs=12, eps_frac=0.35, eps_back=True)
        e = g.ilabel == 0
        n_cyc += int(np.any(g.dst[e] < g.src[e]))
        rng = np.random.default_rng(seed + 11)
        T = int(rng.integers(1, 5))
        ll = rng.uniform(-3, 0, (T, 4)).astype(np.float32)
        paths = BF.enumerate_paths(g, ll, simple_eps=True)
        og = oracle_mod.OracleGraph(g)
        try:
            r = og.decode(ll, INF, 0)
        except oracle_mod.OracleError as ex:
            assert ex.rc == 7 and not paths, seed
            continue
        pool, fin = BF.best_of_enumeration(paths)
        assert bool(r.reached_final) == fin, seed
        assert abs(r.cost - pool[0][0]) <= 1e-4 * max(1.0, abs(pool[0][0])), seed
        n_checked += 1
        second = next((p[0] for p in pool[1:] if p[1] != pool[0][1]), INF)
        if second - pool[0][0] > 1e-4:
            canon = BF.canonical_order(g)
            assert [int(canon[a]) for a in r.arcs] == pool[0][1], seed
            n_path += 1
    assert n_checked > 150 and n_path > 100 and n_cyc > 100


def test_eps_general_order_invariance(oracle_mod):
    """R7 (least fixed point, any relaxation order): on the epsilon-general, id-permuted
    generator (back-off chains of 5, skip arcs, positive 2-cycles) a permutation of the input arc
    order -- which changes the canonical ids and hence the closure's visiting order -- leaves the
    decoded path (as input arcs) and its cost unchanged at finite beam and max-active."""
    g = I.hclg_graph_eps(6000, 6.0, 300, seed=12)
    perm = np.random.default_rng(1).permutation(g.n_arcs)
    h = I._mk(g.n_states, g.start, g.src[perm], g.dst[perm], g.ilabel[perm], g.olabel[perm], g.weight[perm], g.final)
    og, oh = oracle_mod.OracleGraph(g), oracle_mod.OracleGraph(h)
    cg, ch = BF.canonical_order(g), BF.canonical_order(h)
    n_eps = 0
    for s in range(4):
        ll = _stream_ll(g, 51, s, 30, 300, "clean")
        a, b = og.decode(ll, 10.0, 150), oh.decode(ll, 10.0, 150)
        pa = [int(cg[x]) for x in a.arcs]
        assert pa == [int(perm[ch[x]]) for x in b.arcs]
        assert a.cost32 == b.cost32
        n_eps += sum(int(g.ilabel[x] == 0) for x in pa)
    assert n_eps > 0
