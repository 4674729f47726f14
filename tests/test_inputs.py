"""The seeded input generators (paper_1910_10032_b200/inputs.py) — CPU only."""
import json
import math
import os

import numpy as np

from paper_1910_10032_b200 import inputs as I

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _splitmix_py(z: int) -> int:
    """splitmix64 finaliser in plain Python integers (independent of numpy's uint64 wrap)."""
    M = (1 << 64) - 1
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
    return z ^ (z >> 31)


def test_loglike_hash_matches_plain_python():
    seed, stream, T, P = 30003, 77, 3, 11
    ll = I.loglikes_stream(seed, stream, T, P, None, 1.0, 0.0)
    M = (1 << 64) - 1
    sw = _splitmix_py((seed + 0x9E3779B97F4A7C15) & M)
    scale = np.float32(1.0 * math.sqrt(6.0))
    for t in range(T):
        for p in range(P):
            key = (stream << 40) | (t << 20) | p
            h = _splitmix_py(((key ^ sw) + 0x9E3779B97F4A7C15) & M)
            u0 = np.float32(h >> 41) * np.float32(2.0 ** -23)
            u1 = np.float32((h >> 18) & 0x7FFFFF) * np.float32(2.0 ** -23)
            x = np.float32(np.float32(np.float32(u0 + u1) - np.float32(1.0)) * scale)
            assert ll[t, p].view(np.uint32) == np.float32(x + np.float32(0.0)).view(np.uint32)


def test_loglikes_golden_and_determinism():
    with open(os.path.join(GOLD, "loglikes_head.json")) as f:
        cases = json.load(f)
    for c in cases:
        ll = I.loglikes_stream(c["seed"], c["stream"], c["T"], c["P"], c["planted"], c["sigma"], c["boost"])
        assert [int(x) for x in ll.view(np.uint32).ravel()] == c["bits"]


def test_loglike_distribution_and_boost():
    ll = I.loglikes_stream(5, 3, 200, 400, np.arange(200) % 400, 1.0, 4.0)
    base = I.loglikes_stream(5, 3, 200, 400, None, 1.0, 0.0)
    d = ll - base
    assert np.all(d[np.arange(200), np.arange(200) % 400] == np.float32(4.0)) or \
        np.allclose(d[np.arange(200), np.arange(200) % 400], 4.0, atol=1e-5)
    mask = np.ones_like(d, bool)
    mask[np.arange(200), np.arange(200) % 400] = False
    assert np.all(d[mask] == 0)
    assert abs(float(base.std()) - 1.0) < 0.02 and abs(float(base.mean())) < 0.02
    assert base.min() >= -math.sqrt(6.0) - 1e-5 and base.max() <= math.sqrt(6.0) + 1e-5


def test_c1_graph_shape():
    g = I.c1_graph()
    assert g.n_states == 20 and g.n_arcs == 60
    eps = g.ilabel == 0
    assert eps.sum() >= 6 and np.all(g.src[eps] < g.dst[eps])
    assert np.bincount(g.src, minlength=20).max() >= 8
    assert np.isfinite(g.final).sum() >= 2
    assert (g.olabel != 0).sum() >= 5
    assert len(set(zip(g.src.tolist(), g.dst.tolist()))) == g.n_arcs   # no parallel arcs
    assert g.max_pdf <= 9
    # epsilon chain of length >= 2 (0 -> 3 -> 7 -> 12)
    e = {(int(s), int(d)) for s, d in zip(g.src[eps], g.dst[eps])}
    assert (0, 3) in e and (3, 7) in e and (7, 12) in e


def test_hclg_generator_targets():
    g = I.hclg_graph(50_000, 6.0, 2000, seed=2)
    assert g.n_states == 50_000
    assert abs(g.n_arcs / g.n_states - 6.0) < 0.05
    eps = g.ilabel == 0
    assert np.all(g.src[eps] < g.dst[eps])         # epsilon arcs low -> high: acyclic
    assert 0 < eps.mean() < 0.05
    assert g.max_pdf < 2000 and g.src.min() >= 0 and g.dst.max() < g.n_states
    deg = np.bincount(g.src, minlength=g.n_states)
    assert deg.max() >= 9000                         # unigram hub fan-out
    assert np.isfinite(g.final).any() and not np.isfinite(g.final[g.n_states - 1])
    g2 = I.hclg_graph(50_000, 6.0, 2000, seed=2)
    assert np.array_equal(g.dst, g2.dst) and np.array_equal(g.weight, g2.weight)
    g3 = I.hclg_graph(20_000, 3.0, 500, seed=3)
    assert abs(g3.n_arcs / g3.n_states - 3.0) < 0.05


def test_planted_walks_valid_and_partition_independent():
    g = I.hclg_graph(20_000, 3.0, 500, seed=3)
    a = I.planted_walks(g, 6, 40, seed=9)
    b = I.planted_walks(g, 3, 40, seed=9, stream0=3)
    assert a.shape == (40, 6) and np.array_equal(a[:, 3:], b)
    assert a.min() >= 0 and a.max() < 500


def test_text_roundtrip(tmp_path):
    g = I.c1_graph()
    p = tmp_path / "c1.txt"
    I.write_text(g, str(p))
    h = I.read_text(str(p))
    assert h.n_states == g.n_states and np.array_equal(h.src, g.src) and np.array_equal(h.weight, g.weight)
    assert np.array_equal(h.final, g.final)


def test_eps_general_generator_shape():
    """hclg_graph_eps: back-off chains of `levels` epsilon arcs, skip arcs, positive epsilon
    2-cycles, epsilon arcs to lower ids, scattered state ids, every epsilon weight > 0."""
    g = I.hclg_graph_eps(20000, 5.0, 400, seed=3, levels=5)
    e = g.ilabel == 0
    assert np.all(g.weight[e] > 0)
    assert np.any(g.dst[e] < g.src[e]) and np.any(g.dst[e] > g.src[e])
    pairs = set(zip(g.src[e].tolist(), g.dst[e].tolist()))
    assert sum((d, s) in pairs for s, d in pairs) >= 20          # 2-cycles
    # longest epsilon chain without repeating a state (DFS over the epsilon subgraph, from sources)
    out = {}
    for s, d in zip(g.src[e].tolist(), g.dst[e].tolist()):
        out.setdefault(s, []).append(d)
    def depth(q, seen):
        return max((1 + depth(d, seen | {d}) for d in out.get(q, []) if d not in seen), default=0)
    assert max(depth(q, {q}) for q in list(out)[:300]) >= 4
    assert g.start != 0 or g.n_states < 2   # ids permuted (start no longer state 0)
