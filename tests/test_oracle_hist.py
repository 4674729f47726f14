"""Pins of the oracle's histogram max-active (row f4, reading R16).  On dyadic inputs (weights
and log-likelihoods multiples of 1/8, beam 8: bin width 1/128) every fp32 operation is exact,
so at the first frame where max-active binds -- identical state in both runs before it -- the
histogram cutoff must equal the closed form best + (floor((k_alpha - best) * 128) + 1) / 128
with k_alpha the exact alpha-th smallest in-beam cost (the exact rule R6, pinned elsewhere)."""
import math

import numpy as np

from paper_1910_10032_b200 import inputs as I

INF = math.inf


def _dyadic_graph():
    g = I.hclg_graph(3000, 6, 200, seed=4)
    g.weight = (np.round(g.weight * 8) / 8).astype(np.float32)
    g.final = np.where(np.isfinite(g.final), np.round(g.final * 8) / 8, np.inf).astype(np.float32)
    return g


def test_hist_cutoff_closed_form_at_first_binding_frame(oracle_mod):
    g = _dyadic_graph()
    og = oracle_mod.OracleGraph(g)
    checked = 0
    for seed in range(12):
        pl = I.planted_walks(g, 1, 30, seed=seed)
        ll = I.loglikes_stream(100 + seed, 0, 30, 200, pl[:, 0], 1.0, 1.0)
        ll = (np.round(ll * 8) / 8).astype(np.float32)
        for alpha in (20, 60, 150):
            ex = og.decode(ll, 8.0, alpha)
            hi = og.decode_hist(ll, 8.0, alpha)
            bind = np.nonzero(np.isfinite(ex.frame_stats[:, 2]))[0]
            if bind.size == 0:
                continue
            t0 = int(bind[0])
            # identical before the first binding frame, and the same best / beam cutoff at it
            assert np.array_equal(ex.frame_stats[:t0 + 1, :2], hi.frame_stats[:t0 + 1, :2])
            assert np.all(~np.isfinite(hi.frame_stats[:t0, 2]))
            best, ka = float(ex.frame_stats[t0, 0]), float(ex.frame_stats[t0, 2])
            want = best + (math.floor((ka - best) * 128) + 1) / 128
            got = float(np.nextafter(hi.frame_stats[t0, 2], np.float32(INF)))
            assert got == want, (seed, alpha, t0, got, want)
            # the histogram keeps everything the exact rule keeps at that frame
            assert hi.frame_counts[t0, 2] >= ex.frame_counts[t0, 2]
            checked += 1
    assert checked >= 20


def test_hist_equals_exact_when_max_active_never_binds(oracle_mod):
    g = I.hclg_graph(3000, 6, 200, seed=4)
    og = oracle_mod.OracleGraph(g)
    pl = I.planted_walks(g, 1, 40, seed=1)
    ll = I.loglikes_stream(7, 0, 40, 200, pl[:, 0], 1.0, 4.0)
    ex = og.decode(ll, 10.0, 100000)
    hi = og.decode_hist(ll, 10.0, 100000)
    assert list(ex.arcs) == list(hi.arcs) and ex.cost32 == hi.cost32
    assert np.array_equal(ex.frame_stats, hi.frame_stats)


def test_hist_infinite_beam_keeps_everything(oracle_mod):
    """beam = +inf: one bin holds every candidate, the cutoff is +inf -> max-active has no
    effect in the histogram rule (documented in R16)."""
    g = I.random_tiny_graph(3, n_states=6, n_arcs=16, n_pdfs=4)
    og = oracle_mod.OracleGraph(g)
    ll = np.random.default_rng(0).uniform(-3, 0, (5, 4)).astype(np.float32)
    a = og.decode(ll, INF, 0)
    h = og.decode_hist(ll, INF, 1)
    assert list(a.arcs) == list(h.arcs) and a.cost32 == h.cost32
