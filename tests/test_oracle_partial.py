"""Pins of the oracle's settled prefix (row f2, reading R15): properties the mathematics fixes
for any correct settled prefix -- every complete decode of a longer input starts with it (all
later paths extend a current survivor), it only grows, it ends with an emitting arc (or is
empty), and with one survivor it is that survivor's whole traceback cut after its last
emitting arc."""
import math
import os
import sys

import numpy as np

from paper_1910_10032_b200 import inputs as I

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import bruteforce as BF  # noqa: E402

INF = math.inf


def _is_prefix(a, b):
    return len(a) <= len(b) and list(a) == list(b[:len(a)])


def test_settled_prefix_is_prefix_of_every_later_decode(oracle_mod):
    g = I.hclg_graph(3000, 6, 200, seed=4)
    og = oracle_mod.OracleGraph(g)
    emit = g.ilabel[BF.canonical_order(g)] != 0
    n_nonempty = 0
    for b in range(4):
        pl = I.planted_walks(g, 4, 60, seed=9)
        ll = I.loglikes_stream(77, b, 60, 200, pl[:, b], 1.0, 4.0)
        prev = np.zeros(0, np.int64)
        for L in (5, 12, 20, 33, 47, 60):
            sp = og.settled_prefix(ll[:L], 10.0, 300)
            assert _is_prefix(prev, sp), (b, L)                  # only grows
            assert len(sp) == 0 or emit[sp[-1]]                  # cut after an emitting arc
            assert int(emit[sp].sum()) <= L
            for L2 in (L, min(60, L + 7), 60):                   # every later decode extends it
                full = og.decode(ll[:L2], 10.0, 300)
                assert _is_prefix(sp, full.arcs), (b, L, L2)
            prev = sp
            n_nonempty += len(sp) > 0
    assert n_nonempty >= 12


def test_single_survivor_settles_everything(oracle_mod):
    """beam -> tiny: one survivor per frame, so the settled prefix is its whole traceback cut
    after the last emitting arc = the best path of the prefix decode."""
    g = I.hclg_graph(2000, 3, 50, seed=3)
    og = oracle_mod.OracleGraph(g)
    emit = g.ilabel[BF.canonical_order(g)] != 0
    pl = I.planted_walks(g, 1, 30, seed=2)
    ll = I.loglikes_stream(5, 0, 30, 50, pl[:, 0], 1.0, 4.0)
    sp = og.settled_prefix(ll, 10.0, 1)
    full = list(og.decode(ll, 10.0, 1).arcs)
    while full and not emit[full[-1]]:
        full.pop()
    assert list(sp) == full and len(sp) >= 30
