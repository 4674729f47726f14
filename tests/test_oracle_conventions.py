"""Pins of the oracle's finite-beam conventions (R3, R5, R6 order, R7, R9, R10)
against hand-derived worked examples (tests/convention_cases.py): survivors per layer, the
per-frame (best, beam cutoff, k_alpha), the one-best path, its olabels, cost and reached-final
flag.  The paper leaves these choices open (P:150-151 accepts nondeterministic pruning), so
only a hand computation can pin them; tests/test_oracle_mutations.py shows that each of the
plausible alternative readings fails at least one case here.  CPU only."""
import numpy as np
import pytest

import convention_cases as CC


@pytest.mark.parametrize("case", CC.CASES, ids=[c["name"] for c in CC.CASES])
def test_convention_case(oracle_mod, case):
    g = CC.graph(case)
    og = oracle_mod.OracleGraph(g)
    ll = CC.loglikes(case)
    assert [int(x) for x in np.argsort(og.perm())] == case["canon"], "canonical arc numbering (S:32)"
    r = og.decode(ll, case["beam"], case["alpha"], survivors=True)
    got_layers = [dict(zip(st.tolist(), [float(c) for c in co])) for st, _, co in r.layers]
    assert got_layers == [{q: float(np.float32(c)) for q, c in L.items()} for L in case["layers"]]
    for t, (best, cut, ka) in enumerate(case["fstats"]):
        assert tuple(float(x) for x in r.frame_stats[t]) == (float(np.float32(best)), float(np.float32(cut)),
                                                            float(np.float32(ka)))
    assert r.reached_final == case["reached"]
    assert r.cost32 == np.float32(case["cost"])
    assert list(r.arcs) == case["path"]
    assert list(r.olabels) == case["olabels"]


def test_cases_are_self_consistent():
    """The hand-written canonical numbering follows S:32 (stable by (src, emitting first)), and
    every path arc leaves the state the previous arc entered (start at 0)."""
    for case in CC.CASES:
        arcs = case["arcs"]
        order = sorted(range(len(arcs)), key=lambda i: (arcs[i][0], arcs[i][2] == 0, i))
        assert [order.index(i) for i in range(len(arcs))] == case["canon"], case["name"]
        q = 0
        for c in case["path"]:
            a = arcs[case["canon"].index(c)]
            assert a[0] == q, case["name"]
            q = a[1]
