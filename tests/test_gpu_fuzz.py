"""Randomised parity sweep of the CUDA path against the oracle: random HCLG-shaped graphs, pdf
counts, beams (finite and infinite), max-active (off, binding, histogram rule), stream counts,
frame counts, decode-call splits and kernel shapes; every stream's path, cost (bit-exact) and
reached-final flag must match."""
import math

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


@pytest.mark.parametrize("case", range(60))
def test_random_configurations(W, torch, oracle_mod, case):
    rng = np.random.default_rng(1000 + case)
    Q = int(rng.integers(200, 6000))
    deg = float(rng.choice([2.5, 3.0, 4.0, 6.0]))
    P = int(rng.integers(20, 400))
    g = I.hclg_graph(Q, deg, P, seed=int(rng.integers(1 << 30)))
    beam = float(rng.choice([4.0, 8.0, 12.0, 16.0, math.inf]))
    alpha = int(rng.choice([0, 20, 150, 1000]))
    hist = bool(rng.random() < 0.25) and alpha > 0 and math.isfinite(beam)
    B = int(rng.integers(1, 10))
    T = int(rng.integers(1, 40))
    sigma, boost = float(rng.choice([0.5, 1.0, 2.0])), float(rng.choice([0.0, 2.0, 4.0]))
    pl = I.planted_walks(g, B, T, seed=int(rng.integers(1 << 30)))
    ll = I.loglikes(int(rng.integers(1 << 30)), range(B), T, P, pl, sigma, boost)
    shape = [(1024, 1), (512, 1), (256, 2)][int(rng.integers(3))] if not hist else (1024, 1)
    opts = dict(threads=shape[0], ctas_per_sm=shape[1], insert_order=int(rng.integers(3)))
    if hist:
        opts["max_active_mode"] = 1
    G = W.Graph.from_arrays(g)
    D = W.Decoder(G, B, beam, alpha, **opts)
    D.reset()
    t = torch.from_numpy(ll).cuda()
    cuts = sorted(set(int(x) for x in rng.integers(1, T + 1, size=int(rng.integers(0, 4))))) + [T]
    t0 = 0
    for c in cuts:
        if c > t0:
            D.decode_frames(t[t0:c].contiguous())
            t0 = c
    res = D.best_paths(cap=4 * T + 64, raise_on_error=False)
    og = oracle_mod.OracleGraph(g)
    for b in range(B):
        try:
            r = og.decode_hist(ll[:, b, :], beam, alpha) if hist else og.decode(ll[:, b, :], beam, alpha)
        except oracle_mod.OracleError as e:   # e.g. no survivor: the GPU must report the same
            assert res["rc"] != 0, (case, b, str(e))
            continue
        n = res["n_arcs"][b]
        assert list(res["arcs"][b, :n]) == list(r.arcs), (case, b)
        assert res["cost"][b] == r.cost32 and res["reached_final"][b] == r.reached_final, (case, b)


@pytest.mark.parametrize("case", range(30))
def test_random_eps_general(W, torch, oracle_mod, case):
    """The same sweep on epsilon-general graphs ("chains of non-emitting arcs"): the
    id-permuted back-off-chain generator (chains of 2-6, skip arcs, positive 2-cycles) and tiny
    random graphs with epsilon arcs in both directions and epsilon cycles (infinite beam too)."""
    rng = np.random.default_rng(5000 + case)
    if case % 3 == 2:
        g = I.random_tiny_graph(int(rng.integers(1 << 30)), n_states=int(rng.integers(3, 9)),
                                n_arcs=int(rng.integers(6, 30)), eps_frac=0.4, eps_back=True)
        P = 4
    else:
        P = int(rng.integers(20, 300))
        g = I.hclg_graph_eps(int(rng.integers(2000, 12000)), float(rng.choice([3.0, 5.0])), P,
                             seed=int(rng.integers(1 << 30)), levels=int(rng.integers(2, 7)),
                             permute_states=bool(rng.random() < 0.8))
    beam = float(rng.choice([5.0, 10.0, 15.0, math.inf]))
    alpha = int(rng.choice([0, 50, 400]))
    B, T = int(rng.integers(1, 8)), int(rng.integers(1, 30))
    pl = I.planted_walks(g, B, T, seed=int(rng.integers(1 << 30)))
    ll = I.loglikes(int(rng.integers(1 << 30)), range(B), T, P, pl, 1.0, float(rng.choice([0.0, 4.0])))
    shape = [(1024, 1), (256, 2)][case % 2]
    G = W.Graph.from_arrays(g)
    D = W.Decoder(G, B, beam, alpha, threads=shape[0], ctas_per_sm=shape[1], insert_order=2 - case % 3)
    D.reset()
    D.decode_frames(torch.from_numpy(ll).cuda())
    res = D.best_paths(cap=8 * T + 64, raise_on_error=False)
    og = oracle_mod.OracleGraph(g)
    for b in range(B):
        try:
            r = og.decode(ll[:, b, :], beam, alpha)
        except oracle_mod.OracleError as e:
            assert res["rc"] != 0, (case, b, str(e))
            continue
        n = res["n_arcs"][b]
        assert list(res["arcs"][b, :n]) == list(r.arcs), (case, b)
        assert res["cost"][b] == r.cost32 and res["reached_final"][b] == r.reached_final, (case, b)
