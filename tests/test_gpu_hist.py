"""Row f4 (NEXT): the histogram max-active rule (R16) on the GPU vs the oracle's decode_hist,
bit-exact (same fp32 operations), on flat posteriors where max-active binds every frame."""
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


@pytest.mark.parametrize("graph,beam,alpha,preset", [((3000, 6, 200, 4), 10.0, 150, (1.0, 0.0)),
                                                     ((50_000, 6, 2000, 2), 10.0, 3000, (1.0, 0.0)),
                                                     ((50_000, 6, 2000, 2), 10.0, 1000, (1.0, 4.0))])
def test_hist_max_active_parity(W, torch, oracle_mod, graph, beam, alpha, preset):
    Q, deg, P, seed = graph
    g = I.hclg_graph(Q, deg, P, seed=seed)
    og = oracle_mod.OracleGraph(g)
    T, B = 40, 6
    pl = I.planted_walks(g, B, T, seed=5)
    ll = I.loglikes(31, range(B), T, P, pl, *preset)
    G = W.Graph.from_arrays(g)
    D = W.Decoder(G, B, beam, alpha, max_active_mode=1)
    D.reset()
    D.decode_frames(torch.from_numpy(ll).cuda())
    res = D.best_paths(cap=4 * T + 64)
    bound = 0
    for b in range(B):
        r = og.decode_hist(ll[:, b, :], beam, alpha)
        n = res["n_arcs"][b]
        assert list(res["arcs"][b, :n]) == list(r.arcs), b
        assert res["cost"][b] == r.cost32 and res["reached_final"][b] == r.reached_final
        fs, fc = D.frame_stats(b)
        assert np.array_equal(fs.view(np.uint32), r.frame_stats.view(np.uint32)), b
        assert np.array_equal(fc[:, 2], r.frame_counts[:, 2]), b   # survivors per frame
        bound += int(np.isfinite(fs[:, 2]).sum())
    assert bound >= 20   # max-active bound on many frames


def test_hist_mode_rejects_bad_mode(W):
    g = I.hclg_graph(2000, 3, 50, seed=1)
    G = W.Graph.from_arrays(g)
    with pytest.raises(W.WfstError):
        W.Decoder(G, 2, 10.0, 100, max_active_mode=2)
