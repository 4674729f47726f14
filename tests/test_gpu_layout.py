"""Log-likelihood column layouts (reading R2, include/wfst_gpu.h opts.ll_columns).

Layout 0 (default): column = ilabel - 1.  Layout 1: column = ilabel,
column 0 unused.  The same scores in layout 1 are layout 0's matrix with one leading column, so
the GPU in layout 1 on [junk | ll] must equal the oracle (layout 0) on ll, bit for bit; a matrix
only wide enough for layout 0 is rejected in layout 1 instead of being read one column off."""
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


@pytest.mark.parametrize("host", [False, True])
def test_ilabel_columns_equal_pdf_columns(W, torch, oracle_mod, host):
    P = 400
    g = I.hclg_graph(20_000, 6.0, P, seed=11)
    og = oracle_mod.OracleGraph(g)
    T, B, beam, alpha = 40, 5, 10.0, 500
    pl = I.planted_walks(g, B, T, seed=4)
    ll = I.loglikes(17, range(B), T, P, pl, **I.preset("clean"))
    # column 0 of the ilabel layout is unused: fill it with values that would change every path
    junk = np.full((T, B, 1), 1e3, np.float32)
    ll1 = np.ascontiguousarray(np.concatenate([junk, ll], axis=2))
    G = W.Graph.from_arrays(g)
    D = W.Decoder(G, B, beam, alpha, ll_columns=1)
    D.reset()
    if host:
        D.decode_frames_host(ll1, chunk_frames=7)
    else:
        D.decode_frames(torch.from_numpy(ll1).cuda())
    res = D.best_paths(cap=4 * T + 64)
    for b in range(B):
        r = og.decode(ll[:, b, :], beam, alpha)
        n = res["n_arcs"][b]
        assert list(res["arcs"][b, :n]) == list(r.arcs), b
        assert res["cost"][b] == r.cost32 and res["reached_final"][b] == r.reached_final


def test_ilabel_columns_reject_pdf_width(W, torch):
    P = 50
    g = I.hclg_graph(2000, 3, P, seed=1)
    G = W.Graph.from_arrays(g)
    width = G.info().max_pdf + 1          # wide enough for layout 0 only
    ll = torch.zeros((3, 2, width), dtype=torch.float32, device="cuda")
    D0 = W.Decoder(G, 2, 10.0, 100)
    D0.reset()
    D0.decode_frames(ll)                     # layout 0 accepts it
    D1 = W.Decoder(G, 2, 10.0, 100, ll_columns=1)
    D1.reset()
    with pytest.raises(W.WfstError, match="PDF_RANGE|too small"):
        D1.decode_frames(ll)
    with pytest.raises(W.WfstError):
        W.Decoder(G, 2, 10.0, 100, ll_columns=2)
