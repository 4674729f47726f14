"""Boundary stream semantics (include/wfst_gpu.h "Conventions"): a decoder's calls are ordered
among themselves across CUDA streams, and result calls wait for that decoder's work only.

* one decoder driven from two CUDA streams alternately gives the results of a one-stream run;
* two decoders on two streams give the oracle's results each;
* best paths of a small decoder return while a long decode of another decoder (on another
  stream, a few SMs) is still running: no device-wide synchronisation.
"""
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


def _inputs(n_streams, T, P=300, seed=5):
    g = I.hclg_graph(8000, 5.0, P, seed=seed)
    pl = I.planted_walks(g, n_streams, T, seed=seed + 1)
    return g, I.loglikes(seed + 2, range(n_streams), T, P, pl, 1.0, 4.0)


def test_one_decoder_two_streams(W, torch, oracle_mod):
    g, ll = _inputs(6, 40)
    G = W.Graph.from_arrays(g)
    t = torch.from_numpy(ll).cuda()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    D = W.Decoder(G, 6, 10.0, 400)
    D.reset(stream=s1)
    for k, t0 in enumerate(range(0, 40, 5)):   # chunks alternate between the two streams
        s = s1 if k % 2 == 0 else s2
        D.decode_frames(t[t0:t0 + 5].contiguous(), stream=s)
    res = D.best_paths(cap=256)
    og = oracle_mod.OracleGraph(g)
    for b in range(6):
        r = og.decode(ll[:, b, :], 10.0, 400)
        assert res["cost"][b] == r.cost32 and list(res["arcs"][b, :res["n_arcs"][b]]) == list(r.arcs)


def test_two_decoders_two_streams(W, torch, oracle_mod):
    g, ll = _inputs(4, 30)
    G = W.Graph.from_arrays(g)
    t = torch.from_numpy(ll).cuda()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    D1, D2 = W.Decoder(G, 4, 10.0, 400, max_ctas=8), W.Decoder(G, 4, 10.0, 400, max_ctas=8)
    D1.reset(stream=s1)
    D2.reset(stream=s2)
    for t0 in range(0, 30, 10):
        D1.decode_frames(t[t0:t0 + 10].contiguous(), stream=s1)
        D2.decode_frames(t[t0:t0 + 10].contiguous(), stream=s2)
    r1, r2 = D1.best_paths(cap=256), D2.best_paths(cap=256)
    og = oracle_mod.OracleGraph(g)
    for b in range(4):
        r = og.decode(ll[:, b, :], 10.0, 400)
        for res in (r1, r2):
            assert res["cost"][b] == r.cost32 and list(res["arcs"][b, :res["n_arcs"][b]]) == list(r.arcs)


def test_results_do_not_wait_for_other_decoders(W, torch):
    g, ll = _inputs(4, 1500, seed=9)
    G = W.Graph.from_arrays(g)
    big = torch.from_numpy(ll).cuda()
    small = big[:10, :1].contiguous()
    s_big, s_small = torch.cuda.Stream(), torch.cuda.Stream()
    Dbig = W.Decoder(G, 4, 10.0, 2000, max_ctas=4)           # 4 SMs, 1500 frames
    Dsmall = W.Decoder(G, 1, 10.0, 2000, max_ctas=4)
    Dbig.reset(stream=s_big)
    Dsmall.reset(stream=s_small)
    torch.cuda.synchronize()
    done = torch.cuda.Event()
    Dbig.decode_frames(big, stream=s_big)
    done.record(s_big)
    Dsmall.decode_frames(small, stream=s_small)
    Dsmall.best_paths(cap=128)
    still_running = not done.query()
    torch.cuda.synchronize()
    assert still_running, "best_paths of one decoder waited for another decoder's work"
    Dbig.sync()
