"""The CUDA path (through the C ABI) on the hand-derived convention cases of
tests/convention_cases.py: survivors per layer, per-frame (best, beam cutoff, k_alpha), path,
olabels, cost and flag must equal the values derived by hand -- the same bar the oracle meets
in tests/test_oracle_conventions.py, so both sides are pinned to the paper's readings
independently of each other.  Run with several kernel shapes and call splits."""
import numpy as np
import pytest

import convention_cases as CC

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


SHAPES = [dict(), dict(threads=256, ctas_per_sm=2), dict(table_slots=64, overflow_slots=64)]


@pytest.mark.parametrize("shape", range(len(SHAPES)))
@pytest.mark.parametrize("case", CC.CASES, ids=[c["name"] for c in CC.CASES])
def test_gpu_convention_case(W, torch, case, shape):
    g = CC.graph(case)
    ll = CC.loglikes(case)
    T = ll.shape[0]
    G = W.Graph.from_arrays(g)
    assert [int(x) for x in np.argsort(G.canonical_perm())] == case["canon"]
    B = 3   # the case on lane 1, neighbours decode the same input (lanes must not interact)
    D = W.Decoder(G, B, case["beam"], case["alpha"], debug_costs=1, **SHAPES[shape])
    D.reset()
    if T:
        D.decode_frames(torch.from_numpy(np.ascontiguousarray(np.repeat(ll[:, None, :], B, axis=1))).cuda())
    torch.cuda.synchronize()
    for lane in range(B):
        for k, L in enumerate(case["layers"]):
            st, ar, co = D.debug_layer(lane, k)
            assert dict(zip(st.tolist(), co.tolist())) == {q: float(np.float32(c)) for q, c in L.items()}
        if case["fstats"]:
            fs, _ = D.frame_stats(lane)
            for t, exp in enumerate(case["fstats"]):
                assert tuple(float(x) for x in fs[t]) == tuple(float(np.float32(x)) for x in exp)
        r = D.best_path(lane)
        assert r["reached_final"] == case["reached"]
        assert r["cost32"] == np.float32(case["cost"])
        assert list(r["arcs"]) == case["path"]
        assert list(r["olabels"]) == case["olabels"]
