"""C-ABI library checks that need no GPU: it builds for sm_100a, loads, exports every symbol
include/wfst_gpu.h declares, and its host-only paths (Eq. 1/Eq. 2, graph validation before
any device work) behave as documented."""
import json
import os
import re
import subprocess

import numpy as np
import pytest

from paper_1910_10032_b200 import build as B
from paper_1910_10032_b200 import inputs as I

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


@pytest.fixture(scope="module")
def W():
    B.build()
    from paper_1910_10032_b200 import wfst_gpu
    wfst_gpu.lib()
    return wfst_gpu


def _declared():
    src = open(os.path.join(ROOT, "include", "wfst_gpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(wfst_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol(W):
    names = _declared()
    assert len(names) >= 20
    out = subprocess.run(["nm", "-D", "--defined-only", W.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (wfst_[a-z0-9_]+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    assert set(W.SYMBOLS) == set(names)
    assert W.lib().wfst_abi_version() == 2


def test_sass_is_sm100a(W):
    out = subprocess.run(["cuobjdump", "--list-elf", W.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_memory_formulas(W):
    """Eq. 1 and Eq. 2 with the worked values of P:126 and SPEC S:64-66."""
    g = json.load(open(os.path.join(GOLD, "memory_formulas.json")))
    for c in g["eq1"]:
        assert W.eq1_bytes(c["Q"], c["E"], c["EE"]) == c["bytes"]
    for c in g["eq2"]:
        assert W.eq2_bytes(c["alpha"], c["nc"], c["nl"]) == c["bytes"]
    assert abs(W.eq2_bytes(10000, 1, 1) / 2 ** 20 - 5.8) < 0.01           # "5.8MB"
    assert abs(W.eq2_bytes(10000, 5000, 500) / 2 ** 30 - 5.5) < 0.02      # "about 5.5GB"


def test_loader_errors_without_device(W, tmp_path):
    """Validation happens before any device work, so these run on a CPU-only box."""
    with pytest.raises(W.WfstError) as e:
        W.Graph.load(os.path.join(GOLD, "spec_eps_cycle.txt"))
    assert e.value.status == "EPS_CYCLE"
    p = tmp_path / "bad.txt"
    p.write_text("0 1 1 1 0.5\n0 2 x 0 1.0\n")
    with pytest.raises(W.WfstError) as e:
        W.Graph.load(str(p))
    assert e.value.status == "PARSE" and "line 2" in str(e.value)
    p.write_text("0 1 1 1 0.5 9\n")
    with pytest.raises(W.WfstError) as e:
        W.Graph.load(str(p))
    assert e.value.status == "PARSE" and "line 1" in str(e.value)
    g = I._mk(2, 0, [0], [5], [1], [0], [1.0], [np.inf, 0.0])          # dangling dst
    with pytest.raises(W.WfstError) as e:
        W.Graph.from_arrays(g)
    assert e.value.status == "GRAPH_INVALID"
    g = I._mk(2, 0, [0, 1], [1, 0], [0, 0], [0, 0], [0.5, -0.5], [np.inf, 0.0])   # weight-0 cycle
    with pytest.raises(W.WfstError) as e:
        W.Graph.from_arrays(g)
    assert e.value.status == "EPS_CYCLE"
    g = I._mk(2, 0, [0, 1], [1, 0], [0, 0], [0, 0], [0.5, -0.75], [np.inf, 0.0])  # negative cycle
    with pytest.raises(W.WfstError) as e:
        W.Graph.from_arrays(g)
    assert e.value.status == "EPS_CYCLE"
    g = I._mk(2, 5, [0], [1], [1], [0], [1.0], [np.inf, 0.0])          # bad start
    with pytest.raises(W.WfstError) as e:
        W.Graph.from_arrays(g)
    assert e.value.status == "GRAPH_INVALID"


def test_packed_row_views(W):
    """The binding's per-stream views over a packed partial-paths result (wfst_get_partial_paths_packed):
    stream i is a[off[i] : off[i] + min(n[i], cap)], in any packing order; indexing, negative indices,
    slices, iteration and len behave like a list of arrays."""
    a = np.array([7, 8, 9, 1, 2, 3, 4, 5], np.int32)
    off = np.array([3, 0, 8, 5], np.int64)   # stream 0 at 3, stream 1 at 0, stream 2 empty, stream 3 at 5
    n = np.array([2, 3, 0, 9], np.int32)     # stream 3 overflowed cap = 3: only cap entries were stored
    rows = W._Rows(a, n, off, 3)
    assert len(rows) == 4
    assert rows[0].tolist() == [1, 2] and rows[1].tolist() == [7, 8, 9] and rows[2].tolist() == []
    assert rows[3].tolist() == [3, 4, 5]     # (over cap: the cap entries that were stored)
    assert rows[-3].tolist() == [7, 8, 9]
    assert [r.tolist() for r in rows[1:3]] == [[7, 8, 9], []]
    assert [r.size for r in rows] == [2, 3, 0, 3]
    with pytest.raises(IndexError):
        rows[4]
