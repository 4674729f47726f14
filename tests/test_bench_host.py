"""Host-side pieces of bench.py (no GPU): the algorithmic byte model of SURVEY §8.5, the stream
partitions of the multi-GPU path (weak: C3, strong: C5), the self-launcher command, result
digests, decoder options from the command line, the traffic tag check."""
import argparse
import json
import os

import numpy as np

import bench
from paper_1910_10032_b200 import inputs as I


def test_algorithmic_bytes_model():
    st = {"emit_arcs": 1000, "eps_arcs": 10, "survivors": 100, "candidates": 300, "select_entries": 50}
    # 16 n_src + 12 n_arc_e + 4 P + 8 n_cand + 16 n_surv + 16 n_arc_eps + 4 n_select
    assert bench.algorithmic_bytes(st, frames=5, P=200) == \
        16 * 100 + 12 * 1000 + 4 * 200 * 5 + 8 * 300 + 16 * 100 + 16 * 10 + 4 * 50


def test_rank_streams_partition_is_disjoint_and_complete():
    world, per = 8, 512
    ids = [list(bench.rank_streams(r, world, per)) for r in range(world)]
    flat = [i for chunk in ids for i in chunk]
    assert flat == list(range(world * per))


def test_strong_partition_c5():
    """C5 (BASELINE configs[4]): 4096 streams split 4096/N over N = 1, 2, 4, 8 (and ragged N)."""
    c = I.CONFIGS["c5"]
    assert c["scaling"] == "strong" and c["streams"] == 4096
    for n in (1, 2, 3, 4, 7, 8):
        blocks = [bench.config_streams(c, r, n) for r in range(n)]
        assert [i for b in blocks for i in b] == list(range(4096))
        assert max(map(len, blocks)) - min(map(len, blocks)) <= 1
        if 4096 % n == 0:
            assert all(len(b) == 4096 // n for b in blocks)
    c3 = I.CONFIGS["c3"]
    assert [bench.config_streams(c3, r, 4).start for r in range(4)] == [0, 512, 1024, 1536]


def test_launcher_cmd():
    cmd = bench.launcher_cmd(["--gpus", "4", "--config", "c5"], 4, 29555)
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd and "--master-port=29555" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--config", "c5"] and cmd[-5].endswith("bench.py")


def test_result_digest():
    res = dict(cost=np.array([1.5, 2.0], np.float32), reached_final=np.array([1, 0], np.int32),
               n_arcs=np.array([3, 2], np.int32), arcs=np.array([[4, 5, 6, 9], [1, 2, 7, 7]], np.int32))
    a, b = bench.result_digest(res, 0), bench.result_digest(res, 1)
    assert a[:3] == (int(np.float32(1.5).view(np.uint32)), 1, 3) and a != b
    res2 = dict(res, arcs=np.array([[4, 5, 6, 0], [1, 2, 0, 0]], np.int32))   # beyond n_arcs: ignored
    assert bench.result_digest(res2, 0) == a and bench.result_digest(res2, 1) == b


def test_gather_single_rank():
    out = bench.gather_results(None, 1, range(3, 6), ["a", "b", "c"])
    assert out == {3: "a", 4: "b", 5: "c"}


def test_decoder_opts_from_flags():
    a = argparse.Namespace(threads=512, ctas_per_sm=2, table_slots=0, frames_per_item=0, lattice=8.0, hist=True)
    o = bench.decoder_opts(a)
    assert o == {"threads": 512, "ctas_per_sm": 2, "lattice": 1, "lattice_beam": 8.0, "max_active_mode": 1}
    b = argparse.Namespace(threads=0, ctas_per_sm=0, table_slots=0, frames_per_item=0, lattice=None, hist=False)
    assert bench.decoder_opts(b) == {}


def test_traffic_only_for_this_build(tmp_path, monkeypatch):
    """roofline.traffic comes from an ncu capture tagged with the kernel sources' hash; a capture
    of another build is refused."""
    prof = tmp_path / "profiles"
    prof.mkdir()
    monkeypatch.setattr(bench, "ROOT", str(tmp_path))
    os.makedirs(tmp_path / "paper_1910_10032_b200" / "csrc")
    (tmp_path / "paper_1910_10032_b200" / "csrc" / "k.cu").write_text("kernel v1")
    sha = bench.kernel_source_sha()
    (prof / "r09_traffic.json").write_text(json.dumps({"dram_bytes_per_launch": 5e9, "kernel_src_sha": sha,
                                                       "config": "c3/clean"}))
    t, src = bench.measured_traffic("c3", "clean")
    assert t == 5e9 and sha in src
    (tmp_path / "paper_1910_10032_b200" / "csrc" / "k.cu").write_text("kernel v2")
    t, src = bench.measured_traffic("c3", "clean")
    assert t is None and "no ncu capture" in src


def test_bench_launcher_two_ranks_gloo():
    """`bench.py --gpus 2` launches its own two ranks (torch.distributed.run, gloo here): C5's
    4096 streams are split 2048/2048 (strong scaling), C3 is weak-scaled (512 per rank); each
    rank's stand-in results reach rank 0's gather exactly once, equal to a single process's."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for cfg, n, scaling in (("c5", 4096, "strong"), ("c3", 1024, "weak")):
        out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--config", cfg,
                              "--launcher-selftest"], capture_output=True, text=True, timeout=600, cwd=root)
        assert out.returncode == 0, out.stderr[-2000:]
        line = json.loads([x for x in out.stdout.splitlines() if x.startswith("{")][-1])
        assert line == {"selftest": "launcher", "config": cfg, "world": 2, "streams": n, "expected_streams": n,
                        "scaling": scaling, "ok": True}
