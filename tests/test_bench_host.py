"""Host-side pieces of bench.py (no GPU): the algorithmic byte model of DESIGN.md §5.4, the
stream partition of the multi-GPU path, decoder options from the command line."""
import argparse

import bench


def test_algorithmic_bytes_model():
    st = {"emit_arcs": 1000, "eps_arcs": 10, "survivors": 100}
    # 4P per stream-frame + 12 per emitting arc + 8 per epsilon arc + 36 per survivor
    assert bench.algorithmic_bytes(st, frames=5, P=200) == 4 * 200 * 5 + 12 * 1000 + 8 * 10 + 36 * 100


def test_rank_streams_partition_is_disjoint_and_complete():
    world, per = 8, 512
    ids = [list(bench.rank_streams(r, world, per)) for r in range(world)]
    flat = [i for chunk in ids for i in chunk]
    assert flat == list(range(world * per))


def test_decoder_opts_from_flags():
    a = argparse.Namespace(threads=512, ctas_per_sm=2, table_slots=0, frames_per_item=0, lattice=8.0, hist=True)
    o = bench.decoder_opts(a)
    assert o == {"threads": 512, "ctas_per_sm": 2, "lattice": 1, "lattice_beam": 8.0, "max_active_mode": 1}
    b = argparse.Namespace(threads=0, ctas_per_sm=0, table_slots=0, frames_per_item=0, lattice=None, hist=False)
    assert bench.decoder_opts(b) == {}
