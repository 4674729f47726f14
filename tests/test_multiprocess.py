"""Host-side logic of the multi-GPU path (row e) with world_size 2 over gloo on CPU: stream
partitioning (weak and strong), partition-independent inputs, the max-over-ranks reduction, the
distinct-device count, and bench.py's host-side result gather.  Each rank stands in for a GPU by
decoding its streams with the oracle (test infrastructure); rank 0's gathered table must equal a
single-process decode of every global stream."""
import os

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _digest(r):
    import zlib
    return (int(np.float32(r.cost32).view(np.uint32)), int(r.reached_final), len(r.arcs),
            zlib.crc32(np.ascontiguousarray(r.arcs, np.int32).tobytes()))


def _streams_ll(g, ids, T=12, P=200):
    from paper_1910_10032_b200 import inputs as I
    pl = I.planted_walks(g, len(ids), T, seed=4, stream0=ids.start)
    return I.loglikes(4, ids, T, P, pl, 1.0, 4.0)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from paper_1910_10032_b200 import inputs as I
    import oracle
    g = I.hclg_graph(5000, 3.0, 200, seed=1)
    og = oracle.OracleGraph(g)
    out = {}
    for name, ids in (("weak", bench.rank_streams(rank, world, 3)),
                      ("strong", bench.partition(7, world, rank))):
        ll = _streams_ll(g, ids)
        rs = [og.decode(ll[:, j, :], 12.0, 300) for j in range(len(ids))]
        out[name] = bench.gather_results(dist, world, ids, [_digest(r) for r in rs])
    ms, arcs = bench.reduce_over_ranks(dist, "cpu", 10.0 + rank, 100.0 * (rank + 1))
    allv = [None] * world
    dist.all_gather_object(allv, ("host", "gpu0"))          # both ranks share one "device"
    q.put((rank, out, ms, arcs, len(set(allv))))
    dist.destroy_process_group()


def test_two_ranks_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=240) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    (_, out0, ms0, arcs0, ndev0), (_, out1, ms1, _, _) = res
    assert out1["weak"] is None and out1["strong"] is None          # only rank 0 receives the gather
    assert ms0 == ms1 == 11.0 and arcs0 == 300.0 and ndev0 == 1
    assert sorted(out0["weak"]) == list(range(6)) and sorted(out0["strong"]) == list(range(7))
    # the same global streams decoded by one process give the same results
    from paper_1910_10032_b200 import inputs as I
    import oracle
    g = I.hclg_graph(5000, 3.0, 200, seed=1)
    og = oracle.OracleGraph(g)
    for name, n in (("weak", 6), ("strong", 7)):
        ll = _streams_ll(g, range(n))
        single = {b: _digest(og.decode(ll[:, b, :], 12.0, 300)) for b in range(n)}
        assert out0[name] == single, name
