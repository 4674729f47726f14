"""Host-side logic of the multi-GPU path (row e) with world_size 2 over gloo on CPU:
stream partitioning, partition-independent inputs, and the max-over-ranks reduction."""
import os

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from paper_1910_10032_b200 import inputs as I
    g = I.hclg_graph(5000, 3.0, 200, seed=1)
    ids = bench.rank_streams(rank, world, 3)
    pl = I.planted_walks(g, 3, 12, seed=4, stream0=ids.start)
    ll = I.loglikes(4, ids, 12, 200, pl, 1.0, 4.0)
    import oracle
    og = oracle.OracleGraph(g)
    costs = [og.decode(ll[:, j, :], 12.0, 300).cost for j in range(3)]
    ms, arcs = bench.reduce_over_ranks(dist, "cpu", 10.0 + rank, 100.0 * (rank + 1))
    q.put((rank, list(ids), costs, ms, arcs))
    dist.destroy_process_group()


def test_two_ranks_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = sorted(q.get(timeout=180) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert out[0][1] == [0, 1, 2] and out[1][1] == [3, 4, 5]
    assert all(o[3] == 11.0 and o[4] == 300.0 for o in out)
    # the same global stream decoded by a single process gives the same cost
    from paper_1910_10032_b200 import inputs as I
    import oracle
    g = I.hclg_graph(5000, 3.0, 200, seed=1)
    pl = I.planted_walks(g, 6, 12, seed=4)
    ll = I.loglikes(4, range(6), 12, 200, pl, 1.0, 4.0)
    og = oracle.OracleGraph(g)
    single = [og.decode(ll[:, j, :], 12.0, 300).cost for j in range(6)]
    assert single == out[0][2] + out[1][2]
