"""N>1 host logic on CPU: world_size-2 gloo process group (127.0.0.1).

Each process hosts a contiguous block of the m workers (as bench.py/train
do, one process per GPU). Checked against the compiled-reference golden
vectors / numpy oracle:
  * sharding and per-worker minibatch order are bit-exact and disjoint;
  * the hierarchical average (local subtree -> cross-process sum -> x 1/m)
    equals the reference's allreduce_average bitwise for m = 4, 8.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import parnn_oracle as O


def _tree(vs, lo, hi):
    if hi - lo == 1:
        return np.array(vs[lo], dtype=np.float64, copy=True)
    mid = lo + (hi - lo) // 2
    return _tree(vs, lo, mid) + _tree(vs, mid, hi)


def hierarchical_average(local_vectors, layout, allreduce_sum):
    """The arithmetic the device Averager performs across processes (local
    subtree sum -> cross-process sum -> x 1/m), restated in numpy for the gloo
    test: equals allreduce_average bitwise when m and world are powers of two.
    The device path itself is tested on the GPU (tests/test_gpu_avg.py)."""
    assert len(local_vectors) == layout.local
    return allreduce_sum(_tree(local_vectors, 0, layout.local)) * (1.0 / layout.workers)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, m, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    from paper_1507_01239_b200.parallel import epoch_orders, shard_rows, worker_layout

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lay = worker_layout(m, world, rank)
        n, seed, B = 1000, 11, 16
        rows = shard_rows(n, lay, seed)
        orders = epoch_orders(rows.shape[1], B, lay, seed, epochs=2)
        got = [None] * world
        dist.all_gather_object(got, (rank, rows.tolist(), [[o.tolist() for o in w] for w in orders]))
        vecs = [np.random.default_rng(100 + r).standard_normal(37) for r in lay.ranks]

        def allreduce_sum(x):
            t = torch.from_numpy(x.copy())
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
            return t.numpy()

        avg = hierarchical_average(vecs, lay, allreduce_sum)
        q.put((rank, got, avg))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("m", [4, 8])
def test_two_process_sharding_and_average(m):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, m, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict()
    for _ in range(2):
        rank, got, avg = q.get(timeout=240)
        res[rank] = (got, avg)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got = res[0][0]
    # sharding: the union over processes is the reference partition, shards disjoint
    all_rows = np.concatenate([np.asarray(g[1]) for g in sorted(got)])
    ref = np.stack(O.partition_rows(1000, m, 11))
    assert np.array_equal(all_rows, ref.astype(all_rows.dtype))
    assert len(set(all_rows.ravel().tolist())) == all_rows.size
    # per-worker epoch orders: worker r draws from Rng(11 + r)
    for rank, rows, orders in got:
        for i, w_orders in enumerate(orders):
            r = rank * (m // 2) + i
            rng = O.Rng(11 + r)
            for e in range(2):
                exp = np.stack(O.minibatch_rows(len(rows[i]), 16, rng.next_u64()))
                assert np.array_equal(np.asarray(w_orders[e]), exp.astype(np.int64))
    # averaging: identical on both processes and bitwise equal to the reference tree mean
    vecs = [np.random.default_rng(100 + r).standard_normal(37) for r in range(m)]
    ref_avg = O.allreduce_average(vecs, m)
    assert np.array_equal(res[0][1], res[1][1])
    assert np.array_equal(res[0][1], ref_avg)


def test_layout_errors():
    from paper_1507_01239_b200.parallel import worker_layout
    from paper_1507_01239_b200.parnn import ParnnError
    lay = worker_layout(32, 8, 3)
    assert (lay.rank0, lay.local) == (12, 4)
    with pytest.raises(ParnnError):
        worker_layout(6, 4, 0)
    with pytest.raises(ParnnError):
        worker_layout(0, 1, 0)
