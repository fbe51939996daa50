"""Multi-rank (world_size 2, gloo, CPU) check of the data-parallel decomposition.

Each rank takes its slice of the balanced schedule with the same helper bench.py
uses (paper_2505_22208_b200.dist.shard_ids), computes its worker's loss and
gradient SUM with the oracle (rank r = simulated worker r, denoise streams keyed
by r*B + b), and the ranks all-reduce over gloo; /G must reproduce the
reference's single-process G-worker step (S/trainer.cpp:258-320). The 128-byte
NCCL unique-id exchange path (broadcast of bytes from rank 0) is exercised too.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import cases

CFG = (32, 2, 8, 5.0, 4)
G, B = 2, 4


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _workload():
    import paper_2505_22208_b200 as pk
    pool = cases.mixed_batch(pk, D=CFG[4], seed=31, count=40)
    sched = pk.plan(np.diff(pool["atom_ptr"]), G, B, num_splits=3, seed=5, mode="balanced")
    return pk, pool, sched


def _rank_main(rank, port, out):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(G), LOCAL_RANK=str(rank), MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port))
    from paper_2505_22208_b200.dist import Dist, minibatch_ids, shard_ids
    from oracle import port as oracle_port
    dist = Dist("gloo")
    try:
        pk, pool, sched = _workload()
        P = oracle_port()
        table = cases.random_table(CFG[4], seed=8)
        params = P.init_params(CFG, 4)
        step = 1
        mine = shard_ids(sched, step, dist.rank, G, B)
        full = minibatch_ids(sched, step, G, B)
        # worker_step evaluates worker `rank` of the packed G*B mini-batch
        mb = pk.select(pool, full)
        loss, grads = P.worker_step(CFG, G, B, dist.rank, mb, table, params, seed=9, step=step)
        uid = dist.bcast_bytes(bytes(range(128)) if dist.rank == 0 else None)
        tot_loss = dist.allreduce(loss, "sum")
        tot_grads = dist.allreduce_array(grads, "sum")
        out.put((dist.rank, mine.tolist(), full.tolist(), tot_loss, tot_grads, uid))
    finally:
        dist.close()


@pytest.mark.timeout(300)
def test_two_rank_allreduce_matches_reference_step(oracle_ref):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, port, q)) for r in range(G)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=240) for _ in range(G)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, mine0, full, loss0, g0, uid0), (r1, mine1, _, loss1, g1, uid1) = res
    assert mine0 + mine1 == full and not set(mine0) & set(mine1)
    assert uid0 == uid1 == bytes(range(128))
    assert loss0 == loss1 and np.array_equal(g0, g1)  # every rank holds the same reduced values

    pk, pool, sched = _workload()
    from paper_2505_22208_b200.dist import minibatch_ids
    mb = pk.select(pool, minibatch_ids(sched, 1, G, B))
    table = cases.random_table(CFG[4], seed=8)
    params = oracle_ref.init_params(CFG, 4)
    ref = oracle_ref.train_step(CFG, G, B, mb, table, params, np.zeros_like(params), seed=9, step=1, clip=1e9)
    assert abs(loss0 / G - ref["loss"]) <= 1e-12 * abs(ref["loss"])
    assert np.abs(g0 * (1.0 / G) - ref["grads"]).max() <= 1e-12 * np.abs(ref["grads"]).max()


def test_shards_partition_every_minibatch():
    from paper_2505_22208_b200.dist import minibatch_ids, shard_ids
    pk, pool, sched = _workload()
    for step in range(sched["n_batches"]):
        parts = [shard_ids(sched, step, r, G, B) for r in range(G)]
        assert np.array_equal(np.concatenate(parts), minibatch_ids(sched, step, G, B))
        for r in range(G):
            assert len(parts[r]) == B
