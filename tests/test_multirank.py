"""Multi-rank host logic on CPU (gloo, world size 2): sharding and the deterministic reduction.

The device path reduces per-batch FP64 payloads across ranks with NCCL
(engine.Engine.reduce_partials). Here the same gather / tree logic runs with
gloo on host tensors, with payloads computed by the CPU oracle, and must
reproduce the single-process result bitwise (deterministic mode) or within
reassociation error (fast mode, all_reduce).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2209_13027_b200.execution import allreduce_partials, gather_batch_partials, shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _payload(acc: O.Acc) -> np.ndarray:
    return np.concatenate([acc.c11.ravel(), acc.c22.ravel(), acc.s1.ravel(), acc.s2.ravel(), acc.g1, acc.g2,
                           [float(acc.n)], acc.n_class.astype(np.float64)])


def _problem():
    rng = np.random.default_rng(3)
    m, p, q, classes, batch = 37, 9, 8, 4, 4  # 10 batches, the last one short
    v1 = rng.uniform(size=(m, p, q)).astype(np.float32).astype(np.float64)
    v2 = rng.uniform(size=(m, p, q)).astype(np.float32).astype(np.float64)
    lab = rng.integers(0, classes, m)
    return v1, v2, lab, classes, batch


def _batch_payloads(v1, v2, lab, classes, batch, batches):
    out = []
    geom = O.Geometry(3, 3)
    for r in batches:
        acc = O.layer_stats(v1[r.start:r.stop, None], v2[r.start:r.stop, None], lab[r.start:r.stop], geom, True,
                            classes, batch, O.Pool())
        out.append(_payload(acc))
    return np.stack(out)


def _tree(rows: np.ndarray) -> np.ndarray:
    level = [rows[i] for i in range(rows.shape[0])]
    while len(level) > 1:
        nxt = [level[i] + level[i + 1] for i in range(0, len(level) - 1, 2)]
        if len(level) % 2:
            nxt.append(level[-1])
        level = nxt
    return level[0]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        v1, v2, lab, classes, batch = _problem()
        gb = O.batch_ranges(len(lab), batch)
        mine = shard_range(len(gb), rank, world)
        local = _batch_payloads(v1, v2, lab, classes, batch, [gb[b] for b in mine])
        allp = gather_batch_partials(torch.from_numpy(local), len(gb), world)
        det = _tree(allp.numpy())
        fast = torch.from_numpy(_tree(local))
        dist.all_reduce(fast)
        q.put((rank, list(mine), det, fast.numpy()))
    finally:
        dist.destroy_process_group()


def test_shard_range_covers_batches_contiguously():
    for n in (1, 4, 10, 240, 2392):
        for world in (1, 2, 3, 4, 8):
            got = [b for r in range(world) for b in shard_range(n, r, world)]
            assert got == list(range(n))
            sizes = [len(shard_range(n, r, world)) for r in range(world)]
            assert max(sizes) - min(sizes) <= 1


def test_two_rank_reduction_matches_single_process():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    v1, v2, lab, classes, batch = _problem()
    gb = O.batch_ranges(len(lab), batch)
    single = _tree(_batch_payloads(v1, v2, lab, classes, batch, gb))
    res.sort()
    assert res[0][1] + res[1][1] == list(range(len(gb)))
    for _, _, det, fast in res:
        assert np.array_equal(det, single)  # deterministic mode: bitwise GPU-count invariant
        assert np.allclose(fast, single, rtol=1e-12, atol=1e-12)
    # and the merged payload is the oracle's whole-dataset accumulator
    whole = O.layer_stats(v1[:, None], v2[:, None], lab, O.Geometry(3, 3), True, classes, batch, O.Pool())
    assert np.array_equal(single, _payload(whole))


def _empty_rank_worker(rank, world, port, q):
    """world 3 over 2 batches: rank 2 owns none and must still join both reductions."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        v1, v2, lab, classes, _ = _problem()
        v1, v2, lab, batch = v1[:8], v2[:8], lab[:8], 4
        gb = O.batch_ranges(len(lab), batch)
        mine = shard_range(len(gb), rank, world)
        if len(mine):
            local = _batch_payloads(v1, v2, lab, classes, batch, [gb[b] for b in mine])
        else:
            plen = 2 * 9 * 9 + 2 * 9 * classes + 2 * 9 + 1 + classes
            local = np.zeros((0, plen))
        det = _tree(gather_batch_partials(torch.from_numpy(local), len(gb), world).numpy())
        fast = allreduce_partials(torch.from_numpy(local), lambda t: torch.from_numpy(_tree(t.numpy())))
        q.put((rank, len(mine), det, fast.numpy()))
    finally:
        dist.destroy_process_group()


def test_rank_without_batches_joins_reductions():
    """More ranks than batches (engine.reduce_partials): the batchless rank contributes a zero
    payload in fast mode and padding in deterministic mode; nobody hangs, all agree."""
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_empty_rank_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    v1, v2, lab, classes, _ = _problem()
    gb = O.batch_ranges(8, 4)
    single = _tree(_batch_payloads(v1[:8], v2[:8], lab[:8], classes, 4, gb))
    assert [n for _, n, _, _ in res] == [1, 1, 0]
    for _, _, det, fast in res:
        assert np.array_equal(det, single)
        assert np.allclose(fast, single, rtol=1e-12, atol=1e-12)
