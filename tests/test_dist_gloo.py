"""Multi-rank host logic on CPU (gloo, world_size 2): pair and host sharding,
the stamp merge by allreduce(MAX), and host-sharded estimation reassemble the
single-rank result.  The per-rank stamps come from the oracle's serial pool
(nowLBP1 of the rank's shard), encoded as the fast layout's
stamp word (T << 5) | rank."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_1810_13132_b200 import (all_gather_shards, merge_stamps_tensor, reduce_scatter_max,
                                   shard_range)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _stamps(now: np.ndarray, tick: int, prev: np.ndarray) -> np.ndarray:
    out = prev.copy()
    hit = now > 0
    out[hit] = (tick << 5) | now[hit].astype(np.int64)
    return out.astype(np.int32)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tr = synth.CONFIGS["tiny"]
        cfg = oracle.PoolConfig(b=5, k=4, z=1 << 12)
        stamps = np.zeros(cfg.z, np.int32)
        ok = True
        for t in range(6):
            pairs = synth.generate(tr, t)
            a, b = shard_range(len(pairs), rank, world)
            mine = oracle.Pool(cfg, "serial")
            mine.begin_slice()
            mine.scan(pairs[a:b])
            local = torch.from_numpy(_stamps(mine.now(), t + 1, stamps))
            merged = merge_stamps_tensor(local).numpy()
            whole = oracle.Pool(cfg, "serial")
            whole.begin_slice()
            whole.scan(pairs)
            ok &= np.array_equal(merged, _stamps(whole.now(), t + 1, stamps))
            stamps = merged
        # host-sharded estimation reassembles the single-rank vector
        ref = oracle.Pool(cfg, "serial")
        for t in range(6):
            ref.slice(synth.generate(tr, t))
        M = ref.readout()
        hosts = tr.host_ids()
        h0, h1 = shard_range(len(hosts), rank, world)
        part = torch.from_numpy(ref.estimate(M, hosts[h0:h1]))
        sizes = [shard_range(len(hosts), r, world) for r in range(world)]
        bufs = [torch.empty(e - s, dtype=torch.float64) for s, e in sizes]
        dist.all_gather(bufs, part)
        ok &= np.array_equal(torch.cat(bufs).numpy(), ref.estimate(M, hosts))
        # sharded merge plumbing (slide_merged 'sharded'): reduce-scatter(MAX)
        # of u8 nowLBP1 deltas, then an all-gather of per-rank register shards
        tr2 = synth.CONFIGS["tiny"]
        pairs = synth.generate(tr2, 9)
        a, b = shard_range(len(pairs), rank, world)
        mine = oracle.Pool(cfg, "serial")
        mine.begin_slice()
        mine.scan(pairs[a:b])
        delta = torch.from_numpy(mine.now().copy())
        n = cfg.z // world
        shard = torch.empty(n, dtype=torch.uint8)
        reduce_scatter_max(delta, shard)
        whole = oracle.Pool(cfg, "serial")
        whole.begin_slice()
        whole.scan(pairs)
        ok &= np.array_equal(shard.numpy(), whole.now()[rank * n:(rank + 1) * n])
        regs = torch.zeros(cfg.z, dtype=torch.uint8)
        regs[rank * n:(rank + 1) * n] = shard
        all_gather_shards(regs)
        ok &= np.array_equal(regs.numpy(), whole.now())
        # sparse exchange plumbing (slide_merged 'sparse'): per-owner records of
        # the touched BDRs ((j - owner start) << 5 | rank), counts then records
        # all-to-all, folded into the owner's shard with a per-byte max
        from paper_1810_13132_b200.vbdr import _all_to_all
        now = mine.now()
        recs = [np.array([((j - o * n) << 5) | int(now[j]) for j in np.flatnonzero(now[o * n:(o + 1) * n]) + o * n],
                         dtype=np.int32) for o in range(world)]
        counts = torch.tensor([len(r) for r in recs], dtype=torch.int64)
        recv_counts = torch.empty_like(counts)
        _all_to_all(recv_counts, counts, None, None)
        send = torch.from_numpy(np.concatenate(recs))
        recv = torch.empty(int(recv_counts.sum()), dtype=torch.int32)
        _all_to_all(recv, send, recv_counts.tolist(), counts.tolist())
        folded = np.zeros(n, np.uint8)
        r = recv.numpy().view(np.uint32)
        np.maximum.at(folded, (r >> 5).astype(np.int64), (r & 31).astype(np.uint8))
        ok &= np.array_equal(folded, whole.now()[rank * n:(rank + 1) * n])
        # max-over-ranks timing reduction used by bench.py
        t_local = torch.tensor([1.0 + rank], dtype=torch.float64)
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
        ok &= float(t_local[0]) == float(world)
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


def test_two_rank_merge_and_host_sharding():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert results == {0: True, 1: True}


def test_merge_is_noop_without_group():
    x = torch.arange(10, dtype=torch.int32)
    assert merge_stamps_tensor(x) is x
