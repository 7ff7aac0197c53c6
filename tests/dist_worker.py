"""Worker for tests/test_gpu_dist.py: one rank of a multi-rank VBDR run on ONE
GPU with the gloo backend (collectives on the CPU, so ranks never spin on the
GPU waiting for each other), or a single rank with the NCCL backend
(VBDR_TEST_BACKEND=nccl: the NCCL calls and symmetric-memory rendezvous of
every merge execute on the device tensors, with a group of one).  Every rank scans its shard of each 'tiny' slice,
closes it with slide_merged(mode), estimates its shard of the hosts; rank 0
gathers everything and checks it against the oracle.  Exit code 0 = parity."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
from paper_1810_13132_b200 import VBDR, shard_range, slide_merged  # noqa: E402
from paper_1810_13132_b200.vbdr import PeerMerge, make_config  # noqa: E402


def main(mode: str):
    backend = os.environ.get("VBDR_TEST_BACKEND", "gloo")
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    dist.init_process_group(backend, device_id=dev if backend == "nccl" else None)
    rank, world = dist.get_rank(), dist.get_world_size()
    assert backend == "gloo" or world == 1, "one GPU: NCCL with a group of one only"
    cg = dist.new_group(backend="gloo")  # the parity checks' host-tensor collectives
    tr = synth.CONFIGS["tiny"]
    cfg = oracle.PoolConfig(b=5, k=4, z=1 << 12)
    # "sharded-state": the sharded merge on register-sharded handles (each
    # rank stores only its shard's DRV)
    sharded_state = mode == "sharded-state"
    if sharded_state:
        mode = "sharded"
    state = None
    if mode == "p2p":  # fused merge + slide over symmetric-memory peers
        state = PeerMerge.alloc_state(make_config(32, 4, 1 << 12), dev)
    pool = VBDR(32, 4, 1 << 12, device=dev, drv_shards=world if sharded_state else 0,
                drv_shard=rank if sharded_state else 0, state=state)
    peer = PeerMerge(pool) if mode == "p2p" else None
    ref = oracle.Pool(cfg, "serial") if rank == 0 else None
    ok = True
    for t in range(7):
        pairs = synth.generate(tr, t)
        a, b = shard_range(len(pairs), rank, world)
        pool.scan_slice(torch.from_numpy(pairs[a:b].reshape(-1).view(np.int32)).to(dev))
        if peer is not None:
            peer.close_slice()
        else:
            slide_merged(pool, None, mode)
        torch.cuda.synchronize()
        regs = torch.from_numpy(pool.export_regmax())
        allregs = [torch.empty_like(regs) for _ in range(world)]
        dist.all_gather(allregs, regs, group=cg)
        if rank == 0:
            ref.slice(pairs)
            M = ref.readout()
            ok &= all(np.array_equal(r.numpy(), M) for r in allregs)
            ok &= pool.export_pool_sums() == (
                sum(int(c) << (cfg.L - v) for v, c in enumerate(np.bincount(M, minlength=cfg.L + 1))),
                int((M == 0).sum()))
            if mode == "stamps" or mode == "delta" or world == 1:  # replicas slide all BDRs
                ok &= np.array_equal(pool.export_ages(), ref.drv())
    if mode == "sparse":  # the fixed-capacity record buffers never overflowed
        ok &= pool._sparse_merge.check() <= pool._sparse_merge.cap
    hosts = tr.host_ids()
    h0, h1 = shard_range(len(hosts), rank, world)
    est = pool.estimate(torch.from_numpy(hosts[h0:h1].view(np.int32)).to(dev)).cpu()
    parts = [None] * world
    dist.all_gather_object(parts, est.numpy(), group=cg)
    if rank == 0:
        got = np.concatenate(parts)
        want = ref.estimate(ref.readout(), hosts)
        ok &= bool(np.all(np.abs(got - want) <= 1e-9 * np.maximum(np.abs(want), 1.0)))
        print(f"mode={mode}{' (sharded state)' if sharded_state else ''} world={world} "
              f"parity={'ok' if ok else 'FAILED'}", flush=True)
    dist.barrier(group=cg)
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main(sys.argv[1])
