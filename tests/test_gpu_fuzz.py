"""GPU parity fuzz: seeded random configurations through the C ABI against the
oracle, each run past k slices so expired-but-unsaturated
DRs are compared (SlideDR / IsActiveDR).

Every case draws, from its own seed: the layout (F / P), g (2..256), the pool
size z (2^6..2^16, 2 g <= z), k (1..2^zb - 2), the scan mode, a trace (hosts, pairs per slice, Zipf skew), empty
slices, and a ragged split of each slice into several scan batches (odd
lengths, so the tail pair of a batch is exercised).  At a few boundaries it
checks registers (also against a rebuild from the window's pairs) and DR state
bit for bit, pool and host sums, and the HLL estimates to 1e-9 -- through the
gather estimate and both plan kinds.  (The LogLog / PCSA estimators have their
own parity tests in test_gpu_parity.py.)
"""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1810_13132_b200 import VBDR  # noqa: E402
from test_gpu_parity import check_estimates, compare_boundary, dev_u32, est_floor  # noqa: E402

DEV = torch.device("cuda:0")


def draw(seed: int):
    rng = np.random.default_rng(1_000_003 * seed + 17)
    layout = "packed" if rng.random() < 0.5 else "fast"
    b = int(rng.integers(1, 9))           # g = 2..256
    z_log2 = int(rng.integers(max(6, b + 1), 17))
    zb = int(rng.integers(2, 7))
    k = int(rng.integers(1, (1 << zb) - 1))  # leaves room for P's extra saturation level
    scan_mode = int(rng.choice([0, 2, 5]))
    hosts = int(rng.integers(1, 400))
    pairs = int(rng.integers(0, 6000))
    return dict(layout=layout, b=b, z_log2=z_log2, k=k, scan_mode=scan_mode,
                hosts=hosts, pairs=pairs, seed=seed, rng=rng)


@pytest.mark.parametrize("seed", range(96))
def test_random_config_parity(seed):
    d = draw(seed)
    rng = d["rng"]
    g, z, k = 1 << d["b"], 1 << d["z_log2"], d["k"]
    cfg = oracle.PoolConfig(b=d["b"], k=k, z=z)
    if d["layout"] == "packed" and (1 << cfg.zb) - 2 < k:
        cfg = oracle.PoolConfig(b=d["b"], k=k, z=z, zb=cfg.zb + 1)
    ref = oracle.Pool(cfg, "serial" if d["layout"] == "fast" else "gsmall")
    pool = VBDR(g, k, z, layout=d["layout"], scan_mode=d["scan_mode"], device=DEV)
    assert pool.info()["zbits"] == cfg.zb
    tr = synth.TraceConfig(f"fuzz{seed}", hosts=d["hosts"], pairs_per_slice=max(d["pairs"], 1),
                           U0=int(rng.integers(16, 1 << 16)), seed=seed + 99)
    hosts_np = tr.host_ids()
    hosts = dev_u32(hosts_np)
    n_slices = k + int(rng.integers(2, 6))
    check_at = {n_slices - 1, int(rng.integers(0, n_slices))}
    plans = {kind: pool.plan(hosts, kind=kind) for kind in ("staged", "sorted")
             if _plan_ok(pool, hosts, kind)}
    slices = []
    for t in range(n_slices):
        pairs = synth.generate(tr, t)[: d["pairs"]] if rng.random() > 0.15 else \
            np.zeros((0, 2), np.uint32)
        slices.append(pairs)
        # a ragged split of the slice into scan batches
        cuts = np.sort(rng.integers(0, len(pairs) + 1, int(rng.integers(0, 4))))
        for part in np.split(pairs, cuts):
            if len(part):
                pool.scan_slice(dev_u32(part))
        pool.slide()
        ref.slice(pairs)
        if t in check_at:
            window = np.concatenate(slices[max(0, t - k + 1):t + 1])
            compare_boundary(pool, ref, [], hosts_np, hosts, window)
            want = pool.estimate(hosts).cpu().numpy()
            M = ref.readout()
            check_estimates(want, ref.estimate(M, hosts_np), est_floor(ref, M, hosts_np))
            for kind, plan in plans.items():
                assert np.array_equal(pool.estimate_plan(plan).cpu().numpy(), want), kind
    for plan in plans.values():
        pool.plan_check(plan)


def _plan_ok(pool, hosts, kind):
    try:
        pool.plan(hosts, kind=kind).release()
        return True
    except ValueError:
        return False
