"""GPU parity at BASELINE.json's full sizes ('10G': 100M pairs/slice, 2^26
BDRs, m=256, k=10; 'bigwin': 2^28 BDRs, 16.7M pairs/slice, m=256, k=60) in the
launch configuration bench.py times.  The oracle cannot hold these pools one DR
per uint16, so it checks:
  - every register M[j] against the rebuild from scratch (PAPER.md:42, 137-140:
    the windowed max rank) and the exact pool sums;
  - the DR ages of sampled BDRs against Alg.1's definition (the age of rank r
    is the number of slices since r was a slice's max rank at j, saturating);
  - estimates and integer host sums of sampled hosts (100k random + the 1000
    heaviest) against the oracle's estimator on the rebuilt registers.
"""
import multiprocessing as mp
from concurrent.futures import ProcessPoolExecutor

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1810_13132_b200 import VBDR  # noqa: E402
from test_gpu_parity import (check_estimates, dev_u32, oracle_pool_sums)  # noqa: E402

DEV = torch.device("cuda:0")


def _chunk(args):
    name, t, start, count = args
    return synth.generate(synth.CONFIGS[name], t, start, count)


def generate_parallel(name: str, t: int, chunk: int = 8_000_000) -> np.ndarray:
    """synth.generate (numpy twin) of one whole slice, chunked over processes."""
    n = synth.CONFIGS[name].pairs_per_slice
    jobs = [(name, t, s, min(chunk, n - s)) for s in range(0, n, chunk)]
    with ProcessPoolExecutor(max_workers=min(16, mp.cpu_count()),
                             mp_context=mp.get_context("fork")) as ex:
        parts = list(ex.map(_chunk, jobs))
    return np.concatenate(parts)


def expected_ages(per_slice_M, idx, L, zb):
    """Alg.1 ages at the last boundary for BDRs idx: rank r has age t_last - t
    for the latest slice t whose max rank at j was r, else the sentinel."""
    S = (1 << zb) - 1
    T = len(per_slice_M)
    ages = np.full((len(idx), L), S, dtype=np.uint16)
    for t, M in enumerate(per_slice_M):  # later slices overwrite
        m = M[idx].astype(np.int64)
        rows = np.flatnonzero(m > 0)
        ages[rows, m[rows] - 1] = min(T - 1 - t, S)
    return ages


def run_large(name, m, k, n_phys, n_slices, layout="fast", plan_kinds=("sorted",)):
    tr = synth.CONFIGS[name]
    b = m.bit_length() - 1
    L = 32 - b
    pool = VBDR(m, k, n_phys, layout=layout, device=DEV)
    inf = pool.info()
    rng = np.random.default_rng(11)
    sample = np.sort(rng.choice(n_phys, size=200_000, replace=False))
    hosts_all = tr.host_ids()
    hs = np.unique(np.concatenate([np.arange(1000), rng.choice(tr.hosts, 100_000, replace=False)]))
    hosts = hosts_all[hs]
    per_slice = []
    for t in range(n_slices):
        pairs = generate_parallel(name, t)
        pool.scan_slice(dev_u32(pairs))
        pool.slide()
        per_slice.append(oracle.rebuild(pairs, b, L, n_phys, 0x5EED0001, 0x5EED0002))
        del pairs
    window = per_slice[-k:]  # W(t-k+1..t): the registers rebuilt from the last k slices
    M = window[0]
    for x in window[1:]:
        M = np.maximum(M, x)
    got = pool.export_regmax()
    assert np.array_equal(got, M), "regmax != rebuild from scratch"
    assert pool.export_pool_sums() == oracle_pool_sums(M, L)
    if layout == "fast":
        ages = pool.export_ages_at(sample)
        want = expected_ages(per_slice, sample, L, inf["zbits"])
        assert np.array_equal(ages, want)
        S_ = (1 << inf["zbits"]) - 1
        if n_slices > k:  # expired but unsaturated DRs (k <= age < S) were compared
            assert ((want >= k) & (want < S_)).any()
    S, V = pool.host_sums(dev_u32(hosts))
    Z, Vo = oracle.host_sums_M(M, hosts, b, n_phys)
    assert np.array_equal(V.cpu().numpy().astype(np.uint64), Vo)
    assert np.array_equal(S.cpu().numpy().astype(np.float64) * 2.0 ** -L, Z)
    est = pool.estimate(dev_u32(hosts)).cpu().numpy()
    for kind in plan_kinds:  # every plan kind this pool takes, on the sampled hosts
        plan = pool.plan(dev_u32(hosts), kind=kind)
        assert np.array_equal(pool.estimate_plan(plan).cpu().numpy(), est), kind
        S2, V2 = pool.host_sums_plan(plan)
        assert torch.equal(S2, S) and torch.equal(V2, V), kind
        del plan
    # the bench's launch configuration: ONE plan (auto) over ALL hosts of the
    # config, bit-identical to the gather estimate of all hosts; the sampled
    # hosts are checked against the oracle below
    all_dev = dev_u32(hosts_all)
    plan = pool.plan(all_dev)
    est_all = pool.estimate_plan(plan).cpu().numpy()
    assert plan.kind == "auto"
    del plan
    assert np.array_equal(est_all, pool.estimate(all_dev).cpu().numpy())
    assert np.array_equal(est_all[hs], est)
    want = oracle.estimate_M(M, hosts, b, n_phys)
    g, z = m, n_phys
    Es = oracle.alpha(g) * g * g / Z
    lc = (Es <= 2.5 * g) & (Vo > 0)
    Es = np.where(lc, g * np.log(g / np.maximum(Vo, 1).astype(float)), Es)
    check_estimates(est, want, (z * g) / (z - g) * Es / g)
    return inf


def test_10G_full_size():
    """12 slices > k = 10: the sampled DR ages include expired, unsaturated
    values (k <= age < S = 15) of the Swar<4> instantiation."""
    inf = run_large("10G", 256, 10, 1 << 26, 12)
    assert inf["zbits"] == 4 and inf["words"] == 3


def test_bigwin_full_size_multipass_estimate():
    """2^28 BDRs: the estimate runs in 4 passes over 64 MiB register ranges."""
    inf = run_large("bigwin", 256, 60, 1 << 28, 3, plan_kinds=("sorted", "passid"))
    assert inf["zbits"] == 6 and inf["words"] == 5


def test_10G_full_size_packed():
    """Layout P (gsmall semantics) at full 10G size past k slices: registers
    against the window's rebuild, pool and host sums, every plan estimate
    bit-identical to the gather, sampled hosts against the oracle."""
    inf = run_large("10G", 256, 10, 1 << 26, 12, layout="packed")
    assert inf["zbits"] == 4


def test_10G_full_size_stamps():
    """Layout S (per-(BDR, rank) u32 stamps, 6 GiB at 10G) at full size past k
    slices: registers against the window's rebuild, sums, plan estimates."""
    run_large("10G", 256, 10, 1 << 26, 12, layout="stamps")
