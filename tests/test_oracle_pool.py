"""Pool-level pins for the oracle: sliding correctness
against a rebuild from scratch, variant equivalence, order and partition
independence, window locality."""
import numpy as np
import pytest

import oracle
import synth

VARIANTS = ("serial", "gfast", "gsmall")


def _random_slices(rng, n_slices, n_pairs, n_hosts=40, n_peers=3000):
    hosts = rng.integers(0, 1 << 32, size=n_hosts, dtype=np.uint64)
    peers = rng.integers(0, 1 << 32, size=n_peers, dtype=np.uint64)
    out = []
    for _ in range(n_slices):
        cnt = int(rng.integers(0, n_pairs + 1))
        p = np.empty((cnt, 2), dtype=np.uint32)
        p[:, 0] = hosts[rng.integers(0, n_hosts, size=cnt)]
        p[:, 1] = peers[rng.integers(0, n_peers, size=cnt)]
        out.append(p)
    return out


def _rebuild_python(window, cfg):
    """M*[j] = max rank over the window's pairs mapping to j, per pair through
    the oracle's pinned front end, accumulated here in Python."""
    M = np.zeros(cfg.z, dtype=np.uint8)
    for sl in window:
        for a, b in sl:
            j, r = oracle.pair_index(int(a), int(b), cfg.b, cfg.L, cfg.A0, cfg.A1, cfg.z)
            M[j] = max(M[j], r)
    return M


@pytest.mark.parametrize("b,k,z", [(2, 1, 64), (3, 4, 128), (5, 4, 1 << 10), (4, 7, 256),
                                   (6, 10, 1 << 9)])
def test_pool_sliding_correctness_and_variant_equivalence(b, k, z):
    rng = np.random.default_rng(b * 100 + k)
    cfg = oracle.PoolConfig(b=b, k=k, z=z)
    pools = {v: oracle.Pool(cfg, v) for v in VARIANTS}
    slices = _random_slices(rng, 3 * k + 6, 300)
    for t, sl in enumerate(slices):
        for p in pools.values():
            p.slice(sl)
        window = slices[max(0, t - k + 1):t + 1]
        want = _rebuild_python(window, cfg)
        for v, p in pools.items():
            assert np.array_equal(p.readout(), want), (v, t)
        # serial == gfast on the raw DR state (F3: both record one rank per slice)
        assert np.array_equal(pools["serial"].drv(), pools["gfast"].drv())
        # the C rebuild agrees with the Python one
        cat = np.concatenate(window) if window else np.zeros((0, 2), np.uint32)
        assert np.array_equal(oracle.rebuild(cat, cfg.b, cfg.L, cfg.z, cfg.A0, cfg.A1), want)


def test_tiny_trace_all_boundaries():
    cfg = oracle.PoolConfig(b=5, k=4, z=1 << 12)
    tr = synth.CONFIGS["tiny"]
    slices = [synth.generate(tr, t) for t in range(8)]
    pools = {v: oracle.Pool(cfg, v) for v in VARIANTS}
    for t in range(8):
        for p in pools.values():
            p.slice(slices[t])
        cat = np.concatenate(slices[max(0, t - 3):t + 1])
        want = oracle.rebuild(cat, cfg.b, cfg.L, cfg.z, cfg.A0, cfg.A1)
        for p in pools.values():
            assert np.array_equal(p.readout(), want)


def test_order_and_duplication_invariance():
    """Permuting and duplicating pairs within a slice gives a bit-identical
    pool."""
    rng = np.random.default_rng(1)
    cfg = oracle.PoolConfig(b=4, k=3, z=256)
    slices = _random_slices(rng, 7, 400)
    for v in VARIANTS:
        a, b = oracle.Pool(cfg, v), oracle.Pool(cfg, v)
        for sl in slices:
            a.slice(sl)
            dup = np.concatenate([sl, sl[: len(sl) // 2]])
            b.slice(dup[rng.permutation(len(dup))])
            assert np.array_equal(a.drv(), b.drv()), v


def test_partition_merge_by_max():
    """Scanning a slice in N shards and merging nowLBP1 by elementwise max
    equals scanning it whole (the basis of the multi-GPU merge)."""
    rng = np.random.default_rng(2)
    cfg = oracle.PoolConfig(b=5, k=4, z=1 << 10)
    sl = _random_slices(rng, 1, 5000)[0]
    whole = oracle.Pool(cfg, "serial")
    whole.begin_slice()
    whole.scan(sl)
    for N in (2, 4, 8):
        merged = np.zeros(cfg.z, dtype=np.uint8)
        for r in range(N):
            p = oracle.Pool(cfg, "serial")
            p.begin_slice()
            p.scan(sl[r::N])
            merged = np.maximum(merged, p.now())
        assert np.array_equal(merged, whole.now())


def test_window_locality():
    """Replaying only the last k slices into a fresh pool gives the same C_k and
    M -- but not necessarily the same raw DR ages."""
    rng = np.random.default_rng(4)
    cfg = oracle.PoolConfig(b=4, k=3, z=512)
    slices = _random_slices(rng, 10, 500)
    for v in VARIANTS:
        full = oracle.Pool(cfg, v)
        for sl in slices:
            full.slice(sl)
        fresh = oracle.Pool(cfg, v)
        for sl in slices[-cfg.k:]:
            fresh.slice(sl)
        assert np.array_equal(full.ck(), fresh.ck()), v
        assert np.array_equal(full.readout(), fresh.readout()), v


def test_silent_host_registers_come_from_others_only():
    """Register-level replacement for SPEC acceptance 7: after a
    host is silent for k slices, its virtual registers equal those rebuilt from
    the other hosts' pairs of the window alone."""
    rng = np.random.default_rng(6)
    cfg = oracle.PoolConfig(b=4, k=3, z=256)
    slices = _random_slices(rng, 9, 400, n_hosts=10)
    victim = int(slices[0][0, 0])
    for t in range(3, 9):
        slices[t] = slices[t][slices[t][:, 0] != victim]
    p = oracle.Pool(cfg, "serial")
    for sl in slices:
        p.slice(sl)
    others = np.concatenate(slices[-cfg.k:])
    rebuilt = oracle.rebuild(others, cfg.b, cfg.L, cfg.z, cfg.A0, cfg.A1)
    assert np.array_equal(p.gather(p.readout(), victim), p.gather(rebuilt, victim))


def test_alg5_sum_equals_gather_sum():
    cfg = oracle.PoolConfig(b=5, k=4, z=1 << 12)
    tr = synth.CONFIGS["tiny"]
    p = oracle.Pool(cfg, "serial")
    for t in range(4):
        p.slice(synth.generate(tr, t))
    M = p.readout()
    for aip in tr.host_ids()[:10]:
        assert p.sum_lbp1(M, int(aip)) == int(p.gather(M, int(aip)).sum())
    # fresh pool -> 0
    q = oracle.Pool(cfg, "serial")
    assert q.sum_lbp1(q.readout(), 12345) == 0


def test_exact_cardinality_definition():
    # SPEC.md:385-386
    s0 = np.array([[1, 9]] * 5, dtype=np.uint32)
    assert oracle.exact_cardinality([s0], 1) == 1
    s1 = np.array([[1, 9], [1, 10], [2, 9]], dtype=np.uint32)
    assert oracle.exact_cardinality([s1], 1) == 2
    assert oracle.exact_cardinalities([s0, s1]) == {1: 2, 2: 1}


def test_estimate_from_register_array_matches_pool():
    cfg = oracle.PoolConfig(b=5, k=4, z=1 << 12)
    tr = synth.CONFIGS["tiny"]
    p = oracle.Pool(cfg, "serial")
    for t in range(5):
        p.slice(synth.generate(tr, t))
    M = p.readout()
    hosts = tr.host_ids()
    assert np.array_equal(oracle.estimate_M(M, hosts, cfg.b, cfg.z), p.estimate(M, hosts))
    Z, V = oracle.host_sums_M(M, hosts, cfg.b, cfg.z)
    Z2, V2 = p.host_sums(M, hosts)
    assert np.array_equal(Z, Z2) and np.array_equal(V, V2)
