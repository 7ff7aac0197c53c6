"""Pins for the estimator the paper delegates to: closed
forms, the textbook HyperLogLog special case, and statistical sanity."""
import os

import numpy as np
import pytest

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _parse_regs(spec):
    out = []
    for part in spec.split(","):
        v, n = part.split("*")
        out += [int(v)] * int(n)
    return np.array(out, dtype=np.uint8)


def test_closed_forms_from_golden():
    n_hll = n_vhll = 0
    for line in open(os.path.join(GOLD, "hll_closed_forms.txt")):
        if line.startswith("#") or not line.strip():
            continue
        f = line.split()
        if f[0].startswith("vhll"):
            z, g, Es, Et, want = int(f[1]), int(f[2]), float(f[3]), float(f[4]), float(f[5])
            assert oracle.vhll(z, g, Es, Et) == pytest.approx(want, rel=1e-14, abs=1e-12)
            n_vhll += 1
        else:
            s, regs, want = int(f[1]), _parse_regs(f[2]), float(f[3])
            assert regs.size == s
            assert oracle.hll_raw(regs) == pytest.approx(want, rel=1e-14, abs=1e-12)
            n_hll += 1
    assert n_hll == 5 and n_vhll == 4


def test_alpha_values():
    # SPEC.md:260
    assert oracle.alpha(16) == 0.673
    assert oracle.alpha(32) == 0.697
    assert oracle.alpha(64) == 0.709
    assert oracle.alpha(128) == pytest.approx(0.7213 / (1 + 1.079 / 128), rel=0)


def test_hll_monotone_in_equal_registers():
    # all-equal registers r -> strictly increasing in r
    vals = [oracle.hll_raw(np.full(64, r, np.uint8)) for r in range(0, 20)]
    assert all(b > a for a, b in zip(vals[1:], vals[2:]))


def _textbook_registers(bips, b, L, A1):
    """Plain HyperLogLog for ONE host: register vidx keeps the max rank.  The
    rank uses int.bit_length, independent of the oracle's LBP1 loop."""
    reg = np.zeros(1 << b, dtype=np.uint8)
    for bip in bips:
        h = oracle.H(int(bip), 1 << 32, A1)
        vidx = h >> (32 - b)
        w = (h << b) & 0xFFFFFFFF
        r = min(33 - w.bit_length() if w else 33, L)
        reg[vidx] = max(reg[vidx], r)
    return reg


def test_no_sharing_special_case_is_textbook_hll():
    """One host alone in a large pool whose g physical indices are distinct:
    the gathered virtual vector equals a textbook HLL register vector, and its
    raw estimate has RMS error ~1.04/sqrt(g) (c.4/c.5 pin)."""
    b, g = 5, 32
    cfg = oracle.PoolConfig(b=b, k=4, z=1 << 15)
    rng = np.random.default_rng(12)
    errs, errs_v = [], []
    n = 3000
    seeds = 48
    for s in range(seeds):
        aip = int(rng.integers(0, 1 << 32))
        idx = {oracle.getPhyIdx(aip, i, cfg.A0, cfg.z) for i in range(g)}
        if len(idx) < g:
            continue
        bips = rng.choice(1 << 32, size=n, replace=False).astype(np.uint32)
        pairs = np.stack([np.full(n, aip, np.uint32), bips], axis=1)
        p = oracle.Pool(cfg, "serial")
        p.slice(pairs)
        M = p.readout()
        regs = p.gather(M, aip)
        if s < 8:
            assert np.array_equal(regs, _textbook_registers(bips, b, cfg.L, cfg.A1))
        errs.append(oracle.hll_raw(regs) / n - 1)
        errs_v.append(p.estimate(M, np.array([aip], np.uint32))[0] / n - 1)
    rms = float(np.sqrt(np.mean(np.square(errs))))
    se = 1.04 / np.sqrt(g)
    assert 0.7 * se <= rms <= 1.3 * se, rms
    assert abs(np.mean(errs)) < 0.1
    # the vHLL noise term is ~0 here (no other host): same accuracy class
    assert float(np.sqrt(np.mean(np.square(errs_v)))) <= 1.3 * se


def test_spec_acceptance5_single_host():
    """SPEC.md:521 (scaled to 30 trials): n = 50,000, g = 512, m = 2^16, k = 8:
    |estimate - n|/n <= 14% (3 standard errors) in >= 95% of trials."""
    cfg = oracle.PoolConfig(b=9, k=8, z=1 << 16)
    rng = np.random.default_rng(21)
    ok = 0
    trials = 30
    for _ in range(trials):
        aip = int(rng.integers(0, 1 << 32))
        bips = rng.choice(1 << 32, size=50_000, replace=False).astype(np.uint32)
        p = oracle.Pool(cfg, "gsmall")
        p.slice(np.stack([np.full(bips.size, aip, np.uint32), bips], axis=1))
        est = p.estimate(p.readout(), np.array([aip], np.uint32))[0]
        ok += abs(est / 50_000 - 1) <= 0.14
    assert ok >= 0.95 * trials


def test_tiny_shared_pool_statistics():
    """c.5 (2): on the tiny workload (shared, skewed pool) report bias/RMS
    against Definition 1 counts; assert only loose sanity for hosts with
    n >= 300.  (Accuracy on shared pools is parity-unpinned vs the paper.)"""
    cfg = oracle.PoolConfig(b=5, k=4, z=1 << 12)
    se = 1.04 / np.sqrt(cfg.g)
    rel = []
    for seed in range(1, 13):
        tr = synth.TraceConfig("tiny", hosts=64, pairs_per_slice=10_000, U0=4000, seed=seed)
        slices = [synth.generate(tr, t) for t in range(8)]
        p = oracle.Pool(cfg, "serial")
        for sl in slices:
            p.slice(sl)
        exact = oracle.exact_cardinalities(slices[-cfg.k:])
        hosts = tr.host_ids()
        est = p.estimate(p.readout(), hosts)
        for a, e in zip(hosts.tolist(), est.tolist()):
            n = exact.get(a, 0)
            if n >= 300:
                rel.append(e / n - 1)
    rel = np.array(rel)
    assert rel.size > 50
    assert abs(rel.mean()) <= 0.3
    assert np.sqrt(np.mean(rel ** 2)) <= 2.5 * se


def test_fresh_pool_estimates_zero():
    # fresh pool, any aip -> 0
    cfg = oracle.PoolConfig(b=5, k=4, z=1 << 12)
    p = oracle.Pool(cfg, "serial")
    est = p.estimate(p.readout(), np.arange(100, dtype=np.uint32))
    assert (est == 0).all()


# ---------------------------------------------------------------- N4 variants
def test_loglog_alpha_limit_and_monotone():
    """Durand-Flajolet alpha_m -> e^-gamma / sqrt(2) = 0.39701... (closed form),
    from below, with a 1/m approach."""
    import math
    a_inf = math.exp(-0.5772156649015329) / math.sqrt(2)
    prev = 0.0
    for e in range(4, 23):
        m = 1 << e
        a = oracle.loglog_alpha(m)
        assert prev < a < a_inf
        assert abs(a / a_inf - 1) < 2.0 / m
        prev = a


def test_loglog_pcsa_closed_forms():
    # all registers equal to r: LogLog = alpha_s s 2^r; PCSA = (s / 0.77351) 2^r
    for s, r in ((32, 0), (32, 3), (128, 5)):
        regs = np.full(s, r, np.uint8)
        assert oracle.loglog_raw(regs) == pytest.approx(oracle.loglog_alpha(s) * s * 2.0 ** r,
                                                        rel=1e-15)
        assert oracle.pcsa_raw(regs) == pytest.approx(s / 0.77351 * 2.0 ** r, rel=1e-15)
    # mixed: geometric mean of 2^M over the registers
    regs = np.array([0, 2] * 16, np.uint8)
    assert oracle.loglog_raw(regs) == pytest.approx(oracle.loglog_alpha(32) * 32 * 2.0, rel=1e-15)


def test_pcsa_readout_traces():
    k, zb, L = 4, 3, 10
    S = (1 << zb) - 1
    d = np.full(L, S)
    assert oracle.bdr_pcsa_R(d, k) == 0            # nothing active
    d[0] = d[1] = 0
    d[3] = 1                                       # ranks 1, 2, 4 active; 3 not
    assert oracle.bdr_pcsa_R(d, k) == 2
    d[2] = k                                       # rank 3 expired: still 2
    assert oracle.bdr_pcsa_R(d, k) == 2
    d[2] = k - 1
    assert oracle.bdr_pcsa_R(d, k) == 4            # 1..4 active, 5 not
    assert oracle.bdr_pcsa_R(np.zeros(L), k) == L  # all active


def _textbook_bitmaps(bips, b, L, A1):
    """Flajolet-Martin PCSA for ONE host: register vidx collects the set of
    ranks seen; R = lowest missing rank - 1 (int.bit_length for the rank)."""
    seen = [set() for _ in range(1 << b)]
    for bip in bips:
        h = oracle.H(int(bip), 1 << 32, A1)
        w = (h << b) & 0xFFFFFFFF
        seen[h >> (32 - b)].add(min(33 - w.bit_length() if w else 33, L))
    R = []
    for st in seen:
        r = 1
        while r in st and r <= L:
            r += 1
        R.append(r - 1)
    return np.array(R, np.uint8)


def test_pcsa_gsmall_pool_is_textbook_pcsa_and_sliding():
    """One host alone in a gsmall pool: the gathered PCSA registers equal a
    textbook FM bitmap readout; the RMS error of the PCSA raw estimate is
    ~0.78/sqrt(g); after slides the registers equal the bitmaps of the window's
    pairs only (sliding correctness of the PCSA readout)."""
    b, g = 5, 32
    cfg = oracle.PoolConfig(b=b, k=3, z=1 << 15)
    rng = np.random.default_rng(31)
    errs = []
    for s in range(40):
        aip = int(rng.integers(0, 1 << 32))
        if len({oracle.getPhyIdx(aip, i, cfg.A0, cfg.z) for i in range(g)}) < g:
            continue
        n = 4000
        bips = rng.choice(1 << 32, size=n, replace=False).astype(np.uint32)
        p = oracle.Pool(cfg, "gsmall")
        p.slice(np.stack([np.full(n, aip, np.uint32), bips], axis=1))
        regs = p.gather(p.readout_pcsa(), aip)
        if s < 6:
            assert np.array_equal(regs, _textbook_bitmaps(bips, b, cfg.L, cfg.A1))
        errs.append(oracle.pcsa_raw(regs) / n - 1)
        if s < 3:  # slide k more slices with other peers: only the window counts
            later = []
            for t in range(cfg.k):
                nb = rng.choice(1 << 32, size=500, replace=False).astype(np.uint32)
                later.append(nb)
                p.slice(np.stack([np.full(nb.size, aip, np.uint32), nb], axis=1))
            regs = p.gather(p.readout_pcsa(), aip)
            assert np.array_equal(regs, _textbook_bitmaps(np.concatenate(later), b, cfg.L,
                                                          cfg.A1))
    rms = float(np.sqrt(np.mean(np.square(errs))))
    assert 0.6 * 0.78 / np.sqrt(g) <= rms <= 1.5 * 0.78 / np.sqrt(g), rms


def test_loglog_textbook_special_case():
    """One host alone: LogLog on the gathered registers has RMS ~1.30/sqrt(g)."""
    b, g = 6, 64
    cfg = oracle.PoolConfig(b=b, k=3, z=1 << 16)
    rng = np.random.default_rng(17)
    errs = []
    for _ in range(40):
        aip = int(rng.integers(0, 1 << 32))
        n = 20000
        bips = rng.choice(1 << 32, size=n, replace=False).astype(np.uint32)
        p = oracle.Pool(cfg, "serial")
        p.slice(np.stack([np.full(n, aip, np.uint32), bips], axis=1))
        errs.append(oracle.loglog_raw(p.gather(p.readout(), aip)) / n - 1)
    rms = float(np.sqrt(np.mean(np.square(errs))))
    assert 0.6 * 1.30 / np.sqrt(g) <= rms <= 1.5 * 1.30 / np.sqrt(g), rms


def test_estimate_variant_hll_matches_pool_estimate():
    cfg = oracle.PoolConfig(b=5, k=4, z=1 << 12)
    tr = synth.CONFIGS["tiny"]
    p = oracle.Pool(cfg, "gsmall")
    for t in range(5):
        p.slice(synth.generate(tr, t))
    M = p.readout()
    hosts = tr.host_ids()
    assert np.array_equal(oracle.estimate_variant(M, hosts, cfg.b, cfg.z, "hll"),
                          p.estimate(M, hosts))
    est = oracle.estimate_variant(p.readout_pcsa(), hosts, cfg.b, cfg.z, "pcsa")
    assert (est >= 0).all() and est.max() > 100
