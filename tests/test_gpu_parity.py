"""GPU parity: the CUDA path through the C ABI against the oracle, element by
element, on the same seeded synthetic inputs.

Bit-exact: registers M, DR state (layout fast: raw ages vs the serial oracle;
layout packed: canonical C_k vs the gsmall oracle), pool sums, per-host (S, V).
fp64 estimates: |gpu - oracle| <= 1e-9 * max(|oracle|, C * E_s / g).
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

DEV = torch.device("cuda:0")
TOL = 1e-9


def dev_u32(a: np.ndarray):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint32).reshape(-1).view(np.int32)).to(DEV)


def oracle_pool_sums(M: np.ndarray, L: int):
    """S_tot = sum_j 2^(L - M_j) and V_tot = #{M_j = 0}, exact integers."""
    counts = np.bincount(M, minlength=L + 1).astype(object)
    S = sum(int(counts[r]) << (L - r) for r in range(L + 1))
    return S, int(counts[0])


def check_estimates(gpu, want, Es_over_g_C):
    floor = np.maximum(np.abs(want), Es_over_g_C)
    bad = np.abs(gpu - want) > TOL * np.maximum(floor, 1e-300)
    assert not bad.any(), (np.flatnonzero(bad)[:5], gpu[bad][:5], want[bad][:5])


def est_floor(ref: oracle.Pool, M, hosts):
    """C * E_s / g per host (the scale of the cancelling vHLL terms)."""
    cfg = ref.cfg
    Z, V = ref.host_sums(M, hosts)
    g, z = cfg.g, cfg.z
    C = (z * g) / (z - g)
    Es = oracle.alpha(g) * g * g / Z
    lc = (Es <= 2.5 * g) & (V > 0)
    Es = np.where(lc, g * np.log(g / np.maximum(V, 1).astype(float)), Es)
    return C * Es / g


def compare_boundary(pool, ref: oracle.Pool, refs_other, hosts_np, hosts_dev, window_pairs,
                     check_ages=True, check_est=True):
    cfg = ref.cfg
    M = ref.readout()
    got = pool.export_regmax()
    assert np.array_equal(got, M), "regmax != oracle Alg.2 readout"
    for o in refs_other:
        assert np.array_equal(o.readout(), M)
    if window_pairs is not None:
        Mstar = oracle.rebuild(window_pairs, cfg.b, cfg.L, cfg.z, cfg.A0, cfg.A1)
        assert np.array_equal(got, Mstar), "regmax != rebuild from scratch"
    if check_ages:
        if pool.layout == "fast":
            assert np.array_equal(pool.export_ages(), ref.drv()), "DR ages"
        else:
            assert np.array_equal(pool.export_ages(canonical=True), ref.ck()), "C_k"
            # raw stored values: Alg.8's SlideDR of the next slice already applied
            # (saturating at S), so ages in [k, S) are checked too, not only C_k
            S_ = (1 << cfg.zb) - 1
            assert np.array_equal(pool.export_ages().astype(np.int64),
                                  np.minimum(ref.drv().astype(np.int64) + 1, S_)), "raw DR ages"
    assert pool.export_pool_sums() == oracle_pool_sums(M, cfg.L)
    if hosts_np is not None:
        S, V = pool.host_sums(hosts_dev)
        Z, Vo = ref.host_sums(M, hosts_np)
        assert np.array_equal(V.cpu().numpy().astype(np.uint64), Vo)
        assert np.array_equal(S.cpu().numpy().astype(np.float64) * 2.0 ** -cfg.L, Z)
        if check_est:
            est = pool.estimate(hosts_dev).cpu().numpy()
            want = ref.estimate(M, hosts_np)
            check_estimates(est, want, est_floor(ref, M, hosts_np))


@pytest.mark.parametrize("layout", ["fast", "packed"])
@pytest.mark.parametrize("scan_mode,est_lanes,passes", [(2, 0, 0), (2, 1, 0), (5, 8, 10), (2, 32, 0),
                                                       (5, 2, 7), (0, 0, 11), (5, 4, 0),
                                                       (0, 16, 0)])
def test_tiny_every_boundary(layout, scan_mode, est_lanes, passes):
    """configs[0] 'tiny': 10k pairs/slice, 64 hosts, m=32, 2^12 BDRs, k=4."""
    tr = synth.CONFIGS["tiny"]
    cfg = oracle.PoolConfig(b=5, k=4, z=1 << 12)
    variant = "serial" if layout == "fast" else "gsmall"
    ref = oracle.Pool(cfg, variant)
    others = [oracle.Pool(cfg, v) for v in ("gfast", "gsmall" if layout == "fast" else "serial")]
    pool = VBDR(32, 4, 1 << 12, layout=layout, scan_mode=scan_mode, est_lanes=est_lanes,
                est_pass_log2=passes, device=DEV)
    hosts_np = tr.host_ids()
    hosts = dev_u32(hosts_np)
    slices = []
    # before the first slide everything estimates 0 (empty window)
    assert (pool.estimate(hosts).cpu().numpy() == 0).all()
    for t in range(12):
        pairs = synth.generate(tr, t)
        slices.append(pairs)
        # several batches per slice, odd sizes (ragged tails)
        for a, b in ((0, 3), (3, 4001), (4001, 10_000)):
            pool.scan_slice(dev_u32(pairs[a:b]))
        pool.slide()
        for p in [ref] + others:
            p.slice(pairs)
        compare_boundary(pool, ref, others, hosts_np, hosts,
                         np.concatenate(slices[max(0, t - 3):t + 1]))


@pytest.mark.parametrize("scan_mode", [0, 2])
@pytest.mark.parametrize("layout", ["fast", "packed"])
@pytest.mark.parametrize("k,m,n_phys", [(1, 2, 64), (3, 16, 1 << 10), (7, 64, 1 << 14),
                                        (15, 8, 1 << 8), (10, 256, 1 << 16), (60, 256, 1 << 16),
                                        (300, 4, 1 << 9)])
def test_configs_sweep_with_empty_slices(layout, k, m, n_phys, scan_mode):
    """Edge cases: k = 1 (discrete window), k = 2^zb - 1, big k (zb up to 9),
    g < 32 (several hosts per warp), empty slices, tiny pools.  Every config
    runs past k + 5 slices, so DRs sit expired but unsaturated (k <= age < S)
    -- in particular the 10G (zb = 4, k = 10) and bigwin (zb = 6, k = 60)
    field widths of the Swar<4> / Swar<6> IsActiveDR instantiations
    (SlideDR / IsActiveDR; SPEC.md:128 expiry)."""
    b = m.bit_length() - 1
    tr = synth.TraceConfig("sweep", hosts=200, pairs_per_slice=3001, U0=3000, seed=k * 7 + m)
    cfg = oracle.PoolConfig(b=b, k=k, z=n_phys)
    if layout == "packed" and (1 << cfg.zb) - 2 < k:
        cfg = oracle.PoolConfig(b=b, k=k, z=n_phys, zb=cfg.zb + 1)
    ref = oracle.Pool(cfg, "serial" if layout == "fast" else "gsmall")
    pool = VBDR(m, k, n_phys, layout=layout, scan_mode=scan_mode, device=DEV)
    assert pool.info()["zbits"] == cfg.zb
    hosts_np = tr.host_ids()
    hosts = dev_u32(hosts_np)
    n_slices = max(min(2 * k + 5, 40), k + 6)
    ages_seen = set()
    slices = []
    for t in range(n_slices):
        pairs = synth.generate(tr, t) if t % 4 != 2 else np.zeros((0, 2), np.uint32)
        slices.append(pairs)
        if len(pairs):
            pool.scan_slice(dev_u32(pairs))
        pool.slide()
        ref.slice(pairs)
        if t % 3 == 0 or t == n_slices - 1:
            compare_boundary(pool, ref, [], hosts_np, hosts,
                             np.concatenate(slices[max(0, t - k + 1):t + 1]))
            ages_seen |= set(np.unique(ref.drv()).tolist())
    S = (1 << cfg.zb) - 1
    if S - 1 >= k:  # the expired-but-unsaturated ages were really exercised
        assert any(k <= a < S for a in ages_seen), (k, S, sorted(ages_seen))


@pytest.mark.parametrize("layout", ["fast", "packed"])
def test_long_run_saturation(layout):
    """>= 1000 slices of 'tiny' shape: long-run ageing and DR saturation."""
    cfg = oracle.PoolConfig(b=5, k=4, z=1 << 12)
    ref = oracle.Pool(cfg, "serial" if layout == "fast" else "gsmall")
    pool = VBDR(32, 4, 1 << 12, layout=layout, device=DEV)
    tr = synth.TraceConfig("long", hosts=64, pairs_per_slice=600, U0=4000, seed=99)
    for t in range(1030):
        pairs = synth.generate(tr, t) if t % 50 < 45 else np.zeros((0, 2), np.uint32)
        if len(pairs):
            pool.scan_slice(dev_u32(pairs))
        pool.slide()
        ref.slice(pairs)
        if t % 257 == 0 or t >= 1025:
            compare_boundary(pool, ref, [], None, None, None)
    assert pool.info()["slices_closed"] == 1030


def test_negative_control_skipped_slide_breaks_parity():
    """a pipeline that skips one slide must fail the comparison."""
    tr = synth.CONFIGS["tiny"]
    cfg = oracle.PoolConfig(b=5, k=4, z=1 << 12)
    ref = oracle.Pool(cfg, "serial")
    pool = VBDR(32, 4, 1 << 12, device=DEV)
    for t in range(6):
        pairs = synth.generate(tr, t)
        pool.scan_slice(dev_u32(pairs))
        if t != 3:
            pool.slide()
        ref.slice(pairs)
    assert not np.array_equal(pool.export_ages(), ref.drv())


def test_order_split_and_duplicates_give_identical_state():
    tr = synth.CONFIGS["tiny"]
    a = VBDR(32, 4, 1 << 12, device=DEV)
    b = VBDR(32, 4, 1 << 12, device=DEV, scan_mode=5)
    rng = np.random.default_rng(0)
    for t in range(5):
        pairs = synth.generate(tr, t)
        a.scan_slice(dev_u32(pairs))
        shuffled = np.concatenate([pairs, pairs[:999]])[rng.permutation(len(pairs) + 999)]
        for part in np.array_split(shuffled, 7):
            b.scan_slice(dev_u32(part))
        a.slide()
        b.slide()
        assert np.array_equal(a.export_ages(), b.export_ages())
        assert np.array_equal(a.export_regmax(), b.export_regmax())


@pytest.mark.parametrize("layout", ["fast", "packed"])
@pytest.mark.parametrize("scan_mode", [2, 5])
def test_bursty_trains_every_scan_mode(layout, scan_mode):
    """Packet trains (consecutive duplicate pairs: whole warps hitting the
    same BDR, the case warp aggregation and the block cache target): state
    and estimates equal the oracle's in every scan mode."""
    tr = synth.TraceConfig("tiny_bursty", hosts=64, pairs_per_slice=10_000, U0=4000, burst=8)
    cfg = oracle.PoolConfig(b=5, k=4, z=1 << 12)
    ref = oracle.Pool(cfg, "serial" if layout == "fast" else "gsmall")
    pool = VBDR(32, 4, 1 << 12, layout=layout, scan_mode=scan_mode, device=DEV)
    hosts_np = tr.host_ids()
    hosts = dev_u32(hosts_np)
    slices = []
    for t in range(7):
        pairs = synth.generate(tr, t)
        slices.append(pairs)
        pool.scan_slice(dev_u32(pairs))
        pool.slide()
        ref.slice(pairs)
    compare_boundary(pool, ref, [], hosts_np, hosts, np.concatenate(slices[-4:]))


def test_sparse_extract_counts_and_cap():
    """vbdr_sparse_extract: exact per-owner counts even when the cap is too
    small (the binding then raises), and no records at all for an empty slice."""
    pool = VBDR(32, 4, 1 << 12, device=DEV)
    rec, cnt = pool.sparse_extract(4)
    assert int(cnt.sum()) == 0
    pairs = synth.generate(synth.CONFIGS["tiny"], 0)
    pool.scan_slice(dev_u32(pairs))
    rec, cnt = pool.sparse_extract(4)
    assert int(cnt.sum()) == int((pool.stamp_delta() > 0).sum())
    with pytest.raises(RuntimeError, match="cap"):
        pool.sparse_extract(4, cap=int(cnt.max()) - 1)
    with pytest.raises(RuntimeError, match="EINVAL"):
        pool.sparse_extract(3)  # 4096 BDRs do not split in 3


@pytest.mark.parametrize("layout", ["fast", "packed"])
def test_estimate_overlapping_next_slide(layout):
    """Two register buffers and four pool-sum slots: the estimate of slice t
    (second stream) may run while slice t+1 is scanned and slid; every
    slice's estimates still equal the oracle's at that boundary."""
    tr = synth.CONFIGS["tiny"]
    cfg = oracle.PoolConfig(b=5, k=4, z=1 << 12)
    ref = oracle.Pool(cfg, "serial" if layout == "fast" else "gsmall")
    pool = VBDR(32, 4, 1 << 12, layout=layout, device=DEV)
    hosts_np = tr.host_ids()
    hosts = dev_u32(hosts_np)
    plan = pool.plan(hosts)
    main, side = torch.cuda.current_stream(DEV), torch.cuda.Stream(DEV)
    ev_closed, ev_est = torch.cuda.Event(), [torch.cuda.Event(), torch.cuda.Event()]
    slices = [synth.generate(tr, t) for t in range(9)]
    dev_slices = [dev_u32(p) for p in slices]
    outs = [torch.empty(len(hosts_np), dtype=torch.float64, device=DEV) for _ in slices]
    pool.scan_slice(dev_slices[0])
    pool.slide()
    for t in range(len(slices)):
        ev_closed.record(main)
        side.wait_event(ev_closed)
        pool.estimate_plan(plan, out=outs[t], stream=side)  # slice t
        ev_est[t & 1].record(side)
        if t + 1 < len(slices):
            pool.scan_slice(dev_slices[t + 1])
            main.wait_event(ev_est[(t - 1) & 1])
            pool.slide()  # slice t+1, concurrent with the estimate of slice t
    torch.cuda.synchronize()
    for t, pairs in enumerate(slices):
        ref.slice(pairs)
        M = ref.readout()
        check_estimates(outs[t].cpu().numpy(), ref.estimate(M, hosts_np), est_floor(ref, M, hosts_np))


def test_register_sharded_state_rules():
    """drv_shards: the DRV of one shard only; closing or exporting the whole
    pool is refused, slide_delta outside the shard is refused."""
    with pytest.raises(ValueError):
        VBDR(32, 4, 1 << 12, device=DEV, layout="packed", drv_shards=2)
    with pytest.raises(ValueError):
        VBDR(32, 4, 1 << 12, device=DEV, drv_shards=2, drv_shard=2)
    pool = VBDR(32, 4, 1 << 12, device=DEV, drv_shards=4, drv_shard=1)
    pool.scan_slice(dev_u32(synth.generate(synth.CONFIGS["tiny"], 0)))
    with pytest.raises(RuntimeError, match="ESTATE"):
        pool.slide()
    with pytest.raises(RuntimeError, match="ESTATE"):
        pool.export_ages()
    delta = pool.stamp_delta()
    with pytest.raises(RuntimeError, match="EINVAL"):
        pool.slide_delta(delta[:1024].clone(), 0, 1024)
    pool.slide_delta(delta[1024:2048].clone(), 1024, 2048)
    ages = pool.export_ages_at(np.array([0, 1024, 2047, 2048], dtype=np.uint64))
    assert (ages[0] == 0).all() and (ages[3] == 0).all()  # outside the shard


def test_host_buffer_path_matches_device_path():
    """vbdr_scan_slice_host / vbdr_estimate_host (the end-to-end entry points)."""
    tr = synth.CONFIGS["tiny"]
    a = VBDR(32, 4, 1 << 12, device=DEV)
    b = VBDR(32, 4, 1 << 12, device=DEV)
    hosts_np = tr.host_ids()
    stage = torch.empty(2 * 1000, dtype=torch.int32, device=DEV)  # forces 10+ chunks
    hstage = torch.empty(len(hosts_np), dtype=torch.int32, device=DEV)
    ostage = torch.empty(len(hosts_np), dtype=torch.float64, device=DEV)
    h_hosts = torch.from_numpy(hosts_np.view(np.int32)).pin_memory()
    h_out = torch.empty(len(hosts_np), dtype=torch.float64).pin_memory()
    for t in range(6):
        pairs = synth.generate(tr, t)
        a.scan_slice(dev_u32(pairs))
        b.scan_slice_host(torch.from_numpy(pairs.reshape(-1).view(np.int32)).pin_memory(), stage)
        a.slide()
        b.slide()
        b.estimate_host(h_hosts, hstage, ostage, h_out)
        torch.cuda.synchronize()
        want = a.estimate(dev_u32(hosts_np)).cpu().numpy()
        assert np.array_equal(h_out.numpy(), want)
        assert np.array_equal(a.export_ages(), b.export_ages())


@pytest.mark.parametrize("name,layout,use_plan", [("caida", "fast", True), ("caida", "packed", True),
                                                   ("tiny", "fast", False)])
def test_e2e_pipelined_loop_matches_oracle(name, layout, use_plan):
    """bench.py's end-to-end loop exactly: vbdr_scan_slice_host through a
    one-slice staging buffer split in halves (each half's copy overlaps the
    other half's scan and, across calls, the previous slice's slide and
    estimate), vbdr_slide, vbdr_estimate_plan_host (or vbdr_estimate_host),
    and NO synchronisation between steps.  Every slice's host-side estimates,
    read after one final sync, equal the oracle's at that boundary (PAPER.md:217:
    only IP pairs are transmitted to the GPU)."""
    tr = synth.CONFIGS[name]
    wl = {"tiny": (32, 4, 1 << 12, 5), "caida": (128, 5, 1 << 22, 7)}[name]
    m, k, z, b = wl
    cfg = oracle.PoolConfig(b=b, k=k, z=z)
    ref = oracle.Pool(cfg, "serial" if layout == "fast" else "gsmall")
    pool = VBDR(m, k, z, layout=layout, device=DEV)
    hosts_np = tr.host_ids()
    n_steps = 7
    slices = [synth.generate(tr, t) for t in range(n_steps)]
    h_inputs = [torch.from_numpy(p.reshape(-1).view(np.int32)).pin_memory() for p in slices]
    stage = torch.empty(2 * len(slices[0]), dtype=torch.int32, device=DEV)  # bench: one slice
    ostage = torch.empty(len(hosts_np), dtype=torch.float64, device=DEV)
    h_outs = [torch.full((len(hosts_np),), -1.0, dtype=torch.float64).pin_memory()
              for _ in range(n_steps)]
    if use_plan:
        plan = pool.plan(dev_u32(hosts_np))
    else:
        h_hosts = torch.from_numpy(hosts_np.view(np.int32)).pin_memory()
        hstage = torch.empty(len(hosts_np), dtype=torch.int32, device=DEV)
    torch.cuda.synchronize()
    for t in range(n_steps):  # no sync inside the loop
        pool.scan_slice_host(h_inputs[t], stage)
        pool.slide()
        if use_plan:
            pool.estimate_plan_host(plan, ostage, h_outs[t])
        else:
            pool.estimate_host(h_hosts, hstage, ostage, h_outs[t])
    torch.cuda.synchronize()
    if use_plan:
        pool.plan_check(plan)
    for t in range(n_steps):
        ref.slice(slices[t])
        M = ref.readout()
        check_estimates(h_outs[t].numpy(), ref.estimate(M, hosts_np), est_floor(ref, M, hosts_np))
    assert np.array_equal(pool.export_regmax(), ref.readout())


def test_synth_cuda_twin_matches_numpy():
    for name in ("tiny", "caida", "caida_bursty"):
        tr = synth.CONFIGS[name]
        dt = synth.DeviceTrace(tr, DEV)
        for t, start, count in ((0, 0, 10_000), (3, 123_457, 40_001)):
            got = dt.generate(t, start, count).cpu().numpy().view(np.uint32).reshape(-1, 2)
            assert np.array_equal(got, synth.generate(tr, t, start, count))


@pytest.mark.parametrize("layout,pass_log2,scan_mode", [("fast", 0, 0), ("packed", 0, 0),
                                                       ("fast", 20, 2), ("packed", 0, 5)])
def test_caida_full_size(layout, pass_log2, scan_mode):
    """configs[1] 'caida' at full size (5M pairs/slice, 2^22 BDRs, m=128, k=5,
    500k hosts) in the launch configuration bench.py times: every register,
    the pool sums and all 500k host sums bit-exact, all estimates to 1e-9,
    DR state on a sample of BDRs, at several boundaries including a full window."""
    tr = synth.CONFIGS["caida"]
    cfg = oracle.PoolConfig(b=7, k=5, z=1 << 22)
    ref = oracle.Pool(cfg, "serial" if layout == "fast" else "gsmall")
    pool = VBDR(128, 5, 1 << 22, layout=layout, est_pass_log2=pass_log2, scan_mode=scan_mode,
                device=DEV)
    hosts_np = tr.host_ids()
    hosts = dev_u32(hosts_np)
    rng = np.random.default_rng(5)
    sample = np.sort(rng.choice(cfg.z, size=200_000, replace=False))
    for t in range(7):
        pairs = synth.generate(tr, t)  # numpy twin: the oracle never sees GPU-made data
        pool.scan_slice(dev_u32(pairs))
        pool.slide()
        ref.slice(pairs)
        if t in (0, 4, 6):
            M = ref.readout()
            assert np.array_equal(pool.export_regmax(), M)
            assert pool.export_pool_sums() == oracle_pool_sums(M, cfg.L)
            if layout == "fast":
                assert np.array_equal(pool.export_ages()[sample], ref.drv()[sample])
            else:
                assert np.array_equal(pool.export_ages(canonical=True)[sample], ref.ck()[sample])
            S, V = pool.host_sums(hosts)
            Z, Vo = ref.host_sums(M, hosts_np)
            assert np.array_equal(V.cpu().numpy().astype(np.uint64), Vo)
            assert np.array_equal(S.cpu().numpy().astype(np.float64) * 2.0 ** -cfg.L, Z)
            est = pool.estimate(hosts).cpu().numpy()
            check_estimates(est, ref.estimate(M, hosts_np), est_floor(ref, M, hosts_np))


@pytest.mark.parametrize("n_ranks", [2, 4, 8])
def test_loopback_multi_rank_merge(n_ranks):
    """N virtual ranks on one GPU: each scans a contiguous shard of every slice
    into its own pool, the stamp arrays merge by elementwise max (what the NCCL
    allreduce(MAX) does across GPUs), every rank slides; all replicas equal the
    single-rank pool and the oracle, and host-sharded estimates reassemble."""
    from paper_1810_13132_b200 import shard_range
    tr = synth.CONFIGS["tiny"]
    cfg = oracle.PoolConfig(b=5, k=4, z=1 << 12)
    ref = oracle.Pool(cfg, "serial")
    ranks = [VBDR(32, 4, 1 << 12, device=DEV) for _ in range(n_ranks)]
    hosts_np = tr.host_ids()
    for t in range(7):
        pairs = synth.generate(tr, t)
        for r, pool in enumerate(ranks):
            a, b = shard_range(len(pairs), r, n_ranks)
            pool.scan_slice(dev_u32(pairs[a:b]))
        merged = ranks[0].sr_view().clone()
        for pool in ranks[1:]:
            merged = torch.maximum(merged, pool.sr_view())
        for pool in ranks:
            pool.sr_view().copy_(merged)
            pool.slide()
        ref.slice(pairs)
        for pool in ranks:
            assert np.array_equal(pool.export_ages(), ref.drv())
            assert np.array_equal(pool.export_regmax(), ref.readout())
    M = ref.readout()
    parts = []
    for r, pool in enumerate(ranks):
        h0, h1 = shard_range(len(hosts_np), r, n_ranks)
        parts.append(pool.estimate(dev_u32(hosts_np[h0:h1])).cpu().numpy())
    check_estimates(np.concatenate(parts), ref.estimate(M, hosts_np), est_floor(ref, M, hosts_np))


@pytest.mark.parametrize("mode", ["delta", "sharded", "sparse", "sharded-state"])
@pytest.mark.parametrize("n_ranks", [2, 8])
def test_loopback_delta_merge(mode, n_ranks):
    """The u8-delta merges of slide_merged, with the collectives emulated on one
    GPU: 'delta' (elementwise max of the deltas, every rank slides all BDRs)
    and 'sharded' (rank r slides only its 1/N of the BDRs from the merged
    delta, then the registers are all-gathered and the pool sums all-reduced).
    'sparse' builds each rank's shard from the touched-BDR records the other
    ranks extracted for it (vbdr_sparse_extract / vbdr_sparse_apply, the
    all-to-all emulated) and must equal the merged delta's shard byte for byte.
    'sharded-state' is 'sharded' with register-sharded handles (drv_shards =
    N: each rank stores only its shard's DRV).
    Every rank's registers, its shard's DR ages, the pool sums and the
    host-sharded estimates are bit-exact / 1e-9 against the oracle."""
    from paper_1810_13132_b200 import shard_range
    tr = synth.CONFIGS["tiny"]
    cfg = oracle.PoolConfig(b=5, k=4, z=1 << 12)
    ref = oracle.Pool(cfg, "serial")
    if mode == "sharded-state":
        ranks = [VBDR(32, 4, 1 << 12, device=DEV, drv_shards=n_ranks, drv_shard=r)
                 for r in range(n_ranks)]
        full = VBDR(32, 4, 1 << 12, device=DEV)
        assert ranks[0].info()["state_bytes"] < full.info()["state_bytes"]
    else:
        ranks = [VBDR(32, 4, 1 << 12, device=DEV) for _ in range(n_ranks)]
    n = cfg.z // n_ranks
    hosts_np = tr.host_ids()
    for t in range(7):
        pairs = synth.generate(tr, t)
        for r, pool in enumerate(ranks):
            a, b = shard_range(len(pairs), r, n_ranks)
            pool.scan_slice(dev_u32(pairs[a:b]))
        deltas = [pool.stamp_delta() for pool in ranks]
        merged = deltas[0].clone()
        for d in deltas[1:]:
            merged = torch.maximum(merged, d)
        ref.slice(pairs)
        if mode == "delta":
            for pool in ranks:
                pool.slide_delta(merged)
        else:
            if mode == "sparse":
                out = [pool.sparse_extract(n_ranks) for pool in ranks]
                # SparseMerge's fixed-capacity form: zero-initialised rows of
                # a larger cap (slots past each count stay zero)
                cap = max(int(c.max()) for _, c in out) + 37
                rows_all = []
                for src in ranks:
                    rows = torch.zeros((n_ranks, cap), dtype=torch.int32, device=DEV)
                    cnt = torch.empty(n_ranks, dtype=torch.int64, device=DEV)
                    src.sparse_extract_into(rows, cnt)
                    rows_all.append(rows)
                for src, (rec, cnt) in enumerate(out):  # the touched BDRs, exactly
                    d = deltas[src].cpu().numpy()
                    for o in range(n_ranks):
                        got = rec[o, :int(cnt[o])].cpu().numpy().view(np.uint32)
                        pos = (got >> 5).astype(np.int64)
                        assert np.array_equal(np.sort(pos), np.flatnonzero(d[o * n:(o + 1) * n]))
                        assert np.array_equal(d[o * n + pos], (got & 31).astype(np.uint8))
            for r, pool in enumerate(ranks):
                if mode == "sparse":
                    shard = torch.zeros(n, dtype=torch.uint8, device=DEV)
                    for rec, cnt in out:
                        pool.sparse_apply(rec[r, :int(cnt[r])].contiguous(), shard)
                    assert torch.equal(shard, merged[r * n:(r + 1) * n])
                    # the padded rows applied whole: zero records are no-ops
                    padded = torch.zeros(n, dtype=torch.uint8, device=DEV)
                    for rows in rows_all:
                        pool.sparse_apply(rows[r].contiguous(), padded)
                    assert torch.equal(padded, shard)
                else:
                    shard = merged[r * n:(r + 1) * n].clone()
                pool.slide_delta(shard, r * n, (r + 1) * n)
            full = torch.cat([pool.regmax_view()[r * n:(r + 1) * n] for r, pool in enumerate(ranks)])
            acc = sum(pool.acc_view() for pool in ranks)
            for pool in ranks:
                pool.regmax_view().copy_(full)
                pool.acc_view().copy_(acc)
        M = ref.readout()
        drv = ref.drv()
        for r, pool in enumerate(ranks):
            assert np.array_equal(pool.export_regmax(), M)
            assert pool.export_pool_sums() == oracle_pool_sums(M, cfg.L)
            j0, j1 = (0, cfg.z) if mode == "delta" else (r * n, (r + 1) * n)
            if mode == "sharded-state":  # only the shard's DRV exists
                idx = np.arange(j0, j1, dtype=np.uint64)
                assert np.array_equal(pool.export_ages_at(idx), drv[j0:j1])
            else:
                assert np.array_equal(pool.export_ages()[j0:j1], drv[j0:j1])
    parts = []
    for r, pool in enumerate(ranks):
        h0, h1 = shard_range(len(hosts_np), r, n_ranks)
        parts.append(pool.estimate(dev_u32(hosts_np[h0:h1])).cpu().numpy())
    check_estimates(np.concatenate(parts), ref.estimate(M, hosts_np), est_floor(ref, M, hosts_np))


def test_delta_matches_stamps():
    tr = synth.CONFIGS["tiny"]
    pool = VBDR(32, 4, 1 << 12, device=DEV)
    cfg = oracle.PoolConfig(b=5, k=4, z=1 << 12)
    for t in range(3):
        pairs = synth.generate(tr, t)
        pool.scan_slice(dev_u32(pairs))
        d = pool.stamp_delta().cpu().numpy()
        o = oracle.Pool(cfg, "serial")
        o.begin_slice()
        o.scan(pairs)
        assert np.array_equal(d, o.now())  # the paper's nowLBP1
        pool.slide()


@pytest.mark.parametrize("layout", ["fast", "packed"])
def test_tick_wraparound(layout):
    """Stamps are (T << 5) | rho with T < 2^26; at the limit the slide clears
    the stamps and restarts T.  Parity must hold straight through the wrap."""
    tr = synth.CONFIGS["tiny"]
    cfg = oracle.PoolConfig(b=5, k=4, z=1 << 12)
    ref = oracle.Pool(cfg, "serial" if layout == "fast" else "gsmall")
    pool = VBDR(32, 4, 1 << 12, layout=layout, device=DEV)
    pool.debug_set_tick((1 << 26) - 7)  # 1 mod 4: register buffers / sum slots rotate
    hosts_np = tr.host_ids()
    for t in range(10):
        pairs = synth.generate(tr, t)
        pool.scan_slice(dev_u32(pairs))
        pool.slide()
        ref.slice(pairs)
        compare_boundary(pool, ref, [], hosts_np, dev_u32(hosts_np), None)
    assert pool.info()["tick"] < 16


def test_abi_errors():
    """Argument and state errors are reported synchronously, nothing launched
    (scan mode 5: one launch per scan call)."""
    pool = VBDR(32, 4, 1 << 12, device=DEV, scan_mode=5)
    before = pool.info()["launches"]
    bad = torch.zeros(9, dtype=torch.int32, device=DEV)[1:]  # 4-byte aligned only
    with pytest.raises(RuntimeError, match="EINVAL"):
        pool.scan_slice(bad)
    with pytest.raises(RuntimeError, match="EINVAL"):
        pool.slide_delta(torch.zeros(8192, dtype=torch.uint8, device=DEV), 0, 4097)
    with pytest.raises(RuntimeError, match="EINVAL"):
        pool.slide_delta(torch.zeros(4096, dtype=torch.uint8, device=DEV), 2, 10)
    with pytest.raises(RuntimeError, match="ESTATE"):
        VBDR(32, 4, 1 << 12, layout="packed", device=DEV).stamp_delta()
    with pytest.raises(RuntimeError, match="EINVAL"):
        pool.debug_set_tick(2)
    pool.scan_slice(dev_u32(synth.generate(synth.CONFIGS["tiny"], 0)))
    pool.slide()
    with pytest.raises(RuntimeError, match="ESTATE"):
        pool.debug_set_tick(101)
    assert pool.info()["launches"] == before + 2
    # empty inputs are legal no-ops
    pool.scan_slice(torch.zeros(0, dtype=torch.int32, device=DEV))
    assert pool.estimate(torch.zeros(0, dtype=torch.int32, device=DEV)).numel() == 0


@pytest.mark.parametrize("kind", ["staged", "sorted"])
def test_plan_estimate_all_zero_registers(kind):
    """Hosts whose registers are all zero (a fresh pool, and every host after
    the window has passed with empty slices): the staged plan's zero count
    holds V 2^L mod 2^32, which wraps to 0 exactly then (V = g, S' = 0).
    Sums and estimates equal the gather kernel's and the oracle's."""
    tr = synth.CONFIGS["tiny"]
    cfg = oracle.PoolConfig(b=5, k=4, z=1 << 12)
    ref = oracle.Pool(cfg, "serial")
    pool = VBDR(32, 4, 1 << 12, device=DEV)
    hosts_np = tr.host_ids()
    hosts = dev_u32(hosts_np)
    plan = pool.plan(hosts, kind=kind)
    empty = np.zeros((0, 2), np.uint32)
    for t, pairs in enumerate([empty, synth.generate(tr, 1), empty, empty, empty, empty, empty]):
        if len(pairs):
            pool.scan_slice(dev_u32(pairs))
        pool.slide()
        ref.slice(pairs)
        S1, V1 = pool.host_sums_plan(plan)
        S2, V2 = pool.host_sums(hosts)
        assert torch.equal(S1, S2) and torch.equal(V1, V2)
        a = pool.estimate_plan(plan).cpu().numpy()
        assert np.array_equal(a, pool.estimate(hosts).cpu().numpy())
        M = ref.readout()
        if not M.any():  # every register zero: V = g for every host
            assert (V1.cpu().numpy() == 32).all()
        check_estimates(a, ref.estimate(M, hosts_np), est_floor(ref, M, hosts_np))
    pool.plan_check(plan)


def test_plan_abi_errors():
    """Plan calls fail loudly and launch nothing: a plan of another handle, a
    released plan, a buffer too small or misaligned, an unknown kind."""
    import ctypes as C
    from paper_1810_13132_b200.vbdr import lib
    a = VBDR(32, 4, 1 << 12, device=DEV)
    b = VBDR(32, 4, 1 << 12, device=DEV)
    hosts = dev_u32(synth.CONFIGS["tiny"].host_ids())
    plan = a.plan(hosts, kind="staged")
    before = b.info()["launches"]
    with pytest.raises(RuntimeError, match="EINVAL"):
        b.estimate_plan(plan)  # built by handle a
    assert b.info()["launches"] == before
    p2 = a.plan(hosts, kind="sorted")
    ptr = p2.buf.data_ptr()
    p2.release()
    with pytest.raises(ValueError, match="released"):
        a.estimate_plan(p2)
    out = torch.empty(hosts.numel(), dtype=torch.float64, device=DEV)
    assert lib().vbdr_estimate_plan(a._h, C.c_void_p(ptr), C.c_void_p(out.data_ptr()), None) == -1
    need = C.c_uint64()
    assert lib().vbdr_plan_bytes_kind(a._h, hosts.numel(), 1, C.byref(need)) == 0
    buf = torch.empty(need.value + 512, dtype=torch.uint8, device=DEV)
    rc = lib().vbdr_plan_build_kind(a._h, C.c_void_p(hosts.data_ptr()), hosts.numel(), 1,
                                    C.c_void_p(buf.data_ptr()), need.value - 256, None)
    assert rc == -4  # ENOMEM: buffer too small
    rc = lib().vbdr_plan_build_kind(a._h, C.c_void_p(hosts.data_ptr()), hosts.numel(), 1,
                                    C.c_void_p(buf.data_ptr() + 16), need.value, None)
    assert rc == -1  # EINVAL: not 256-byte aligned
    assert lib().vbdr_plan_bytes_kind(a._h, hosts.numel(), 9, C.byref(need)) == -1
    with pytest.raises(KeyError):
        a.plan(hosts, kind="nope")
    # the plan of handle a still works
    assert np.array_equal(a.estimate_plan(plan).cpu().numpy(), a.estimate(hosts).cpu().numpy())


@pytest.mark.parametrize("n_ranks", [2, 4, 8])
def test_loopback_fused_peer_merge_slide(n_ranks):
    """vbdr_slide_peers with virtual peers on one GPU: rank r's kernel reads
    every rank's delta in place for its BDR shard, merges with a per-byte max,
    slides the shard and writes registers and pool sums into every rank.  The
    same kernel runs over NVLink-mapped peer pointers on a multi-GPU box."""
    from paper_1810_13132_b200 import shard_range
    tr = synth.CONFIGS["tiny"]
    cfg = oracle.PoolConfig(b=5, k=4, z=1 << 12)
    ref = oracle.Pool(cfg, "serial")
    ranks = [VBDR(32, 4, 1 << 12, device=DEV) for _ in range(n_ranks)]
    deltas = [torch.empty(cfg.z, dtype=torch.uint8, device=DEV) for _ in range(n_ranks)]
    n = cfg.z // n_ranks
    acc = [p.acc_ptr() for p in ranks]
    hosts_np = tr.host_ids()
    for t in range(7):
        pairs = synth.generate(tr, t)
        regmax = [p.regmax_ptr(next=True) for p in ranks]  # alternates with the tick
        for r, pool in enumerate(ranks):
            a, b = shard_range(len(pairs), r, n_ranks)
            pool.scan_slice(dev_u32(pairs[a:b]))
            pool.stamp_delta(deltas[r])
        for r, pool in enumerate(ranks):
            pool.slide_peers([d.data_ptr() for d in deltas], r * n, (r + 1) * n, regmax, acc)
        ref.slice(pairs)
        M = ref.readout()
        drv = ref.drv()
        for r, pool in enumerate(ranks):
            assert np.array_equal(pool.export_regmax(), M)
            assert pool.export_pool_sums() == oracle_pool_sums(M, cfg.L)
            assert np.array_equal(pool.export_ages()[r * n:(r + 1) * n], drv[r * n:(r + 1) * n])
    parts = []
    for r, pool in enumerate(ranks):
        h0, h1 = shard_range(len(hosts_np), r, n_ranks)
        parts.append(pool.estimate(dev_u32(hosts_np[h0:h1])).cpu().numpy())
    check_estimates(np.concatenate(parts), ref.estimate(M, hosts_np), est_floor(ref, M, hosts_np))
    # without peer register/accumulator lists it is a local merge + slide
    solo = VBDR(32, 4, 1 << 12, device=DEV)
    ref2 = oracle.Pool(cfg, "serial")
    pairs = synth.generate(tr, 0)
    solo.scan_slice(dev_u32(pairs))
    d = solo.stamp_delta()
    solo.slide_peers([d.data_ptr()], 0, cfg.z)
    ref2.slice(pairs)
    assert np.array_equal(solo.export_ages(), ref2.drv())


def variant_floor(V, hosts, b, z, estimator):
    """C * E_s / g per host for the LogLog / PCSA estimators (tolerance floor)."""
    g = 1 << b
    C = (z * g) / (z - g)
    out = []
    for aip in hosts:
        regs = np.array([V[oracle.getPhyIdx(int(aip), i, 0x5EED0001, z)] for i in range(g)],
                        np.uint8)
        Es = oracle.loglog_raw(regs) if estimator == "loglog" else oracle.pcsa_raw(regs)
        out.append(C * Es / g)
    return np.array(out)


@pytest.mark.parametrize("layout,estimator", [("fast", "loglog"), ("packed", "loglog"),
                                              ("packed", "pcsa")])
def test_estimator_variants_tiny(layout, estimator):
    """N4: the BDR pool under LogLog (Alg.5's sum of LBP1) and PCSA (sliding
    FM bitmap = the gsmall DRV's active ranks), bit-exact registers and sums,
    estimates to 1e-9 against the oracle, at every boundary."""
    tr = synth.CONFIGS["tiny"]
    cfg = oracle.PoolConfig(b=5, k=4, z=1 << 12)
    ref = oracle.Pool(cfg, "serial" if layout == "fast" else "gsmall")
    pool = VBDR(32, 4, 1 << 12, layout=layout, estimator=estimator, device=DEV)
    hosts_np = tr.host_ids()
    hosts = dev_u32(hosts_np)
    assert (pool.estimate(hosts).cpu().numpy() == 0).all() or estimator != "hll"
    for t in range(9):
        pairs = synth.generate(tr, t)
        pool.scan_slice(dev_u32(pairs))
        pool.slide()
        ref.slice(pairs)
        V = ref.readout_pcsa() if estimator == "pcsa" else ref.readout()
        assert np.array_equal(pool.export_regmax(), V)
        assert pool.export_pool_sums() == (int(V.astype(np.int64).sum()), int((V == 0).sum()))
        S, Vz = pool.host_sums(hosts)
        for h, aip in enumerate(hosts_np[:16]):
            regs = np.array([V[oracle.getPhyIdx(int(aip), i, cfg.A0, cfg.z)] for i in range(32)])
            assert int(S[h]) == int(regs.sum()) and int(Vz[h]) == int((regs == 0).sum())
        est = pool.estimate(hosts).cpu().numpy()
        want = oracle.estimate_variant(V, hosts_np, cfg.b, cfg.z, estimator)
        check_estimates(est, want, variant_floor(V, hosts_np, cfg.b, cfg.z, estimator))


def test_pcsa_needs_packed():
    with pytest.raises(ValueError):
        VBDR(32, 4, 1 << 12, layout="fast", estimator="pcsa", device=DEV)


@pytest.mark.parametrize("layout,estimator", [("fast", "loglog"), ("packed", "pcsa")])
def test_estimator_variants_caida(layout, estimator):
    tr = synth.CONFIGS["caida"]
    cfg = oracle.PoolConfig(b=7, k=5, z=1 << 22)
    ref = oracle.Pool(cfg, "serial" if layout == "fast" else "gsmall")
    pool = VBDR(128, 5, 1 << 22, layout=layout, estimator=estimator, device=DEV)
    hosts_np = tr.host_ids()
    sample = hosts_np[np.random.default_rng(2).choice(len(hosts_np), 3000, replace=False)]
    for t in range(6):
        pairs = synth.generate(tr, t)
        pool.scan_slice(dev_u32(pairs))
        pool.slide()
        ref.slice(pairs)
    V = ref.readout_pcsa() if estimator == "pcsa" else ref.readout()
    assert np.array_equal(pool.export_regmax(), V)
    assert pool.export_pool_sums() == (int(V.astype(np.int64).sum()), int((V == 0).sum()))
    est = pool.estimate(dev_u32(sample)).cpu().numpy()
    want = oracle.estimate_variant(V, sample, cfg.b, cfg.z, estimator)
    check_estimates(est, want, variant_floor(V, sample, cfg.b, cfg.z, estimator))
    # the bench's plan path for all 500k hosts: bit-identical to the gather
    hosts = dev_u32(hosts_np)
    plan = pool.plan(hosts)
    assert np.array_equal(pool.estimate_plan(plan).cpu().numpy(),
                          pool.estimate(hosts).cpu().numpy())
    pool.plan_check(plan)


@pytest.mark.parametrize("layout", ["fast", "packed"])
@pytest.mark.parametrize("m,n_phys,k,zbits,rank_cap", [(1 << 14, 1 << 16, 3, 0, 0),
                                                      (64, 1 << 12, 4, 5, 9),
                                                      (4, 1 << 8, 2, 0, 1)])
def test_unusual_configs(layout, m, n_phys, k, zbits, rank_cap):
    """Huge virtual vectors (g = 2^14 > the shared s1 table), explicit wide DRs,
    a rank cap (R#3: rho = min(rho, L)), and L = 1."""
    b = m.bit_length() - 1
    cfg = oracle.PoolConfig(b=b, k=k, z=n_phys, zb=zbits, L=rank_cap)
    if layout == "packed" and zbits == 0 and (1 << cfg.zb) - 2 < k:
        cfg = oracle.PoolConfig(b=b, k=k, z=n_phys, zb=cfg.zb + 1, L=rank_cap)
    ref = oracle.Pool(cfg, "serial" if layout == "fast" else "gsmall")
    pool = VBDR(m, k, n_phys, layout=layout, zbits=zbits, rank_cap=rank_cap, device=DEV)
    tr = synth.TraceConfig("odd", hosts=300, pairs_per_slice=5001, U0=5000, seed=m + k)
    hosts_np = tr.host_ids()
    slices = []
    for t in range(k + 3):
        pairs = synth.generate(tr, t)
        slices.append(pairs)
        pool.scan_slice(dev_u32(pairs))
        pool.slide()
        ref.slice(pairs)
    compare_boundary(pool, ref, [], hosts_np, dev_u32(hosts_np),
                     np.concatenate(slices[-k:]))


@pytest.mark.parametrize("kind", ["sorted", "staged"])
@pytest.mark.parametrize("layout,estimator", [("fast", "hll"), ("packed", "hll"),
                                              ("packed", "pcsa"), ("fast", "loglog")])
def test_plan_estimate_tiny(layout, estimator, kind):
    """vbdr_estimate_plan: plan sums equal the gather kernel's bit for bit and
    the oracle to 1e-9, at every boundary."""
    tr = synth.CONFIGS["tiny"]
    cfg = oracle.PoolConfig(b=5, k=4, z=1 << 12)
    ref = oracle.Pool(cfg, "serial" if layout == "fast" else "gsmall")
    pool = VBDR(32, 4, 1 << 12, layout=layout, estimator=estimator, device=DEV)
    hosts_np = tr.host_ids()
    hosts = dev_u32(hosts_np)
    plan = pool.plan(hosts, kind=kind)
    for t in range(7):
        pairs = synth.generate(tr, t)
        pool.scan_slice(dev_u32(pairs))
        pool.slide()
        ref.slice(pairs)
        a = pool.estimate_plan(plan).cpu().numpy()
        b = pool.estimate(hosts).cpu().numpy()
        assert np.array_equal(a, b)
        S1, V1 = pool.host_sums_plan(plan)
        S2, V2 = pool.host_sums(hosts)
        assert torch.equal(S1, S2) and torch.equal(V1, V2)
        if estimator == "hll":
            check_estimates(a, ref.estimate(ref.readout(), hosts_np),
                            est_floor(ref, ref.readout(), hosts_np))
    pool.plan_check(plan)


@pytest.mark.parametrize("kind", ["auto", "sorted", "staged"])
def test_plan_estimate_caida_full_size(kind):
    """configs[1] at full size: the plan covers all 500k hosts of the bench."""
    tr = synth.CONFIGS["caida"]
    cfg = oracle.PoolConfig(b=7, k=5, z=1 << 22)
    ref = oracle.Pool(cfg, "serial")
    pool = VBDR(128, 5, 1 << 22, device=DEV)
    hosts_np = tr.host_ids()
    hosts = dev_u32(hosts_np)
    plan = pool.plan(hosts, kind=kind)
    for t in range(6):
        pairs = synth.generate(tr, t)
        pool.scan_slice(dev_u32(pairs))
        pool.slide()
        ref.slice(pairs)
    a = pool.estimate_plan(plan).cpu().numpy()
    assert np.array_equal(a, pool.estimate(hosts).cpu().numpy())
    M = ref.readout()
    check_estimates(a, ref.estimate(M, hosts_np), est_floor(ref, M, hosts_np))
    pool.plan_check(plan)


@pytest.mark.parametrize("kind", ["sorted", "staged"])
@pytest.mark.parametrize("g,z_log2,n_hosts", [(64, 12, 1001), (16, 12, 3),
                                               (32, 20, 7 * 512 * 148 - 5), (2, 7, 33),
                                               (256, 24, 300_001), (128, 22, 1_200_001)])
def test_plan_accumulator_modes_and_ragged_hosts(g, z_log2, n_hosts, kind):
    """Plan rounds for a host list with duplicates and a ragged tail, for 3
    hosts (almost every round is padding) and for the largest host count a
    plan takes (20 blocks of 2^16 registers): bit-identical to the gather
    estimate and sums."""
    tr = synth.CONFIGS["tiny"]
    pool = VBDR(g, 4, 1 << z_log2, device=DEV)
    rng = np.random.default_rng(g + n_hosts)
    hosts_np = rng.integers(0, 2**32, n_hosts, dtype=np.uint64).astype(np.uint32)
    hosts_np[1::7][:64] = hosts_np[0]  # duplicates (many would pile into a few blocks)
    hosts = dev_u32(hosts_np)
    if kind == "staged" and z_log2 > 22:
        with pytest.raises(ValueError):
            pool.plan(hosts, kind=kind)
        return
    plan = pool.plan(hosts, kind=kind)
    for t in range(6):
        pool.scan_slice(dev_u32(synth.generate(tr, t)))
        pool.slide()
        if t >= 3:
            assert np.array_equal(pool.estimate_plan(plan).cpu().numpy(),
                                  pool.estimate(hosts).cpu().numpy())
            S1, V1 = pool.host_sums_plan(plan)
            S2, V2 = pool.host_sums(hosts)
            assert torch.equal(S1, S2) and torch.equal(V1, V2)
    pool.plan_check(plan)


@pytest.mark.parametrize("g,pass_log2", [(64, 21), (128, 22), (256, 21), (2048, 22)])
def test_pass_id_plan_multipass(g, pass_log2):
    """Pools beyond the staged plan whose gather estimate runs in 2..4 passes
    get a pass-id plan: estimates and sums bit-identical to the gather kernel's
    (duplicate hosts, a ragged host count, g / 64 = 1..32 lanes)."""
    tr = synth.CONFIGS["tiny"]
    pool = VBDR(g, 4, 1 << 23, est_pass_log2=pass_log2, device=DEV)
    rng = np.random.default_rng(g)
    hosts_np = rng.integers(0, 2**32, 3001, dtype=np.uint64).astype(np.uint32)
    hosts_np[5::11] = hosts_np[0]
    hosts_np[:64] = tr.host_ids()  # hosts with traffic
    hosts = dev_u32(hosts_np)
    plan = pool.plan(hosts, kind="passid")
    before = pool.info()["launches"]
    for t in range(5):
        pool.scan_slice(dev_u32(synth.generate(tr, t)))
        pool.slide()
        a = pool.estimate_plan(plan).cpu().numpy()
        assert np.array_equal(a, pool.estimate(hosts).cpu().numpy())
        S1, V1 = pool.host_sums_plan(plan)
        S2, V2 = pool.host_sums(hosts)
        assert torch.equal(S1, S2) and torch.equal(V1, V2)
    assert pool.info()["launches"] > before
    pool.plan_check(plan)


def test_plan_refuses_what_does_not_fit():
    """staged: pools above 2^22 BDRs; sorted: a group's accumulators beyond the
    SM's shared memory; auto: neither (and one estimate pass, so no pass ids)."""
    pool = VBDR(256, 10, 1 << 23, device=DEV)
    with pytest.raises(ValueError):
        pool.plan(dev_u32(np.arange(10, dtype=np.uint32)), kind="staged")
    many = torch.arange(6_000_000, dtype=torch.int32, device=DEV)
    with pytest.raises(ValueError):
        pool.plan(many, kind="sorted")
    with pytest.raises(ValueError):
        pool.plan(many)
    with pytest.raises(KeyError):
        pool.plan(many, kind="nope")


def test_query_top_super_spreaders():
    """hosts at or above a threshold, sorted by estimate
    (descending), ties by ascending aip -- against the oracle's estimates."""
    tr = synth.CONFIGS["tiny"]
    cfg = oracle.PoolConfig(b=5, k=4, z=1 << 12)
    ref = oracle.Pool(cfg, "serial")
    pool = VBDR(32, 4, 1 << 12, device=DEV)
    hosts_np = tr.host_ids()
    hosts = dev_u32(hosts_np)
    for t in range(6):
        pairs = synth.generate(tr, t)
        pool.scan_slice(dev_u32(pairs))
        pool.slide()
        ref.slice(pairs)
    want = ref.estimate(ref.readout(), hosts_np)
    for thr in (0.0, 100.0, 500.0, 1e9):
        aips, ests = pool.query_top(hosts, thr)
        sel = want >= thr
        exp_a = hosts_np[sel]
        order = np.lexsort((exp_a, -want[sel]))
        assert np.array_equal(aips, exp_a[order]), thr
        assert np.allclose(ests, want[sel][order], rtol=1e-9)
    plan = pool.plan(hosts)
    a2, e2 = pool.query_top(hosts, 100.0, plan=plan)
    a1, e1 = pool.query_top(hosts, 100.0)
    assert np.array_equal(a1, a2) and np.array_equal(e1, e2)


@pytest.mark.parametrize("via", ["self", "multicast"])
@pytest.mark.parametrize("layout,estimator", [("fast", "hll"), ("packed", "hll"),
                                              ("packed", "pcsa"), ("fast", "loglog")])
def test_nvls_slide_one_device(layout, estimator, via):
    """vbdr_slide_multicast (the fused NVLS merge + slide) for a
    group of one GPU: "multicast" through a one-device multicast object
    (vbdr_mc_alloc: multimem.ld_reduce MAX of the stamps / AND of the packed
    words, multimem.st of registers and words, multimem.red of the pool
    sums); "self" with the handle's own state as the group address (the same
    kernel, the multimem operations replaced by what they reduce to over one
    member).  Every boundary of 11 slices (past k: expired, unsaturated DRs)
    is bit-exact against the oracle; estimates within 1e-9."""
    from paper_1810_13132_b200 import McBuffer, make_config, state_bytes
    tr = synth.CONFIGS["tiny"]
    cfg = oracle.PoolConfig(b=5, k=4, z=1 << 12)
    buf = None
    state = None
    if via == "multicast":
        nbytes = state_bytes(make_config(32, 4, 1 << 12, layout=layout, estimator=estimator))
        try:
            buf = McBuffer(nbytes, DEV)
        except RuntimeError as e:  # e.g. cuMulticastCreate refused in this container
            pytest.skip(f"no multicast object on this device: {e}")
        state = buf.tensor
    try:
        pool = VBDR(32, 4, 1 << 12, layout=layout, estimator=estimator, device=DEV, state=state)
        mc = buf.mc if buf is not None else pool.state.data_ptr()
        ref = oracle.Pool(cfg, "serial" if layout == "fast" else "gsmall")
        hosts_np = tr.host_ids()
        hosts = dev_u32(hosts_np)
        slices = []
        for t in range(11):
            pairs = synth.generate(tr, t)
            slices.append(pairs)
            pool.scan_slice(dev_u32(pairs))
            pool.slide_multicast(mc)
            ref.slice(pairs)
            if estimator == "hll":
                compare_boundary(pool, ref, [], hosts_np, hosts, np.concatenate(slices[-4:]))
                continue
            V = ref.readout_pcsa() if estimator == "pcsa" else ref.readout()
            assert np.array_equal(pool.export_regmax(), V)
            assert pool.export_pool_sums() == (int(V.astype(np.int64).sum()), int((V == 0).sum()))
            est = pool.estimate(hosts).cpu().numpy()
            want = oracle.estimate_variant(V, hosts_np, cfg.b, cfg.z, estimator)
            check_estimates(est, want, variant_floor(V, hosts_np, cfg.b, cfg.z, estimator))
        assert pool.info()["slices_closed"] == 11
        pool.close()
        torch.cuda.synchronize()
    finally:
        if buf is not None:
            buf.free()


def test_nvls_slide_shard_self():
    """The multicast slide over a register-sharded handle's shard [j0, j1)
    (layout fast, drv_shards = 2): a rank of two closes its shard; ranges
    outside the shard are refused."""
    tr = synth.CONFIGS["tiny"]
    cfg = oracle.PoolConfig(b=5, k=4, z=1 << 12)
    ref = oracle.Pool(cfg, "serial")
    n = cfg.z // 2
    pools = [VBDR(32, 4, 1 << 12, device=DEV, drv_shards=2, drv_shard=r) for r in range(2)]
    with pytest.raises(RuntimeError):
        pools[0].slide_multicast(pools[0].state.data_ptr(), n, 2 * n)  # not its shard
    for t in range(7):
        pairs = synth.generate(tr, t)
        ref.slice(pairs)
        for r, pool in enumerate(pools):
            pool.scan_slice(dev_u32(pairs))  # the whole slice on both (no merge to emulate)
            pool.slide_multicast(pool.state.data_ptr(), r * n, (r + 1) * n)
        M = ref.readout()
        for r, pool in enumerate(pools):
            assert np.array_equal(pool.export_regmax()[r * n:(r + 1) * n], M[r * n:(r + 1) * n])
            ages = pool.export_ages_at(np.arange(r * n, (r + 1) * n, dtype=np.uint64))
            assert np.array_equal(ages, ref.drv()[r * n:(r + 1) * n])


def test_nvls_slide_rejects_bad_ranges():
    pool = VBDR(32, 4, 1 << 12, device=DEV)
    base = pool.state.data_ptr()
    for j0, j1 in ((0, 0), (2, 64), (0, (1 << 12) + 4)):
        with pytest.raises(RuntimeError):
            pool.slide_multicast(base, j0, j1)
    with pytest.raises(RuntimeError):
        pool.slide_multicast(base + 16)  # not 256-byte aligned
    packed = VBDR(32, 4, 1 << 12, layout="packed", device=DEV)
    packed.slide_multicast(packed.state.data_ptr())  # full range: fine


@pytest.mark.parametrize("estimator,scan_mode", [("hll", 0), ("hll", 2), ("pcsa", 0),
                                                 ("loglog", 5)])
def test_stamps_layout_tiny(estimator, scan_mode):
    """Layout S (per-(BDR, rank) last-seen stamps) against the
    oracle's VBDR-gsmall pool (Alg.8 + Alg.9): canonical C_k = min(age, k),
    registers, pool sums and estimates at every boundary of 12 slices, ragged
    batches, an empty slice."""
    tr = synth.CONFIGS["tiny"]
    cfg = oracle.PoolConfig(b=5, k=4, z=1 << 12)
    ref = oracle.Pool(cfg, "gsmall")
    pool = VBDR(32, 4, 1 << 12, layout="stamps", estimator=estimator, scan_mode=scan_mode,
                device=DEV)
    inf = pool.info()
    assert inf["words"] == cfg.L and inf["fields"] == 1
    hosts_np = tr.host_ids()
    hosts = dev_u32(hosts_np)
    slices = []
    for t in range(12):
        pairs = synth.generate(tr, t) if t != 6 else np.zeros((0, 2), np.uint32)
        slices.append(pairs)
        for a, b in ((0, 3), (3, 4001), (4001, len(pairs))):
            if b > a:
                pool.scan_slice(dev_u32(pairs[a:b]))
        pool.slide()
        ref.slice(pairs)
        assert np.array_equal(pool.export_ages(canonical=True), ref.ck()), "C_k"
        if estimator == "hll":
            compare_boundary(pool, ref, [], hosts_np, hosts, np.concatenate(slices[-4:]),
                             check_ages=False)
            continue
        V = ref.readout_pcsa() if estimator == "pcsa" else ref.readout()
        assert np.array_equal(pool.export_regmax(), V)
        assert pool.export_pool_sums() == (int(V.astype(np.int64).sum()), int((V == 0).sum()))
        est = pool.estimate(hosts).cpu().numpy()
        want = oracle.estimate_variant(V, hosts_np, cfg.b, cfg.z, estimator)
        check_estimates(est, want, variant_floor(V, hosts_np, cfg.b, cfg.z, estimator))


def test_stamps_layout_caida_sampled():
    """Layout S at the caida pool (2^22 BDRs, 100 planes of stamps = 400 MiB),
    k + 2 full-size slices: registers = the rebuild from the window's pairs,
    exact pool sums, sampled hosts' estimates against the oracle."""
    tr = synth.CONFIGS["caida"]
    b, k, z = 7, 5, 1 << 22
    L = 32 - b
    pool = VBDR(128, k, z, layout="stamps", device=DEV)
    per_slice = []
    for t in range(k + 2):
        pairs = synth.generate(tr, t)
        pool.scan_slice(dev_u32(pairs))
        pool.slide()
        per_slice.append(oracle.rebuild(pairs, b, L, z, 0x5EED0001, 0x5EED0002))
    M = per_slice[-k]
    for x in per_slice[-k + 1:]:
        M = np.maximum(M, x)
    assert np.array_equal(pool.export_regmax(), M)
    assert pool.export_pool_sums() == oracle_pool_sums(M, L)
    hosts = tr.host_ids()[:: 997]
    est = pool.estimate(dev_u32(hosts)).cpu().numpy()
    want = oracle.estimate_M(M, hosts, b, z)
    assert np.allclose(est, want, rtol=1e-9, atol=1e-9 * np.abs(want).max())
