"""Pins for the distance recorder and single-BDR algorithms (PAPER.md:89-140,
222-277): SPEC.md example vectors and the sliding-correctness property against
a brute-force windowed maximum (acceptance 1 at SPEC.md:517)."""
import ctypes as C

import numpy as np
import pytest

import oracle


def _dr(v):
    return C.c_uint16(v)


def test_dr_ops_spec_vectors():
    L = oracle.lib()
    d = _dr(0)
    # InitDR
    for zb, want in ((3, 7), (1, 1), (8, 255)):
        L.orc_InitDR(C.byref(d), zb)
        assert d.value == want
    # SetDR
    for v in (7, 0, 3):
        d.value = v
        L.orc_SetDR(C.byref(d))
        assert d.value == 0
    # SlideDR saturating (R#1)
    for v, want in ((0, 1), (6, 7), (7, 7)):
        d.value = v
        L.orc_SlideDR(C.byref(d), 3)
        assert d.value == want
    # IsActiveDR
    assert L.orc_IsActiveDR(3, 5) == 1
    assert L.orc_IsActiveDR(5, 5) == 0
    assert L.orc_IsActiveDR(7, 5) == 0


def test_alg1_end_slice_serial_traces():
    # k=4, zb=3, all 7, nowLBP1=5 -> drv[5]=0, others 7
    d = oracle.bdr_end_slice_serial(np.full(10, 7), 3, 5)
    assert d[4] == 0 and all(d[i] == 7 for i in range(10) if i != 4)
    # nowLBP1=0, drv[2]=1 -> drv[2]=2, nothing set (R#9)
    d0 = np.full(10, 7)
    d0[1] = 1
    d = oracle.bdr_end_slice_serial(d0, 3, 0)
    assert d[1] == 2 and (d[np.arange(10) != 1] == 7).all()


def test_alg6_end_slice_gfast_trace():
    # bits {2,5} -> drv[5]=0, drv[2] only slid (R#10)
    d0 = np.full(10, 3)
    d = oracle.bdr_end_slice_gfast(d0, 3, (1 << 1) | (1 << 4))
    assert d[4] == 0 and d[1] == 4 and (d[[0, 2, 3, 5, 6, 7, 8, 9]] == 4).all()
    # empty bit string: only slides
    assert (oracle.bdr_end_slice_gfast(d0, 3, 0) == 4).all()


def test_alg8_begin_slice_traces():
    # SPEC.md:111-113
    assert oracle.bdr_begin_slice_gsmall(np.array([0, 3, 7]), 3).tolist() == [1, 4, 7]
    assert (oracle.bdr_begin_slice_gsmall(np.full(5, 7), 3) == 7).all()
    k = 4
    d = oracle.bdr_begin_slice_gsmall(np.array([k - 1]), 3)
    assert d[0] == k and oracle.bdr_GetLBP1(d, k) == 0


def test_alg2_readout_traces():
    k, zb, L = 4, 3, 12
    S = (1 << zb) - 1
    # fresh -> 0
    assert oracle.bdr_GetLBP1(np.full(L, S), k) == 0
    # drv[5]=0, drv[9]=k (expired), rest sentinel -> 5
    d = np.full(L, S)
    d[4] = 0
    d[8] = k
    assert oracle.bdr_GetLBP1(d, k) == 5
    # drv[3]=1, drv[7]=k-1 -> 7
    d = np.full(L, S)
    d[2] = 1
    d[6] = k - 1
    assert oracle.bdr_GetLBP1(d, k) == 7


@pytest.mark.parametrize("k", [1, 2, 4, 8, 60, 300])
def test_sliding_correctness_single_bdr(k):
    """Every variant's Alg.2 readout at every boundary equals the brute-force
    max rank over the last k slices (zero tolerance), on
    random per-slice rank streams (with empty slices)."""
    rng = np.random.default_rng(k)
    zb = max(1, int(np.ceil(np.log2(k + 1))))
    zb_small = zb + (1 if (1 << zb) - 2 < k else 0)
    for L in (3, 9, 27):
        for trial in range(6):
            n_slices = 3 * k + 20
            stream = []
            for _ in range(n_slices):
                cnt = rng.integers(0, 4)
                stream.append(rng.integers(1, L + 1, size=cnt).tolist())
            S = (1 << zb) - 1
            ser = np.full(L, S)
            gf = np.full(L, S)
            gs = np.full(L, (1 << zb_small) - 1)
            for t, ranks in enumerate(stream):
                gs = oracle.bdr_begin_slice_gsmall(gs, zb_small)
                now, bs = 0, 0
                for r in ranks:
                    now = max(now, r)
                    bs |= 1 << (r - 1)
                    gs[r - 1] = 0
                ser = oracle.bdr_end_slice_serial(ser, zb, now)
                gf = oracle.bdr_end_slice_gfast(gf, zb, bs)
                window = [r for s in stream[max(0, t - k + 1):t + 1] for r in s]
                want = max(window) if window else 0
                assert oracle.bdr_GetLBP1(ser, k) == want
                assert oracle.bdr_GetLBP1(gf, k) == want
                assert oracle.bdr_GetLBP1(gs, k) == want


def test_expiry_exactly_k():
    """A rank recorded only in slice t is active at boundaries t..t+k-1 and
    inactive from t+k on."""
    for k in (1, 3, 5, 10):
        zb = int(np.ceil(np.log2(k + 1)))
        d = np.full(8, (1 << zb) - 1)
        d = oracle.bdr_end_slice_serial(d, zb, 6)  # boundary t = 0
        for t in range(0, 3 * k):
            assert (oracle.bdr_GetLBP1(d, k) == 6) == (t < k), (k, t)
            d = oracle.bdr_end_slice_serial(d, zb, 0)


def test_table1_memory_bits():
    # b=8, k=15 -> gsmall 96, gfast 120, serial 101
    assert oracle.memory_bits("gsmall", 8, 15) == 96
    assert oracle.memory_bits("gfast", 8, 15) == 120
    assert oracle.memory_bits("serial", 8, 15) == 101
    # BASELINE.md Table 1 instantiations (tiny, caida, 10G, bigwin)
    for b, k, want in ((5, 4, (86, 108, 81)), (7, 5, (80, 100, 75)), (8, 10, (101, 120, 96)),
                       (8, 60, (149, 168, 144))):
        got = tuple(oracle.memory_bits(v, b, k) for v in ("serial", "gfast", "gsmall"))
        assert got == want


def test_lfpm_spec_vectors():
    # SPEC.md:393-401
    l = oracle.LFPM()
    l.insert(0, 3)
    l.insert(0, 5)
    assert len(l) == 1 and l.query(0, 4) == 5          # dominated cell removed
    l2 = oracle.LFPM()
    l2.insert(0, 5)
    l2.insert(0, 3)
    assert len(l2) == 2
    assert oracle.LFPM().query(10, 4) == 0              # empty list
    l3 = oracle.LFPM()
    l3.insert(2, 7)
    assert l3.query(4, 4) == 7 and l3.query(6, 4) == 0  # inside, then expired


@pytest.mark.parametrize("k", [1, 3, 8, 60])
def test_bdr_equals_lfpm_windowed_max(k):
    """SPEC.md:412, acceptance 2: the BDR (Alg.1 + Alg.2) and the
    prior-art LFPM give the same windowed maximum at every boundary, for random
    rank streams -- the paper's claim that BDR replaces LFPM."""
    rng = np.random.default_rng(100 + k)
    zb = max(1, int(np.ceil(np.log2(k + 1))))
    for L in (5, 24):
        for trial in range(10):
            d = np.full(L, (1 << zb) - 1)
            l = oracle.LFPM()
            for t in range(4 * k + 30):
                ranks = rng.integers(1, L + 1, size=int(rng.integers(0, 5))).tolist()
                for r in ranks:
                    l.insert(t, r)
                d = oracle.bdr_end_slice_serial(d, zb, max(ranks) if ranks else 0)
                assert oracle.bdr_GetLBP1(d, k) == l.query(t, k)


def test_lfpm_length_is_logarithmic():
    """SPEC.md:395 / acceptance 9: with i.i.d. geometric ranks the LFPM holds
    about ln(n) cells after n inserts (within a factor of 2), against the BDR's
    fixed L * zb bits (PAPER.md:76 vs Table 1)."""
    rng = np.random.default_rng(9)
    for n in (100, 1000, 10000):
        lens = []
        for _ in range(30):
            l = oracle.LFPM()
            # a fresh slice per insert (worst case for LFPM); rank ~ Geometric(1/2)
            ranks = np.minimum(rng.geometric(0.5, size=n), 24)
            for i, r in enumerate(ranks):
                l.insert(i, int(r))
            lens.append(len(l))
        assert 0.5 * np.log(n) <= np.mean(lens) <= 2 * np.log(n), (n, np.mean(lens))
