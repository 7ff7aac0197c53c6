"""Pins for the oracle's hashing and indexing layer."""
import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _rotl(x, r):
    return ((x << r) | (x >> (32 - r))) & 0xFFFFFFFF


def _murmur3_x86_32(key: bytes, seed: int) -> int:
    """Published MurmurHash3_x86_32 body for keys of 0 or 4 bytes; the final
    mix is the ORACLE's fmix32, so the published vectors pin it."""
    h = seed
    if key:
        k1 = int.from_bytes(key, "little")
        k1 = (k1 * 0xCC9E2D51) & 0xFFFFFFFF
        k1 = _rotl(k1, 15)
        k1 = (k1 * 0x1B873593) & 0xFFFFFFFF
        h ^= k1
        h = _rotl(h, 13)
        h = (h * 5 + 0xE6546B64) & 0xFFFFFFFF
    h ^= len(key)
    return oracle.fmix32(h)


def test_fmix32_matches_published_murmur3_vectors():
    n = 0
    for line in open(os.path.join(GOLD, "murmur3_x86_32.txt")):
        if line.startswith("#") or not line.strip():
            continue
        key, seed, want = line.split()
        kb = b"" if key == "-" else bytes.fromhex(key)
        assert _murmur3_x86_32(kb, int(seed, 16)) == int(want, 16), line
        n += 1
    assert n == 6


def test_H_modulus_one_and_identity():
    # h(x,1,a) = 0; N = 2^32 keeps the whole word (R#6)
    for x in (0, 1, 0xDEADBEEF, 0xFFFFFFFF):
        assert oracle.H(x, 1, 0x1234) == 0
        assert oracle.H(x, 1 << 32, 0x5EED0001) == oracle.fmix32(x ^ 0x5EED0001)
    # power-of-two N keeps the LOW bits (R#6)
    assert oracle.H(77, 1 << 12, 5) == oracle.fmix32(77 ^ 5) & 0xFFF


def test_H_avalanche():
    # flipping one input bit flips ~16 of 32 output bits (12-20)
    rng = np.random.default_rng(7)
    flips = []
    for x in rng.integers(0, 1 << 32, size=400, dtype=np.uint64):
        x = int(x)
        h0 = oracle.H(x, 1 << 32, 0x5EED0002)
        for bit in range(0, 32, 3):
            flips.append(bin(h0 ^ oracle.H(x ^ (1 << bit), 1 << 32, 0x5EED0002)).count("1"))
    assert 12 <= np.mean(flips) <= 20


def test_LB_vectors():
    # SPEC.md:177-179
    assert oracle.LB(0xFFFFFFFF, 4) == 15
    assert oracle.LB(0x80000000, 1) == 1
    assert oracle.LB(0x12345678, 8) == 0x12
    assert oracle.LB(0x12345678, 0) == 0


def test_LBP1_vectors_and_bruteforce():
    # SPEC.md:56-58
    assert oracle.LBP1(0x80000000, 32) == 1
    assert oracle.LBP1(0x00100000, 32) == 12
    assert oracle.LBP1(0, 24) == 24
    # R#4/R#5: 1-based from the MSB, saturating at w -- checked against the
    # integer bit length, an expression independent of the oracle's loop
    rng = np.random.default_rng(3)
    for v in list(rng.integers(0, 1 << 32, size=2000, dtype=np.uint64)) + [1, 2, 3, 1 << 31]:
        v = int(v)
        for w in (1, 5, 20, 27, 31, 32):
            want = 33 - v.bit_length() if v else 33
            assert oracle.LBP1(v, w) == min(want, w)


def test_getPhyIdx_appendix_anchor_and_uniformity():
    # SURVEY Appendix A regression anchor (computed from R#6, not the paper)
    assert oracle.pair_index(0xC0A80001, 0x08080808, 5, 27, 0x5EED0001, 0x5EED0002,
                             1 << 12) == (587, 2)
    # chi-square uniformity of the physical index over [0, m)
    m = 64
    counts = np.zeros(m)
    rng = np.random.default_rng(11)
    aips = rng.integers(0, 1 << 32, size=20000, dtype=np.uint64)
    for a in aips:
        counts[oracle.getPhyIdx(int(a), int(a) % 32, 0x5EED0001, m)] += 1
    exp = len(aips) / m
    chi2 = ((counts - exp) ** 2 / exp).sum()
    assert chi2 < 120  # df = 63, p ~ 1e-5


def test_getPhyIdx_birthday_collisions():
    # two hosts' g=512 virtual vectors in m=2^16 share ~g^2/m = 4 slots
    g, m = 512, 1 << 16
    rng = np.random.default_rng(5)
    shared = []
    for _ in range(60):
        a, b = (int(x) for x in rng.integers(0, 1 << 32, size=2, dtype=np.uint64))
        sa = {oracle.getPhyIdx(a, i, 0x5EED0001, m) for i in range(g)}
        sb = {oracle.getPhyIdx(b, i, 0x5EED0001, m) for i in range(g)}
        shared.append(len(sa & sb))
    assert 2.0 <= np.mean(shared) <= 6.0
