"""Seeded synthetic IP-pair traces -- shared input generator.

This module is the ONLY code the oracle side (``oracle/``, ``tests/``) and the
CUDA side (``paper_1810_13132_b200``, ``bench.py``) have in common.  It holds
none of the method's arithmetic: no H / fmix32, no rank, no register index.
Its mixers (splitmix64, lowbias32) are different functions from the paper's
hash H (R#6), chosen so a generator bug cannot mask a hashing bug.

Trace model ("input recipe"; CAIDA traces are not
available offline).  Pair ``i`` of slice ``t`` under ``seed``:

    x    = sm64(sm64(seed ^ (t << 32)) ^ i)              counter-based RNG
    u    = (x >> 11) * 2^-53                             exact in fp64
    h    = first index with cdf[h] > u                   Zipf(s) host rank
    aip  = lowbias32(h ^ 0xA5A5A5A5)                     bijection: H distinct hosts
    y    = sm64(x)
    v    = 2^31 | (y & 0x7FFFFFFF)       if (y >> 56) < churn   (fresh peer)
           (y & 0xFFFFFFFF) mod U[h]     otherwise              (persistent universe)
    bip  = lowbias32(((h * 0x9E3779B1 + v) mod 2^32) ^ 0x3C3C3C3C)

Bursty variant (``burst`` > 0, SURVEY.md section 8 d.3 "packet trains"):
position ``j`` continues the train of ``j - 1`` when bit 63 of
``sm64(x_j ^ 0xD1B54A32D192ED03)`` is set (probability 1/2), for at most
``burst - 1`` steps back; pair ``i`` is then the i.i.d. pair of the train's
first position, so trains have length 1 + Geom(1/2) (capped at ``burst``)
and any range of positions can still be generated independently.

``cdf`` (fp64, Zipf weights (h+1)^-s, last entry forced to 1.0) and ``U``
(u32 universe sizes max(1, floor(U0 (h+1)^-s))) are tables built once here with
numpy and handed to both the numpy twin and the CUDA kernel
(``synth/synth_gen.cu``), so the two produce the same bytes.

Pairs are ``uint32[Np, 2]`` rows ``(aip, bip)`` in host-order IPv4 (R#21).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
M32 = np.uint64(0xFFFFFFFF)


def sm64(x: np.ndarray) -> np.ndarray:
    """splitmix64 output function on uint64 arrays (wrapping arithmetic)."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def lowbias32(x: np.ndarray) -> np.ndarray:
    """A 32-bit bijection (xorshift-multiply), as uint64 arrays holding u32."""
    x = np.asarray(x, dtype=np.uint64) & M32
    with np.errstate(over="ignore"):
        x ^= x >> np.uint64(16)
        x = (x * np.uint64(0x7FEB352D)) & M32
        x ^= x >> np.uint64(15)
        x = (x * np.uint64(0x846CA68B)) & M32
        x ^= x >> np.uint64(16)
    return x


@dataclass
class TraceConfig:
    """One synthetic workload (BASELINE.json configs)."""
    name: str
    hosts: int            # H monitored hosts (aip side)
    pairs_per_slice: int  # Np
    U0: int               # universe scale of the largest host
    zipf_s: float = 1.1
    churn: int = 64       # fresh-peer threshold on y >> 56 (64/256 = 25 %)
    seed: int = 1
    burst: int = 0        # > 0: packet trains of 1 + Geom(1/2) copies, at most `burst`
    _tables: tuple = field(default=None, init=False, repr=False, compare=False)

    def tables(self):
        """(cdf float64[H], U uint32[H]) -- built once, shared by both sides."""
        if self._tables is None:
            r = np.arange(1, self.hosts + 1, dtype=np.float64)
            w = r ** (-self.zipf_s)
            c = np.cumsum(w)
            cdf = c / c[-1]
            cdf[-1] = 1.0
            U = np.maximum(1.0, np.floor(self.U0 * w)).astype(np.uint32)
            self._tables = (np.ascontiguousarray(cdf), np.ascontiguousarray(U))
        return self._tables

    def host_ids(self) -> np.ndarray:
        """aip of every host rank h = 0..H-1 (distinct: lowbias32 is a bijection)."""
        h = np.arange(self.hosts, dtype=np.uint64)
        return lowbias32(h ^ np.uint64(0xA5A5A5A5)).astype(np.uint32)


def generate(cfg: TraceConfig, t: int, start: int = 0, count: int | None = None) -> np.ndarray:
    """Pairs ``start .. start+count-1`` of slice ``t`` as uint32[count, 2] (numpy twin)."""
    if count is None:
        count = cfg.pairs_per_slice - start
    cdf, U = cfg.tables()
    i = np.arange(start, start + count, dtype=np.uint64)
    base = sm64(np.uint64(cfg.seed) ^ (np.uint64(t) << np.uint64(32)))
    if cfg.burst > 0:  # walk back to the first position of the train
        src = i.copy()
        live = np.ones(count, dtype=bool)
        for _ in range(cfg.burst - 1):
            cont = (sm64(sm64(base ^ src) ^ np.uint64(0xD1B54A32D192ED03)) >> np.uint64(63)) == 1
            step = live & cont & (src > 0)
            src = np.where(step, src - np.uint64(1), src)
            live = step
        i = src
    x = sm64(base ^ i)
    u = (x >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    h = np.searchsorted(cdf, u, side="right").astype(np.uint64)
    aip = lowbias32(h ^ np.uint64(0xA5A5A5A5))
    y = sm64(x)
    fresh = (y >> np.uint64(56)) < np.uint64(cfg.churn)
    v_fresh = np.uint64(0x80000000) | (y & np.uint64(0x7FFFFFFF))
    v_keep = (y & M32) % U[h.astype(np.int64)].astype(np.uint64)
    v = np.where(fresh, v_fresh, v_keep)
    with np.errstate(over="ignore"):
        mixed = ((h * np.uint64(0x9E3779B1) + v) & M32) ^ np.uint64(0x3C3C3C3C)
    bip = lowbias32(mixed)
    out = np.empty((count, 2), dtype=np.uint32)
    out[:, 0] = aip.astype(np.uint32)
    out[:, 1] = bip.astype(np.uint32)
    return out


# The BASELINE.json workloads.  'bigwin' H is our choice.
CONFIGS = {
    "tiny": TraceConfig("tiny", hosts=64, pairs_per_slice=10_000, U0=4000),
    "caida": TraceConfig("caida", hosts=500_000, pairs_per_slice=5_000_000, U0=1 << 20),
    # caida with packet trains (SURVEY.md 8 d.3 bursty variant), for the scan modes
    "caida_bursty": TraceConfig("caida_bursty", hosts=500_000, pairs_per_slice=5_000_000,
                                U0=1 << 20, burst=16),
    "10G": TraceConfig("10G", hosts=4_000_000, pairs_per_slice=100_000_000, U0=1 << 22),
    "bigwin": TraceConfig("bigwin", hosts=1 << 24, pairs_per_slice=16_666_667, U0=1 << 22),
}


# ------------------------------------------------------------ CUDA twin
_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libsynth.so")
_cuda = None


def _cuda_lib():
    global _cuda
    if _cuda is None:
        if not os.path.exists(_SO):
            raise RuntimeError(f"{_SO} missing: run __graft_entry__.build()")
        _cuda = C.CDLL(_SO)
        _cuda.synth_generate.restype = C.c_int
        _cuda.synth_generate.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64,
                                         C.c_uint64, C.c_void_p, C.c_void_p, C.c_uint32,
                                         C.c_uint32, C.c_uint32, C.c_void_p]
    return _cuda


class DeviceTrace:
    """Generates slices directly into HBM with the CUDA twin (bench inputs)."""

    def __init__(self, cfg: TraceConfig, device):
        import torch
        self.cfg = cfg
        cdf, U = cfg.tables()
        self.cdf = torch.from_numpy(cdf).to(device)
        self.U = torch.from_numpy(U.astype(np.int32)).to(device)
        self.device = device

    def generate_into(self, out, t: int, start: int = 0, stream=None):
        """Fill ``out`` (int32/uint32 tensor, 2*count elements) with pairs start.. of slice t."""
        import torch
        count = out.numel() // 2
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        rc = _cuda_lib().synth_generate(out.data_ptr(), count, self.cfg.seed, t, start,
                                        self.cdf.data_ptr(), self.U.data_ptr(), self.cfg.hosts,
                                        self.cfg.churn, self.cfg.burst, C.c_void_p(s.cuda_stream))
        if rc != 0:
            raise RuntimeError(f"synth_generate failed: {rc}")
        return out

    def generate(self, t: int, start: int = 0, count: int | None = None):
        import torch
        if count is None:
            count = self.cfg.pairs_per_slice - start
        out = torch.empty(2 * count, dtype=torch.int32, device=self.device)
        return self.generate_into(out, t, start)
