"""ctypes wrapper around the plain-C VBDR oracle (``oracle/vbdr_oracle.c``).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product path (``paper_1810_13132_b200``) never imports it, and it
imports nothing from the product path.

Every function here is argument marshalling around the C oracle, except
:func:`exact_cardinality`, which is Definition 1 of the paper (PAPER.md:146-149,
"the number of hosts in BN that send packets to or receive packets from it ...
in W(t,k)") written with Python sets.

Parity pins and their status are listed in the C file header and in DESIGN.md
section 4.  Per-host estimates on a shared, skewed pool are "parity unpinned"
against the paper (the paper has no experiments); only the formula pieces are
pinned (closed forms, textbook HyperLogLog special case).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "vbdr_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

SERIAL, GFAST, GSMALL = 0, 1, 2
VARIANTS = {"serial": SERIAL, "gfast": GFAST, "gsmall": GSMALL}


def build(force: bool = False) -> str:
    """Compile the oracle with gcc: -O2, no FMA contraction (R#17)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-Wall",
             "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _declare(_lib)
    return _lib


u8p = C.POINTER(C.c_uint8)
u16p = C.POINTER(C.c_uint16)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
f64p = C.POINTER(C.c_double)


def _declare(L):
    sig = {
        "orc_fmix32": (C.c_uint32, [C.c_uint32]),
        "orc_H": (C.c_uint64, [C.c_uint32, C.c_uint64, C.c_uint32]),
        "orc_LB": (C.c_uint32, [C.c_uint32, C.c_uint32]),
        "orc_LBP1": (C.c_uint32, [C.c_uint32, C.c_uint32]),
        "orc_getPhyIdx": (C.c_uint64, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64]),
        "orc_pair_index": (None, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                  C.c_uint32, C.c_uint64, u64p, u32p]),
        "orc_InitDR": (None, [u16p, C.c_uint32]),
        "orc_SetDR": (None, [u16p]),
        "orc_SlideDR": (None, [u16p, C.c_uint32]),
        "orc_IsActiveDR": (C.c_int, [C.c_uint16, C.c_uint32]),
        "orc_bdr_end_slice_serial": (None, [u16p, C.c_uint32, C.c_uint32, C.c_uint32]),
        "orc_bdr_end_slice_gfast": (None, [u16p, C.c_uint32, C.c_uint32, C.c_uint32]),
        "orc_bdr_begin_slice_gsmall": (None, [u16p, C.c_uint32, C.c_uint32]),
        "orc_bdr_GetLBP1": (C.c_uint32, [u16p, C.c_uint32, C.c_uint32]),
        "orc_pool_new": (C.c_void_p, [C.c_int, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                      C.c_uint64, C.c_uint32, C.c_uint32]),
        "orc_pool_free": (None, [C.c_void_p]),
        "orc_begin_slice": (None, [C.c_void_p]),
        "orc_scan": (None, [C.c_void_p, u32p, C.c_uint64]),
        "orc_end_slice": (None, [C.c_void_p]),
        "orc_readout": (None, [C.c_void_p, u8p]),
        "orc_export_drv": (None, [C.c_void_p, u16p]),
        "orc_import_drv": (None, [C.c_void_p, u16p]),
        "orc_export_now": (None, [C.c_void_p, u8p]),
        "orc_getSumLBP1": (C.c_uint64, [C.c_void_p, u8p, C.c_uint32]),
        "orc_gather": (None, [C.c_void_p, u8p, C.c_uint32, u8p]),
        "orc_alpha": (C.c_double, [C.c_uint64]),
        "orc_hll_sums": (None, [u8p, C.c_uint64, f64p, u64p]),
        "orc_hll_from_sums": (C.c_double, [C.c_uint64, C.c_double, C.c_uint64]),
        "orc_hll_raw": (C.c_double, [u8p, C.c_uint64]),
        "orc_vhll": (C.c_double, [C.c_uint64, C.c_uint32, C.c_double, C.c_double]),
        "orc_estimate": (None, [C.c_void_p, u8p, u32p, C.c_uint64, f64p]),
        "orc_host_sums": (None, [C.c_void_p, u8p, u32p, C.c_uint64, f64p, u64p]),
        "orc_rebuild": (None, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64,
                               u32p, C.c_uint64, u8p]),
        "orc_memory_bits": (C.c_uint64, [C.c_int, C.c_uint32, C.c_uint32]),
        "orc_estimate_M": (None, [C.c_uint32, C.c_uint32, C.c_uint64, u8p, u32p, C.c_uint64, f64p]),
        "orc_bdr_pcsa_R": (C.c_uint32, [u16p, C.c_uint32, C.c_uint32]),
        "orc_lfpm_new": (C.c_void_p, []),
        "orc_lfpm_free": (None, [C.c_void_p]),
        "orc_lfpm_insert": (None, [C.c_void_p, C.c_uint64, C.c_uint32]),
        "orc_lfpm_query": (C.c_uint32, [C.c_void_p, C.c_uint64, C.c_uint32]),
        "orc_lfpm_len": (C.c_uint32, [C.c_void_p]),
        "orc_readout_pcsa": (None, [C.c_void_p, u8p]),
        "orc_loglog_alpha": (C.c_double, [C.c_uint64]),
        "orc_loglog_raw": (C.c_double, [u8p, C.c_uint64]),
        "orc_pcsa_raw": (C.c_double, [u8p, C.c_uint64]),
        "orc_estimate_variant": (None, [C.c_uint32, C.c_uint32, C.c_uint64, u8p, u32p, C.c_uint64,
                                        C.c_int, f64p]),
        "orc_host_sums_M": (None, [C.c_uint32, C.c_uint32, C.c_uint64, u8p, u32p, C.c_uint64,
                                   f64p, u64p]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args


def _ptr(a: np.ndarray, t):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(t)


# ---------------------------------------------------------------- scalars
def fmix32(x: int) -> int:
    return lib().orc_fmix32(x & 0xFFFFFFFF)


def H(x: int, N: int, A: int) -> int:
    return lib().orc_H(x & 0xFFFFFFFF, N, A & 0xFFFFFFFF)


def LB(x: int, i: int) -> int:
    return lib().orc_LB(x & 0xFFFFFFFF, i)


def LBP1(v: int, w: int) -> int:
    return lib().orc_LBP1(v & 0xFFFFFFFF, w)


def getPhyIdx(aip: int, i: int, A0: int, z: int) -> int:
    return lib().orc_getPhyIdx(aip & 0xFFFFFFFF, i, A0 & 0xFFFFFFFF, z)


def pair_index(aip, bip, b, L, A0, A1, z):
    p = C.c_uint64()
    r = C.c_uint32()
    lib().orc_pair_index(aip, bip, b, L, A0, A1, z, C.byref(p), C.byref(r))
    return p.value, r.value


def alpha(s: int) -> float:
    return lib().orc_alpha(s)


def hll_raw(M: np.ndarray) -> float:
    M = np.ascontiguousarray(M, dtype=np.uint8)
    return lib().orc_hll_raw(_ptr(M, u8p), M.size)


def hll_sums(M: np.ndarray):
    M = np.ascontiguousarray(M, dtype=np.uint8)
    Z = C.c_double()
    V = C.c_uint64()
    lib().orc_hll_sums(_ptr(M, u8p), M.size, C.byref(Z), C.byref(V))
    return Z.value, V.value


def vhll(z: int, g: int, E_s: float, E_tot: float) -> float:
    return lib().orc_vhll(z, g, E_s, E_tot)


def memory_bits(variant: str, b: int, k: int) -> int:
    return lib().orc_memory_bits(VARIANTS[variant], b, k)


def rebuild(pairs: np.ndarray, b, L, z, A0, A1) -> np.ndarray:
    pairs = np.ascontiguousarray(pairs, dtype=np.uint32).reshape(-1)
    out = np.zeros(z, dtype=np.uint8)
    lib().orc_rebuild(b, L, A0, A1, z, _ptr(pairs, u32p), pairs.size // 2, _ptr(out, u8p))
    return out


def estimate_M(M: np.ndarray, hosts: np.ndarray, b: int, z: int, A0: int = 0x5EED0001):
    """Per-host estimates from a register array (e.g. a rebuild), no pool."""
    M = np.ascontiguousarray(M, dtype=np.uint8)
    hosts = np.ascontiguousarray(hosts, dtype=np.uint32)
    out = np.empty(hosts.size, dtype=np.float64)
    lib().orc_estimate_M(b, A0, z, _ptr(M, u8p), _ptr(hosts, u32p), hosts.size, _ptr(out, f64p))
    return out


ESTIMATORS = {"hll": 0, "loglog": 1, "pcsa": 2}


class LFPM:
    """The prior-art list of future possible maxima."""

    def __init__(self):
        self._h = lib().orc_lfpm_new()

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_lfpm_free(self._h)
            self._h = None

    def insert(self, slice_: int, rank: int):
        lib().orc_lfpm_insert(self._h, slice_, rank)

    def query(self, t: int, k: int) -> int:
        return lib().orc_lfpm_query(self._h, t, k)

    def __len__(self):
        return lib().orc_lfpm_len(self._h)


def loglog_alpha(m: int) -> float:
    return lib().orc_loglog_alpha(m)


def loglog_raw(M: np.ndarray) -> float:
    M = np.ascontiguousarray(M, dtype=np.uint8)
    return lib().orc_loglog_raw(_ptr(M, u8p), M.size)


def pcsa_raw(R: np.ndarray) -> float:
    R = np.ascontiguousarray(R, dtype=np.uint8)
    return lib().orc_pcsa_raw(_ptr(R, u8p), R.size)


def bdr_pcsa_R(drv: np.ndarray, k: int) -> int:
    d = np.ascontiguousarray(drv, dtype=np.uint16)
    return lib().orc_bdr_pcsa_R(_ptr(d, u16p), d.size, k)


def estimate_variant(V: np.ndarray, hosts: np.ndarray, b: int, z: int, estimator: str,
                     A0: int = 0x5EED0001) -> np.ndarray:
    """Per-host estimates with register values V under 'hll', 'loglog' (V = M)
    or 'pcsa' (V = R), noise-subtracted as vHLL (R#15)."""
    V = np.ascontiguousarray(V, dtype=np.uint8)
    hosts = np.ascontiguousarray(hosts, dtype=np.uint32)
    out = np.empty(hosts.size, dtype=np.float64)
    lib().orc_estimate_variant(b, A0, z, _ptr(V, u8p), _ptr(hosts, u32p), hosts.size,
                               ESTIMATORS[estimator], _ptr(out, f64p))
    return out


def host_sums_M(M: np.ndarray, hosts: np.ndarray, b: int, z: int, A0: int = 0x5EED0001):
    M = np.ascontiguousarray(M, dtype=np.uint8)
    hosts = np.ascontiguousarray(hosts, dtype=np.uint32)
    Z = np.empty(hosts.size, dtype=np.float64)
    V = np.empty(hosts.size, dtype=np.uint64)
    lib().orc_host_sums_M(b, A0, z, _ptr(M, u8p), _ptr(hosts, u32p), hosts.size, _ptr(Z, f64p),
                          _ptr(V, u64p))
    return Z, V


# --------------------------------------------------------- single-BDR ops
def bdr_end_slice_serial(drv: np.ndarray, zb: int, now: int) -> np.ndarray:
    d = np.ascontiguousarray(drv, dtype=np.uint16).copy()
    lib().orc_bdr_end_slice_serial(_ptr(d, u16p), d.size, zb, now)
    return d


def bdr_end_slice_gfast(drv: np.ndarray, zb: int, bs: int) -> np.ndarray:
    d = np.ascontiguousarray(drv, dtype=np.uint16).copy()
    lib().orc_bdr_end_slice_gfast(_ptr(d, u16p), d.size, zb, bs)
    return d


def bdr_begin_slice_gsmall(drv: np.ndarray, zb: int) -> np.ndarray:
    d = np.ascontiguousarray(drv, dtype=np.uint16).copy()
    lib().orc_bdr_begin_slice_gsmall(_ptr(d, u16p), d.size, zb)
    return d


def bdr_GetLBP1(drv: np.ndarray, k: int) -> int:
    d = np.ascontiguousarray(drv, dtype=np.uint16)
    return lib().orc_bdr_GetLBP1(_ptr(d, u16p), d.size, k)


# ------------------------------------------------------------------- pool
@dataclass
class PoolConfig:
    """The paper's problem statement: g = 2^b virtual BDRs per host
    (PAPER.md:152), window k, pool size z,
    seeds A0/A1 (defaults R#7), DR width zb,
    rank range L (R#3)."""
    b: int
    k: int
    z: int
    A0: int = 0x5EED0001
    A1: int = 0x5EED0002
    zb: int = 0
    L: int = 0

    def __post_init__(self):
        if self.zb == 0:
            zb = 0
            while (1 << zb) < self.k + 1:
                zb += 1
            self.zb = max(zb, 1)
        if self.L == 0:
            self.L = 32 - self.b

    @property
    def g(self) -> int:
        return 1 << self.b


class Pool:
    """One BDR pool BDRP in one of the paper's three variants (Table 1 rows):
    'serial' (Alg.4 + Alg.1), 'gfast' (Alg.7 + Alg.6), 'gsmall' (Alg.9 + Alg.8).

    Slice protocol (R#13): begin_slice(); scan(...) any number of times;
    end_slice().  After end_slice() the pool is at boundary t and readout()
    gives the windowed registers M of W(t-k+1..t)."""

    def __init__(self, cfg: PoolConfig, variant: str):
        self.cfg = cfg
        self.variant = variant
        self._h = lib().orc_pool_new(VARIANTS[variant], cfg.b, cfg.L, cfg.k, cfg.zb, cfg.z,
                                     cfg.A0, cfg.A1)
        if not self._h:
            raise ValueError(f"invalid oracle pool config {cfg}")

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().orc_pool_free(h)
            self._h = None

    def begin_slice(self):
        lib().orc_begin_slice(self._h)

    def scan(self, pairs: np.ndarray):
        p = np.ascontiguousarray(pairs, dtype=np.uint32).reshape(-1)
        lib().orc_scan(self._h, _ptr(p, u32p), p.size // 2)

    def end_slice(self):
        lib().orc_end_slice(self._h)

    def slice(self, pairs: np.ndarray):
        """One whole slice: open, scan, close."""
        self.begin_slice()
        self.scan(pairs)
        self.end_slice()

    def readout(self) -> np.ndarray:
        M = np.empty(self.cfg.z, dtype=np.uint8)
        lib().orc_readout(self._h, _ptr(M, u8p))
        return M

    def drv(self) -> np.ndarray:
        """Raw DR values, shape (z, L); column r-1 is rank r."""
        out = np.empty(self.cfg.z * self.cfg.L, dtype=np.uint16)
        lib().orc_export_drv(self._h, _ptr(out, u16p))
        return out.reshape(self.cfg.z, self.cfg.L)

    def set_drv(self, drv: np.ndarray):
        d = np.ascontiguousarray(drv, dtype=np.uint16).reshape(-1)
        assert d.size == self.cfg.z * self.cfg.L
        lib().orc_import_drv(self._h, _ptr(d, u16p))

    def now(self) -> np.ndarray:
        out = np.empty(self.cfg.z, dtype=np.uint8)
        lib().orc_export_now(self._h, _ptr(out, u8p))
        return out

    def readout_pcsa(self) -> np.ndarray:
        """PCSA registers R[j] (meaningful for the gsmall variant, which records
        every rank: the sliding bitmap)."""
        R = np.empty(self.cfg.z, dtype=np.uint8)
        lib().orc_readout_pcsa(self._h, _ptr(R, u8p))
        return R

    def ck(self) -> np.ndarray:
        """Canonical state C_k[j][r] = min(DR, k)."""
        return np.minimum(self.drv(), self.cfg.k).astype(np.uint16)

    def gather(self, M: np.ndarray, aip: int) -> np.ndarray:
        M = np.ascontiguousarray(M, dtype=np.uint8)
        out = np.empty(self.cfg.g, dtype=np.uint8)
        lib().orc_gather(self._h, _ptr(M, u8p), aip, _ptr(out, u8p))
        return out

    def sum_lbp1(self, M: np.ndarray, aip: int) -> int:
        M = np.ascontiguousarray(M, dtype=np.uint8)
        return lib().orc_getSumLBP1(self._h, _ptr(M, u8p), aip)

    def estimate(self, M: np.ndarray, hosts: np.ndarray) -> np.ndarray:
        M = np.ascontiguousarray(M, dtype=np.uint8)
        hosts = np.ascontiguousarray(hosts, dtype=np.uint32)
        out = np.empty(hosts.size, dtype=np.float64)
        lib().orc_estimate(self._h, _ptr(M, u8p), _ptr(hosts, u32p), hosts.size,
                           _ptr(out, f64p))
        return out

    def host_sums(self, M: np.ndarray, hosts: np.ndarray):
        M = np.ascontiguousarray(M, dtype=np.uint8)
        hosts = np.ascontiguousarray(hosts, dtype=np.uint32)
        Z = np.empty(hosts.size, dtype=np.float64)
        V = np.empty(hosts.size, dtype=np.uint64)
        lib().orc_host_sums(self._h, _ptr(M, u8p), _ptr(hosts, u32p), hosts.size,
                            _ptr(Z, f64p), _ptr(V, u64p))
        return Z, V


def exact_cardinality(window_slices, aip: int) -> int:
    """Definition 1: |OP(aip, t, k)| = number of distinct
    bip paired with aip in the window's slices."""
    seen = set()
    for pairs in window_slices:
        p = np.asarray(pairs, dtype=np.uint32).reshape(-1, 2)
        for a, b in p[p[:, 0] == aip]:
            seen.add(int(b))
    return len(seen)


def exact_cardinalities(window_slices) -> dict:
    """Definition 1 for every aip present in the window."""
    allp = np.concatenate([np.asarray(s, dtype=np.uint32).reshape(-1, 2) for s in window_slices])
    key = (allp[:, 0].astype(np.uint64) << np.uint64(32)) | allp[:, 1].astype(np.uint64)
    uniq = np.unique(key)
    aips, counts = np.unique((uniq >> np.uint64(32)).astype(np.uint32), return_counts=True)
    return dict(zip(aips.tolist(), counts.tolist()))
