#!/usr/bin/env python
"""The scan's memory-path ceiling on the bench's own update stream (round 2).

For a workload (caida, 10G, bigwin) this builds the slice's IP pairs with the
bench's generator, hashes them to (register index j, stamp value (T << 5) | rho)
records in torch (Alg.4 lines 180-184 restated here: bip' = fmix32(bip ^ A1),
vidx = top b bits, rho = min(clz(bip' << b) + 1, L), j = fmix32(aip ^
fmix32(vidx ^ A0)) & (z - 1) -- tooling only, the product and the oracle keep
their own), and times tools/ubench_scanpath.cu streaming them through the
scan's global-memory path (check load + atomicMax; or atomicMax only), the
stamp array reset before and L2 flushed before every run (as bench.py).  Prints
one JSON object; `--write` merges it into profiles/ceilings_b200.json under
"scan_path_Gpairs_s", which bench.py uses as the scan's roofline peak.

usage: python tools/scan_ceiling.py [--configs caida,10G,bigwin] [--write]"""
import argparse
import ctypes
import json
import os
import subprocess
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402

WL = {"caida": (128, 1 << 22), "10G": (256, 1 << 26), "bigwin": (256, 1 << 28)}
K = {"caida": 5, "10G": 10, "bigwin": 60}
A0, A1 = 0x5EED0001, 0x5EED0002
M32 = 0xFFFFFFFF


def fmix32(t):
    t = t ^ (t >> 16)
    t = (t * 0x85EBCA6B) & M32
    t = t ^ (t >> 13)
    t = (t * 0xC2B2AE35) & M32
    return t ^ (t >> 16)


def clz32(x):
    """Leading zeros of 32-bit values held in int64 (x = 0 -> 32)."""
    n = torch.zeros_like(x)
    for s in (16, 8, 4, 2, 1):
        hi = (x >> (32 - s)) == 0
        n = n + torch.where(hi, s, 0)
        x = torch.where(hi, (x << s) & M32, x)
    return n + (x == 0).to(n.dtype)


def packed_zb(k: int) -> int:
    """Layout P's DR width: ceil(log2(k+1)), one more when 2^zb - 2 < k (vbdr.h zbits)."""
    zb = max(1, k.bit_length())
    return zb + 1 if (1 << zb) - 2 < k else zb


def records(name: str, dev, T: int = 7, packed: bool = False, stamps: bool = False):
    m, z = WL[name]
    b = m.bit_length() - 1
    L = 32 - b
    tr = synth.CONFIGS[name]
    buf = torch.empty(2 * tr.pairs_per_slice, dtype=torch.int32, device=dev)
    synth.DeviceTrace(tr, dev).generate_into(buf, T)
    p = buf.view(-1, 2).to(torch.int64) & M32
    aip, bip = p[:, 0], p[:, 1]
    bp = fmix32(bip ^ A1)
    vidx = bp >> (32 - b)
    w = (bp << b) & M32
    rho = torch.clamp(clz32(w) + 1, max=L)
    j = fmix32(aip ^ fmix32(vidx ^ A0)) & (z - 1)
    val = (T << 5) | rho
    if stamps:  # layout S: the stamp of (rank rho, register j), L planes of z words; value T
        j = (rho - 1) * z + j
        val = torch.full_like(j, T)
    if packed:  # the DRV word of rank rho and the field's mask (plane-major, F fields per word)
        zb = packed_zb(K[name])
        F = 32 // zb
        r = rho - 1
        j = (r // F) * z + j
        val = ((1 << zb) - 1) << (zb * (r % F))
    out = torch.stack([j, val], dim=1).to(torch.int64)
    out = torch.where(out >= 1 << 31, out - (1 << 32), out).to(torch.int32)
    if out.shape[0] % 2:
        out = out[:-1]
    W = -(-(32 - b) // (32 // packed_zb(K[name]))) if packed else (L if stamps else 1)
    return out.contiguous(), z * W


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="caida,10G,bigwin")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--write", action="store_true")
    args = ap.parse_args()
    so = os.path.join(ROOT, "tools", "libubench_scanpath.so")
    src = os.path.join(ROOT, "tools", "ubench_scanpath.cu")
    if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                               "-shared", "-Xcompiler", "-fPIC", "-o", so, src])
    lib = ctypes.CDLL(so)
    lib.sp_run.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_int,
                           ctypes.c_void_p]
    dev = torch.device("cuda:0")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    res = {}
    for name in args.configs.split(","):
        rec, z = records(name, dev)
        sr = torch.zeros(z, dtype=torch.int32, device=dev)
        prec, pz = records(name, dev, packed=True)
        drv = torch.empty(pz, dtype=torch.int32, device=dev)
        srec, sz = records(name, dev, stamps=True) if name != "bigwin" else (None, 0)
        st = torch.zeros(sz, dtype=torch.int32, device=dev) if sz else None
        s = torch.cuda.current_stream(dev)
        out = {}
        modes = [(0, "check_then_atomic"), (1, "atomic_only"), (2, "u8_check_then_cas"),
                 (3, "packed_check_then_and")] + ([(4, "stamps_check_then_atomic")] if sz else [])
        for mode, key in modes:
            ts = []
            arr, recs = {3: (drv, prec), 4: (st, srec)}.get(mode, (sr, rec))
            for r in range(args.reps + 2):
                if mode == 3:
                    arr.fill_(-1)  # InitDR: every field saturated (all ones)
                else:
                    arr.zero_()
                flush.fill_(r & 0xFF)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                assert lib.sp_run(recs.data_ptr(), recs.shape[0], arr.data_ptr(), 0 if mode == 4 else mode,
                                  ctypes.c_void_p(s.cuda_stream)) == 0
                e1.record(s)
                torch.cuda.synchronize()
                if r >= 2:
                    ts.append(e0.elapsed_time(e1))
            ms = sum(ts) / len(ts)
            out[key] = round(recs.shape[0] / (ms * 1e-3) / 1e9, 2)
            out[key + "_ms"] = round(ms, 5)
        res[name] = out
        del rec, sr, prec, drv, srec, st
        torch.cuda.empty_cache()
    print(json.dumps(res))
    if args.write:
        path = os.path.join(ROOT, "profiles", "ceilings_b200.json")
        with open(path) as f:
            c = json.load(f)
        c["scan_path_Gpairs_s"] = {k: v["check_then_atomic"] for k, v in res.items()}
        c["scan_path_packed_Gpairs_s"] = {k: v["packed_check_then_and"] for k, v in res.items()}
        c["scan_path_stamps_Gpairs_s"] = {k: v["stamps_check_then_atomic"] for k, v in res.items()
                                          if "stamps_check_then_atomic" in v}
        c["scan_path_detail"] = res
        c["scan_path_source"] = ("tools/scan_ceiling.py + tools/ubench_scanpath.cu: the bench's "
                                 "slice hashed to (register, stamp) records, streamed through "
                                 "the scan's check load + atomicMax with no hashing and no "
                                 "shared-memory cache; L2 flushed before each run")
        with open(path, "w") as f:
            json.dump(c, f, indent=1)


if __name__ == "__main__":
    main()
