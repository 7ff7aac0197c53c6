"""Estimate accuracy of the method (oracle, CPU) against Definition 1 counts
on the synthetic workloads -- context only: the paper reports no accuracy
numbers, so estimates on shared, skewed pools are parity-unpinned.

usage: python tools/accuracy.py > profiles/r01_accuracy.txt
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import synth  # noqa: E402

BUCKETS = [(1, 10), (10, 100), (100, 1000), (1000, 10**4), (10**4, 10**9)]


def run(name, b, k, z, slices, seeds, estimators):
    rows = {e: {bk: [] for bk in BUCKETS} for e in estimators}
    for seed in seeds:
        base = synth.CONFIGS[name]
        tr = synth.TraceConfig(name, base.hosts, base.pairs_per_slice, base.U0, seed=seed)
        cfg = oracle.PoolConfig(b=b, k=k, z=z)
        ser, gsm = oracle.Pool(cfg, "serial"), oracle.Pool(cfg, "gsmall")
        sl = [synth.generate(tr, t) for t in range(slices)]
        for s in sl:
            ser.slice(s)
            gsm.slice(s)
        exact = oracle.exact_cardinalities(sl[-k:])
        hosts = np.array(sorted(exact), dtype=np.uint32)
        n = np.array([exact[int(h)] for h in hosts])
        M = ser.readout()
        for e in estimators:
            V = gsm.readout_pcsa() if e == "pcsa" else M
            est = oracle.estimate_variant(V, hosts, b, z, e)
            for lo, hi in BUCKETS:
                sel = (n >= lo) & (n < hi)
                rows[e][(lo, hi)].extend((est[sel] / n[sel] - 1).tolist())
    print(f"\n## {name}: g={1 << b}, n_phys=2^{z.bit_length() - 1}, k={k}, {slices} slices, "
          f"seeds {list(seeds)}; relative error (estimate/exact - 1) of hosts seen in the window")
    print(f"{'estimator':9s} {'cardinality':>14s} {'hosts':>8s} {'mean':>8s} {'RMS':>8s} "
          f"{'median':>8s}")
    for e in estimators:
        for (lo, hi), v in rows[e].items():
            if not v:
                continue
            v = np.array(v)
            print(f"{e:9s} {f'[{lo},{hi})':>14s} {len(v):8d} {v.mean():+8.3f} "
                  f"{np.sqrt(np.mean(v ** 2)):8.3f} {np.median(v):+8.3f}")


if __name__ == "__main__":
    print("# VBDR estimate accuracy on synthetic Zipf traces (oracle; tools/accuracy.py)")
    print("# textbook HLL standard error 1.04/sqrt(g): g=32 -> 0.184, g=128 -> 0.092")
    run("tiny", 5, 4, 1 << 12, 8, range(1, 13), ("hll", "loglog", "pcsa"))
    run("caida", 7, 5, 1 << 22, 6, [1], ("hll", "loglog", "pcsa"))
