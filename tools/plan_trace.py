#!/usr/bin/env python
"""Where the staged-plan estimate's time goes (round 2 diagnostics).

Needs a libvbdr.so built with -DVBDR_PLAN_TRACE (tools/build_variant.py trace
VBDR_PLAN_TRACE=1, copied over the in-tree library on the GPU box): every CTA
stamps %globaltimer at its start, at each phase's full-barrier wait start / end
and release (consumer warp 0), at each refill issue (producer), at the end of
the loop and at the end of the finish.  Runs the caida estimate after an L2
flush and prints per-phase and per-part means over the 148 CTAs.
usage: python tools/plan_trace.py"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1810_13132_b200 import VBDR  # noqa: E402
from paper_1810_13132_b200.vbdr import lib  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    tr = synth.CONFIGS["caida"]
    pool = VBDR(128, 5, 1 << 22, device=dev)
    gen = synth.DeviceTrace(tr, dev)
    buf = torch.empty(2 * tr.pairs_per_slice, dtype=torch.int32, device=dev)
    for t in range(6):
        gen.generate_into(buf, t)
        pool.scan_slice(buf)
        pool.slide()
    hosts = torch.from_numpy(tr.host_ids().view(np.int32)).to(dev)
    plan = pool.plan(hosts, kind="staged")
    out = torch.empty(tr.hosts, dtype=torch.float64, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    L = lib()
    L.vbdr_debug_plan_trace.argtypes = [ctypes.c_void_p, ctypes.c_uint64]
    tr_host = np.zeros((148, 65, 4), dtype=np.uint64)
    runs = []
    for r in range(6):
        flush.fill_(r)
        torch.cuda.synchronize()
        pool.estimate_plan(plan, out=out)
        torch.cuda.synchronize()
        assert L.vbdr_debug_plan_trace(tr_host.ctypes.data, tr_host.nbytes) == 0
        runs.append(tr_host.astype(np.int64).copy())
    x = np.stack(runs[2:])  # [run, cta, phase, k]
    t0 = x[:, :, 64, 0].min(axis=1)[:, None]
    start = (x[:, :, 64, 0] - t0).mean()
    loop_end = (x[:, :, 64, 1] - t0).mean()
    fin_end = (x[:, :, 64, 2] - t0).mean()
    last = (x[:, :, 64, 2] - t0).max(axis=1).mean()
    wait = x[:, :, :64, 1] - x[:, :, :64, 0]
    work = x[:, :, :64, 2] - x[:, :, :64, 1]
    issue_lag = x[:, :, 2:64, 3] - x[:, :, :62, 2]  # refill of ph issued after warp 0 released ph-2
    print(f"caida staged-plan estimate, mean over 148 CTAs x {x.shape[0]} launches (us):")
    print(f"  CTA start (after the earliest)   {start / 1e3:7.2f}")
    print(f"  loop end                          {loop_end / 1e3:7.2f}")
    print(f"  finish end                        {fin_end / 1e3:7.2f}   (last CTA {last / 1e3:.2f})")
    print(f"  warp 0 per phase: wait for the stage {wait.mean() / 1e3:6.3f}, rounds {work.mean() / 1e3:6.3f}"
          f"  (sum over 64 phases: wait {wait.sum(axis=2).mean() / 1e3:.2f}, rounds "
          f"{work.sum(axis=2).mean() / 1e3:.2f})")
    print(f"  producer refill issued after warp 0's release of the stage: {issue_lag.mean() / 1e3:6.3f}")
    per_phase_wait = wait.mean(axis=(0, 1)) / 1e3
    print("  wait by phase (first 8, last 4):", np.round(per_phase_wait[:8], 3), np.round(per_phase_wait[-4:], 3))


if __name__ == "__main__":
    main()
