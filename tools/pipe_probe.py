#!/usr/bin/env python
"""Timeline of the pipelined caida step (run on a B200 from the repo root).

The estimate of slice t on a second stream beside the scan and slide of slice
t+1 (bench.py step_pipelined), with CUDA events at every kernel boundary on
both streams; prints the mean start / end of each kernel relative to the step's
first event, so the overlap the schedule actually gets is visible.
usage: python tools/pipe_probe.py [--scan-mode M] [--estimate staged|sorted|gather]"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1810_13132_b200 import VBDR  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scan-mode", type=int, default=0)
    ap.add_argument("--estimate", default="staged")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--config", default="caida", choices=["caida", "10G"])
    ap.add_argument("--order", default="scan-first", choices=["scan-first", "estimate-first"],
                    help="scan-first: bench.py's schedule (the estimate is enqueued after the "
                         "scan, beside the slide); estimate-first: round 1's")
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    tr = synth.CONFIGS[args.config]
    m, k, z = (128, 5, 1 << 22) if args.config == "caida" else (256, 10, 1 << 26)
    pool = VBDR(m, k, z, scan_mode=args.scan_mode, device=dev)
    gen = synth.DeviceTrace(tr, dev)
    inputs = []
    for t in range(8):
        buf = torch.empty(2 * tr.pairs_per_slice, dtype=torch.int32, device=dev)
        gen.generate_into(buf, t, start=0)
        inputs.append(buf)
    hosts = torch.from_numpy(tr.host_ids().view(np.int32)).to(dev)
    plan = pool.plan(hosts, kind=args.estimate) if args.estimate != "gather" else None
    out = torch.empty(tr.hosts, dtype=torch.float64, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    main_s = torch.cuda.current_stream(dev)
    side = torch.cuda.Stream(dev)

    def est(on):
        if plan is not None:
            pool.estimate_plan(plan, out=out, stream=on)
        else:
            pool.estimate(hosts, out=out, stream=on)

    names = ["step0", "est_start", "est_end", "scan_end", "slide_end", "step_end"]
    rec = []
    for i in range(args.steps + 5):
        flush.fill_(i & 0xFF)
        ev = {n: torch.cuda.Event(enable_timing=True) for n in names}
        ev["step0"].record(main_s)
        if args.order == "scan-first":
            pool.scan_slice(inputs[i % 8])
            ev["scan_end"].record(main_s)
        closed = torch.cuda.Event()
        closed.record(main_s)
        side.wait_event(closed)
        ev["est_start"].record(side)
        est(side)
        ev["est_end"].record(side)
        if args.order != "scan-first":
            pool.scan_slice(inputs[i % 8])
            ev["scan_end"].record(main_s)
        pool.slide()
        ev["slide_end"].record(main_s)
        main_s.wait_event(ev["est_end"])
        ev["step_end"].record(main_s)
        rec.append(ev)
    torch.cuda.synchronize()
    t = {n: [] for n in names[1:]}
    for ev in rec[5:]:
        for n in names[1:]:
            t[n].append(ev["step0"].elapsed_time(ev[n]) * 1e3)
    print(f"{args.config}, {args.order}, scan mode {args.scan_mode or 'default'}, {args.estimate} estimate, mean over "
          f"{args.steps} pipelined steps (us from the step's start):")
    for n in names[1:]:
        print(f"  {n:10s} {np.mean(t[n]):8.1f}  (min {np.min(t[n]):.1f}, max {np.max(t[n]):.1f})")


if __name__ == "__main__":
    main()
