#!/usr/bin/env python
"""BASELINE.md section 5 rows from bench.py JSON lines (run here, on the CPU box).

usage: result_table.py <bench line .json> [...]

One markdown row per line: config, layout, N, scan rate and its fraction of the
ceiling the bench reports (layout F: the scan's memory path on the workload's
update stream; P, S: the SM-to-L2 random-request rate), slide time and HBM fraction, merge and
estimate times, gathers/s, the step (pipelined / serial / gather), e2e, the
oracle's rate when the line carries it.  Parity is the GPU test log's verdict
for that config (passed in with --parity, default "green")."""
import json
import sys


def row(d: dict, parity: str) -> str:
    c = d["config"]
    k = d["kernels"]
    sc, sl, es = k["scan"], k["slide"], k["estimate"]
    cpu = d.get("cpu_baseline") or {}
    e2e = d.get("e2e") or {}
    step = d["ms_per_step"]
    serial = d.get("ms_per_step_serial")
    gather = d.get("ms_per_step_gather")
    sb = {"scan_memory_path": "memory path", "l2_requests": "L2 requests"}.get(sc.get("bound"), "?")
    return ("| {w} | {lay} | {n} | {scan:,.0f} | {sfrac:.2f} ({sb}) | {slms:.4f} | {slgb:,.0f} ({slf:.0%}) | "
            "{merge} | {est:.4f} ({path}) | {gps:.1f} G | {step:.4f} / {ser} / {gat} | {val:,.0f} | "
            "{e2e} | {cpu} | {par} |").format(
        w=c["workload"], lay=c["layout"], n=d["n_gpus"],
        scan=d["scan_mpairs_s"], sfrac=sc["frac"], sb=sb, slms=d["slide_ms"], slgb=sl["achieved"],
        slf=sl["frac"], merge="—" if d["n_gpus"] == 1 else f"{d['merge_ms']:.4f}",
        est=d["estimate_ms"], path=c.get("estimate_path", "?"),
        gps=es["gathers_per_s"] / 1e9, step=step,
        ser=f"{serial:.4f}" if serial else "—", gat=f"{gather:.4f}" if gather else "—",
        val=d["value"], e2e=f"{e2e['value']:,.0f}" if e2e.get("value") else "—",
        cpu=f"{cpu['value']:.2f}" if cpu.get("value") else "—", par=parity)


HEADER = ("| config | layout | N | scan Mpairs/s | scan / its ceiling | slide ms | "
          "slide GB/s (of 6549.8) | merge ms | estimate ms (path) | gathers/s | "
          "step ms (headline / serial / gather estimate) | value Mpairs/s | e2e Mpairs/s | "
          "oracle Mpairs/s (1 core) | parity |\n"
          "|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|")


if __name__ == "__main__":
    args = sys.argv[1:]
    parity = "green"
    if args and args[0].startswith("--parity="):
        parity = args.pop(0).split("=", 1)[1]
    print(HEADER)
    for f in args:
        line = [ln for ln in open(f) if ln.startswith("{")][-1]
        print(row(json.loads(line), parity))
