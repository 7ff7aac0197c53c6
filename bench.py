#!/usr/bin/env python
"""bench.py -- the VBDR hot path on B200 (one JSON line on rank 0).

A step is one slice of the method over one batch of synthetic input:
    vbdr_scan_slice (Np pairs) -> [N>1: merge] -> vbdr_slide
    -> estimate of all H hosts (vbdr_estimate_plan with a plan built once
       before the timed region when the pool allows one, else vbdr_estimate)
on BASELINE.json configs[1] ('caida': 5M pairs/slice, 500k Zipf hosts, m=128,
2^22 physical BDRs, k=5) unless --config says otherwise.

value   = pairs/s of whole steps (Mpairs/s), inputs resident in HBM, L2 flushed
          before every step, device time from CUDA events, max over ranks.
e2e     = the same through the host-buffer C ABI entry points (pinned host pairs
          copied in, estimates copied out, inside the timed region).
Under torchrun (N>1) each rank scans 1/N of every slice's pairs and the
ranks merge their slice ranks before the slide (--merge: default "sharded" =
NCCL reduce-scatter(MAX) of the u8 per-BDR ranks, a sharded slide, an
all-gather of the register shards and an all-reduce of the pool sums;
"stamps" = allreduce(MAX) of the stamp words; "delta"; "p2p" = the fused
peer-memory merge+slide); each rank estimates 1/N of the hosts.

--impl reference times the oracle (oracle/, single thread, host cores) on a
1/32-scale replica of the same workload; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

MEASURED_PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback

# BASELINE.json workloads -> (m, k, n_phys)
WORKLOADS = {
    "tiny": dict(m=32, k=4, n_phys=1 << 12),
    "caida": dict(m=128, k=5, n_phys=1 << 22),
    "caida_bursty": dict(m=128, k=5, n_phys=1 << 22),  # caida with packet trains
    "10G": dict(m=256, k=10, n_phys=1 << 26),
    "bigwin": dict(m=256, k=60, n_phys=1 << 28),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="vbdr", choices=["vbdr", "reference"])
    ap.add_argument("--config", default="caida", choices=list(WORKLOADS))
    ap.add_argument("--layout", default="fast", choices=["fast", "packed", "stamps"])
    ap.add_argument("--scan-mode", type=int, default=0)
    ap.add_argument("--est-lanes", type=int, default=0)
    ap.add_argument("--est-pass-log2", type=int, default=0)
    ap.add_argument("--estimator", default="hll", choices=["hll", "loglog", "pcsa"])
    ap.add_argument("--estimate", default="auto",
                    choices=["auto", "gather", "sorted", "staged", "passid"],
                    help="estimate path: gather (any host list) or a plan built once for the "
                         "fixed host list (include/vbdr.h vbdr_plan_kind); auto = every path "
                         "this pool takes, timed on the warm pool, the fastest kept")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo + --same-device: exercise the N>1 control flow on one GPU "
                         "(collectives on the CPU, no GPU-side waiting between ranks)")
    ap.add_argument("--same-device", action="store_true",
                    help="every rank uses cuda:0 (multi-rank logic test on a 1-GPU box)")
    ap.add_argument("--shard-state", action="store_true",
                    help="N>1 with --merge sharded/sparse: each rank stores only its "
                         "shard's DRV (register-sharded state, DRV memory /N)")
    ap.add_argument("--merge", default="sharded",
                    choices=["stamps", "delta", "sharded", "sparse", "p2p", "nvls"],
                    help="N>1 slide merge (paper_1810_13132_b200.slide_merged)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--pipeline", default="auto", choices=["auto", "on", "off"],
                    help="headline from software-pipelined steps: the estimate of slice t "
                         "overlaps the scan and slide of slice t+1 on a second stream "
                         "(profiles/r01_pipeline.txt).  auto = on with the shared-memory plan "
                         "estimate (+9 %% at caida), off with the gather estimate (-24 %% at 10G)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--flush-mib", type=int, default=512)
    return ap.parse_args()


def peaks():
    try:
        with open(MEASURED_PEAKS) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


CEIL_SRC = "profiles/ceilings_b200.json, tools/ubench_gather.cu"


def ceilings():
    with open(os.path.join(ROOT, "profiles", "ceilings_b200.json")) as f:
        return json.load(f)


def load_traffic(config: str, layout: str, est_path: str) -> dict:
    """dram__bytes_read.sum + dram__bytes_write.sum per launch from the last
    committed ncu --set full capture (profiles/traffic.json), or {}.  Keys
    "<config>/<layout>/<kernel>"; the estimate's key names its path
    ("estimate/<path>", e.g. "estimate/staged plan")."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f)
    except Exception:
        return {}
    pre = f"{config}/{layout}/"
    out = {k[len(pre):]: v for k, v in t.items() if k.startswith(pre)}
    out["estimate"] = out.get(f"estimate/{est_path}")
    return out


def plan_stream_bytes(plan, gathers: int, hosts: int, n_phys: int):
    """Bytes a plan estimate streams by design: 4 B of plan entry per gather
    (padding not counted), the register array once, 8 B out per host."""
    if plan is None:
        return None
    if plan.kind == "passid":  # host ids + 2 bits per gather + registers + out
        return 4 * hosts + gathers // 4 + n_phys + 8 * hosts
    return 4 * gathers + n_phys + 8 * hosts


def table1_bits(m: int, k: int) -> dict:
    """Table 1 with log2(n/g) -> L = 32 - log2(m) and
    log2(k+1) -> ceil(log2(k+1)): bits per BDR of the paper's three variants."""
    L = 32 - (m.bit_length() - 1)
    zb = max(1, (k).bit_length())  # ceil(log2(k+1))
    lgL = (L - 1).bit_length()     # ceil(log2 L)
    return {"serial": lgL + L * zb, "gfast": L + L * zb, "gsmall": L * zb}


def algorithmic_bytes_per_bdr(layout: str, words: int) -> int:
    """Slide kernel, per physical BDR: read sr (4 B, fast only), read+write W
    packed DRV words (8 W B), write the register value (1 B); layout stamps:
    read the L stamps (4 L B, words = L), write the register.  DESIGN.md s.6."""
    if layout == "stamps":
        return 4 * words + 1
    return (4 if layout == "fast" else 0) + 8 * words + 1


# ----------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.proc = None
        self.path = os.path.join("/tmp", f"vbdr_clocks_{os.getpid()}.csv")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={gpu_index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def wait_first(self, timeout: float = 5.0):
        """Block until nvidia-smi wrote its first sample (it takes a while to start)."""
        t0 = time.time()
        while self.proc is not None and time.time() - t0 < timeout:
            try:
                if os.path.getsize(self.path) > 0:
                    return
            except OSError:
                pass
            time.sleep(0.02)

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        sms, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sms.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sms:
            return None
        return {"sm_mhz": float(np.median(sms)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sms)}


# ------------------------------------------------------------- reference arm
def oracle_slice_time(tr: synth.TraceConfig, wl: dict, seconds: float, min_slices: int,
                      scale: int):
    """Time the oracle (serial VBDR, single thread) on whole slices of a
    1/scale replica of the workload.  Returns (seconds per slice, pairs/slice,
    slices, sample description)."""
    import oracle
    oracle.lib()
    try:
        os.sched_setaffinity(0, {sorted(os.sched_getaffinity(0))[0]})
    except Exception:
        pass
    n_phys = wl["n_phys"] // scale
    np_pairs = tr.pairs_per_slice // scale
    hosts_n = max(1, tr.hosts // scale)
    b = wl["m"].bit_length() - 1
    cfg = oracle.PoolConfig(b=b, k=wl["k"], z=n_phys)
    pool = oracle.Pool(cfg, "serial")
    hosts = tr.host_ids()[:hosts_n]
    slices = [synth.generate(tr, t, 0, np_pairs) for t in range(min(4, max(min_slices, 1)))]
    pool.slice(slices[0])  # warm: touches the whole pool once
    times, phases = [], []
    t_all = time.perf_counter()
    i = 0
    while (time.perf_counter() - t_all < seconds) or len(times) < min_slices:
        pairs = slices[i % len(slices)]
        t0 = time.perf_counter()
        pool.begin_slice()
        pool.scan(pairs)
        t1 = time.perf_counter()
        pool.end_slice()
        M = pool.readout()
        t2 = time.perf_counter()
        pool.estimate(M, hosts)
        t3 = time.perf_counter()
        times.append(t3 - t0)
        phases.append((t1 - t0, t2 - t1, t3 - t2))
        i += 1
    sample = (f"oracle serial VBDR, 1 thread, {'full-size' if scale == 1 else f'1/{scale}-scale'} "
              f"{tr.name} slices: {np_pairs} pairs scanned + {n_phys} BDRs closed + {hosts_n} "
              f"hosts estimated per slice, {len(times)} slices")
    ph = np.mean(np.array(phases), axis=0)
    detail = {"ns_per_pair_scan": round(ph[0] / np_pairs * 1e9, 2),
              "ns_per_bdr_close": round(ph[1] / n_phys * 1e9, 2),
              "ns_per_host_estimate": round(ph[2] / hosts_n * 1e9, 2),
              "cpu_model": cpu_model(), "host_cpus": os.cpu_count()}
    return float(np.mean(times)), np_pairs, len(times), sample, detail


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    tr = synth.CONFIGS[args.config]
    wl = WORKLOADS[args.config]
    scale = 32 if args.config != "tiny" else 1
    import oracle
    b = wl["m"].bit_length() - 1
    cfg = oracle.PoolConfig(b=b, k=wl["k"], z=wl["n_phys"] // scale)
    pool = oracle.Pool(cfg, "serial")
    np_pairs = tr.pairs_per_slice // scale
    hosts = tr.host_ids()[:max(1, tr.hosts // scale)]
    slices = [synth.generate(tr, t, 0, np_pairs) for t in range(4)]
    try:
        os.sched_setaffinity(0, {sorted(os.sched_getaffinity(0))[0]})
    except Exception:
        pass

    def step(i):
        pool.begin_slice()
        pool.scan(slices[i % 4])
        pool.end_slice()
        pool.estimate(pool.readout(), hosts)

    for i in range(args.warmup):
        step(i)
    t0 = time.perf_counter()
    for i in range(args.steps):
        step(i)
    dt = (time.perf_counter() - t0) / args.steps
    value = np_pairs / dt / 1e6
    sample = (f"oracle serial VBDR, 1 thread, 1/{scale}-scale {args.config}: {np_pairs} pairs + "
              f"{cfg.z} BDRs + {len(hosts)} hosts per step")
    line = {
        "impl": "reference", "metric": "IP pairs scanned per second through whole slices "
        "(scan + slide + estimate)", "value": round(value, 4), "unit": "Mpairs/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": args.config, "layout": "oracle-serial", **wl,
                   "pairs_per_slice": tr.pairs_per_slice, "hosts": tr.hosts,
                   "sample_scale": f"1/{scale}"},
        "cpu_baseline": {"value": round(value, 4), "unit": "Mpairs/s", "cores": 1,
                         "kind": "oracle", "sample": sample},
        "e2e": {"value": round(value, 4), "unit": "Mpairs/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
def run_vbdr(args):
    import torch
    import torch.distributed as dist

    from paper_1810_13132_b200 import (VBDR, NvlsMerge, PeerMerge, SparseMerge,
                                       all_gather_shards, make_config, merge_stamps,
                                       reduce_scatter_max, shard_range)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if args.same_device and args.dist_backend == "nccl" and world > 1:
        raise SystemExit("--same-device needs --dist-backend gloo (NCCL ranks sharing a GPU "
                         "would spin-wait on each other)")
    gpu = 0 if args.same_device else local
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    group = None
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
        group = dist.group.WORLD

    tr = synth.CONFIGS[args.config]
    wl = WORKLOADS[args.config]
    if world > 1 and args.layout == "packed" and args.merge != "nvls":
        raise SystemExit("multi-GPU layout packed needs --merge nvls (NCCL has no bitwise-AND "
                         "reduction; the NVSwitch multimem.ld_reduce has)")
    if world > 1 and args.layout == "stamps" and args.merge != "stamps":
        raise SystemExit("multi-GPU layout stamps merges with --merge stamps (allreduce MAX)")
    if world > 1:
        print(f"rank {rank}: {args.dist_backend} communicator of {dist.get_world_size()} ranks, "
              f"device {torch.cuda.get_device_name(dev)} (cuda:{gpu})", file=sys.stderr, flush=True)
    shard_state = args.shard_state and world > 1 and args.merge in ("sharded", "sparse", "nvls") \
        and args.layout == "fast"
    state, mcbuf, mc_note = None, None, None
    one_nvls = world == 1 and args.merge == "nvls"
    if one_nvls:
        # one GPU: the multicast slide on a one-device multicast object (the
        # kernel's cost without peers; McBuffer = vbdr_mc_alloc), or, where
        # the driver refuses multicast objects, the group-of-one form of the
        # same kernel through the pool's own state
        from paper_1810_13132_b200 import McBuffer, state_bytes
        try:
            mcbuf = McBuffer(state_bytes(make_config(wl["m"], wl["k"], wl["n_phys"],
                                                     layout=args.layout)), dev)
            state = mcbuf.tensor
            mc_note = "slide through a one-device multicast object (NVLS kernel)"
        except RuntimeError as e:
            mc_note = (f"multicast slide kernel, group of one through the pool's own state "
                       f"(no multicast object here: {str(e)[:120]})")
    if world > 1 and args.merge in ("p2p", "nvls"):  # pool state in symmetric memory
        cfg = make_config(wl["m"], wl["k"], wl["n_phys"], layout=args.layout,
                          drv_shards=world if shard_state else 0,
                          drv_shard=rank if shard_state else 0)
        state = PeerMerge.alloc_state(cfg, dev)
    pool = VBDR(wl["m"], wl["k"], wl["n_phys"], layout=args.layout, scan_mode=args.scan_mode,
                est_lanes=args.est_lanes, est_pass_log2=args.est_pass_log2,
                estimator=args.estimator, device=dev, state=state,
                drv_shards=world if shard_state else 0, drv_shard=rank if shard_state else 0)
    peer = None
    if state is not None and world > 1:
        peer = PeerMerge(pool, group) if args.merge == "p2p" else NvlsMerge(pool, group)
    sparse = SparseMerge(pool, group) if world > 1 and args.merge == "sparse" else None
    info = pool.info()
    p0, p1 = shard_range(tr.pairs_per_slice, rank, world)
    h0, h1 = shard_range(tr.hosts, rank, world)
    n_local = p1 - p0
    gen = synth.DeviceTrace(tr, dev)
    n_inputs = min(args.steps + args.warmup, 16)
    inputs = []
    for t in range(n_inputs):
        buf = torch.empty(2 * n_local, dtype=torch.int32, device=dev)
        gen.generate_into(buf, t, start=p0)
        inputs.append(buf)
    hosts_all = tr.host_ids()
    hosts = torch.from_numpy(hosts_all[h0:h1].view(np.int32)).to(dev)
    est_out = torch.empty(h1 - h0, dtype=torch.float64, device=dev)
    # plans of every kind this pool takes for the rank's host list (built once,
    # outside the timed region; the build time is reported)
    plans, plan_build = {}, {}
    kinds = ("sorted", "staged", "passid") if args.estimate == "auto" else \
        (() if args.estimate == "gather" else (args.estimate,))
    for kind in kinds:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        try:
            plans[kind] = pool.plan(hosts, kind=kind)
            plan_build[kind] = round((time.perf_counter() - t0) * 1e3, 2)
        except ValueError:
            if args.estimate != "auto":
                raise
    plan = next(iter(plans.values()), None)

    def estimate(out, on=None):
        if plan is not None:
            pool.estimate_plan(plan, out=out, stream=on)
        else:
            pool.estimate(hosts, out=out, stream=on)
    flush = torch.empty(args.flush_mib << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            if args.dist_backend == "nccl":
                dist.barrier(device_ids=[gpu])
            else:
                dist.barrier()
        torch.cuda.synchronize()

    E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    n_shard = wl["n_phys"] // world
    delta_buf = torch.empty(wl["n_phys"], dtype=torch.uint8, device=dev) if world > 1 else None
    shard_buf = torch.empty(n_shard, dtype=torch.uint8, device=dev) if world > 1 else None

    def mark(evs, j):
        if evs:
            evs[j].record(stream)

    def close_slice(evs=None):
        """slide_merged, spelled out so each phase gets its own events:
        [merge] -> slide kernel -> [register all-gather + pool-sum all-reduce]."""
        if world == 1:
            mark(evs, 2)
            if one_nvls:
                pool.slide_multicast(mcbuf.mc if mcbuf is not None else pool.state.data_ptr())
            else:
                pool.slide()
            mark(evs, 3)
        elif args.merge == "stamps":
            merge_stamps(pool, group)
            mark(evs, 2)
            pool.slide()
            mark(evs, 3)
        elif args.merge in ("p2p", "nvls"):
            peer.close_slice(on_merged=lambda: mark(evs, 2), on_slid=lambda: mark(evs, 3))
        elif args.merge == "sparse":
            sparse.close_slice()
            mark(evs, 2)
            mark(evs, 3)
        elif args.merge == "delta":
            pool.stamp_delta(delta_buf)
            dist.all_reduce(delta_buf, op=dist.ReduceOp.MAX, group=group)
            mark(evs, 2)
            pool.slide_delta(delta_buf)
            mark(evs, 3)
        else:
            pool.stamp_delta(delta_buf)
            reduce_scatter_max(delta_buf, shard_buf, group)
            mark(evs, 2)
            pool.slide_delta(shard_buf, rank * n_shard, (rank + 1) * n_shard)
            mark(evs, 3)
            all_gather_shards(pool.regmax_view(), group)
            dist.all_reduce(pool.acc_view(), op=dist.ReduceOp.SUM, group=group)
        mark(evs, 4)

    def step(i, evs=None):
        x = inputs[i % n_inputs]
        mark(evs, 0)
        pool.scan_slice(x)
        mark(evs, 1)
        close_slice(evs)
        estimate(est_out)
        mark(evs, 5)

    stream_b = torch.cuda.Stream(dev)
    ev_closed, ev_est = torch.cuda.Event(), torch.cuda.Event()

    def step_pipelined(i):
        """Software-pipelined step: the estimate of the slice closed last (t)
        runs on a second stream while the scan AND the slide of slice t+1 run
        on the main one.  The two register buffers alternate with the tick and
        the pool sums have four slots, so the slide of t+1 writes nothing the
        estimate of t reads.  The step ends when both streams are done (the
        main stream joins the estimate), so all of its work is inside the
        step's events and none overlaps the L2 flush between steps.  Same
        work per step as step(): one scan, one slide, one estimate."""
        x = inputs[i % n_inputs]
        ev_closed.record(stream)
        stream_b.wait_event(ev_closed)
        estimate(est_out, stream_b)
        ev_est.record(stream_b)
        pool.scan_slice(x)
        close_slice()
        stream.wait_event(ev_est)

    # warm-up
    for i in range(args.warmup):
        flush.fill_(i & 0xFF)
        step(i)
    barrier()

    # --estimate auto: every path this pool takes (the plans of each kind, the
    # gather) timed on the warm pool; the fastest is kept for this rank's host
    # share (same results on every path: integer sums, one fp64 finish).  A
    # staged plan streams the whole register array through every SM whatever
    # the host count, the gather scales with the hosts, the sorted plan with
    # both; which wins depends on the pool and the host count.
    est_choice = None
    if args.estimate == "auto":
        def time_est(p):
            evs = [(E(), E()) for _ in range(5)]
            for j in range(7):
                flush.fill_(j & 0xFF)
                if j >= 2:
                    evs[j - 2][0].record(stream)
                if p is not None:
                    pool.estimate_plan(p, out=est_out)
                else:
                    pool.estimate(hosts, out=est_out)
                if j >= 2:
                    evs[j - 2][1].record(stream)
            torch.cuda.synchronize()
            return float(np.median([a.elapsed_time(b) for a, b in evs]))
        names = ["sorted", "staged", "passid", "gather"]  # same list on every rank
        times = [time_est(plans.get(n)) if n in plans or n == "gather" else float("inf")
                 for n in names]
        if world > 1:  # one choice for every rank: the slowest rank decides
            t = torch.tensor(times, dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            times = t.cpu().tolist()
        est_choice = {f"{n}_ms": round(t, 5) for n, t in zip(names, times) if t != float("inf")}
        best = names[int(np.argmin(times))]
        plan = plans.get(best)
        for n in list(plans):  # free the plans not kept
            if n != best:
                plans.pop(n).release()
        barrier()
    est_path = "gather" if plan is None else f"{plan.kind} plan"

    # ---- device-resident timed region (clocks sampled through it and the e2e region)
    clocks = ClockSampler(gpu) if rank == 0 else None
    if clocks:
        clocks.wait_first()
    # per-kernel breakdown: a first pass with events between the kernels
    events = [[E() for _ in range(6)] for _ in range(args.steps)]
    barrier()
    for i in range(args.steps):
        flush.fill_(i & 0xFF)
        step(args.warmup + i, events[i])
    barrier()
    ms = np.array([[ev[j].elapsed_time(ev[j + 1]) for j in range(5)] for ev in events])
    ms_k = ms.mean(axis=0)  # scan, merge, slide, gather, estimate
    per_kernel_local = np.array([ms_k[0], ms_k[1] + ms_k[3], ms_k[2], ms_k[4]])
    # serial steps, events only around each step (nothing between its kernels)
    def timed_steps(fn, first):
        evs = [(E(), E()) for _ in range(args.steps)]
        l0 = pool.info()["launches"]
        barrier()
        for i in range(args.steps):
            flush.fill_(i & 0xFF)  # L2 flush (> 126 MB L2), outside the step events
            evs[i][0].record(stream)
            fn(first + i)
            evs[i][1].record(stream)
        barrier()
        per_step = [a.elapsed_time(b) for a, b in evs]
        return float(sum(per_step)), pool.info()["launches"] - l0, per_step

    serial_total, serial_launches, serial_steps = timed_steps(step, args.warmup + args.steps)
    # the pipelined schedule (same work per step: one scan, one slide, one
    # estimate); --pipeline auto times both and the faster is the headline
    pipe = None
    if args.pipeline in ("on", "auto"):
        pipe = timed_steps(step_pipelined, args.warmup + 2 * args.steps)
        if world > 1:  # one choice on every rank
            t = torch.tensor([serial_total, pipe[0]], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            st, pt = float(t[0]), float(t[1])
        else:
            st, pt = serial_total, pipe[0]
    pipelined = pipe is not None and (args.pipeline == "on" or pt < st)
    if pipelined:
        local_total, launches, local_steps = pipe
    else:
        local_total, launches, local_steps = serial_total, serial_launches, serial_steps
    pipelined_ms = pipe[0] / args.steps if pipe is not None else None
    # the step with the gather estimate (any host list, no plan): serial
    gather_ms = None
    if plan is not None:
        kept = plan
        plan = None
        gather_ms = timed_steps(step, args.warmup + 3 * args.steps)[0] / args.steps
        plan = kept
        if world > 1:
            t = torch.tensor([gather_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            gather_ms = float(t[0])
    # per-step spread (median and min over the measured slices)
    step_stats = np.array([np.median(local_steps), np.min(local_steps), np.max(local_steps)])
    if world > 1:
        t = torch.tensor(step_stats.tolist(), dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        step_stats = t.cpu().numpy()
    if world > 1:
        t = torch.tensor([local_total, *per_kernel_local.tolist()], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t[0])
        per_kernel = t[1:].cpu().numpy()
    else:
        total_ms = local_total
        per_kernel = per_kernel_local
    ms_per_step = total_ms / args.steps
    serial_ms = serial_total / args.steps
    if world > 1:
        t = torch.tensor([serial_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        serial_ms = float(t[0])
    value = tr.pairs_per_slice / (ms_per_step * 1e-3) / 1e6

    # ---- end to end through the host-buffer C ABI entry points
    e2e = None
    if not args.no_e2e:
        h_inputs = [inputs[i].cpu().pin_memory() for i in range(min(n_inputs, 4))]
        h_hosts = torch.from_numpy(hosts_all[h0:h1].view(np.int32)).pin_memory()
        h_out = torch.empty(h1 - h0, dtype=torch.float64).pin_memory()
        # two slots of half a slice each: the scan of one half overlaps the copy of
        # the next (tools/e2e_probe.py: 0.742 ms/step vs 0.779 with whole-slice slots)
        stage = torch.empty(2 * n_local, dtype=torch.int32, device=dev)
        hstage = torch.empty(max(h1 - h0, 1), dtype=torch.int32, device=dev)
        ostage = torch.empty(max(h1 - h0, 1), dtype=torch.float64, device=dev)

        def e2e_step(i):
            pool.scan_slice_host(h_inputs[i % len(h_inputs)], stage)
            close_slice()
            if plan is not None:  # the host list lives in the plan (built once)
                pool.estimate_plan_host(plan, ostage, h_out)
            else:
                pool.estimate_host(h_hosts, hstage, ostage, h_out)

        for i in range(3):
            e2e_step(i)
        barrier()
        # One timed region of K steps: the host-to-device copies of step i+1
        # overlap the slide/estimate of step i (vbdr_scan_slice_host).  No L2
        # flush here: every step's input arrives over PCIe from host memory.
        ev0, ev1 = E(), E()
        ev0.record(stream)
        for i in range(args.steps):
            e2e_step(i)
        ev1.record(stream)
        barrier()
        e2e_ms = ev0.elapsed_time(ev1)
        if world > 1:
            t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t[0])
        e2e = {"value": round(tr.pairs_per_slice / (e2e_ms / args.steps * 1e-3) / 1e6, 3),
               "unit": "Mpairs/s",
               "h2d_bytes_per_step": 8 * n_local * world + (0 if plan is not None else 4 * tr.hosts),
               "d2h_bytes_per_step": 8 * tr.hosts,
               "ms_per_step": e2e_ms / args.steps,
               "timing": "one CUDA-event region over all steps, copies pipelined across steps"}

    clk = clocks.stop() if clocks else None
    # a staged plan transfer that timed out leaves NaN estimates and sets the
    # plan's error flag: never report a number from such a run
    if plan is not None:
        pool.plan_check(plan)  # raises (non-zero exit) if any timed estimate failed
    if bool(torch.isnan(est_out).any()):
        raise SystemExit("bench: NaN estimates (a failed plan estimate)")
    if sparse is not None:
        sparse.check()  # raises if a fixed-capacity record buffer ever overflowed
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # ---- roofline of each kernel; the dominant one goes in "roofline".
    # achieved = SURVEY 8(d.4) algorithmic work per launch / the kernel's mean
    # CUDA-event time in the breakdown pass (DESIGN.md section 6 states each).
    hbm, hbm_src = peaks()
    ceil = ceilings()
    names = ["scan", "merge", "slide", "estimate"]
    kern = {n: float(v) for n, v in zip(names, per_kernel)}
    traffic = load_traffic(args.config, args.layout, est_path)
    slide_bytes = algorithmic_bytes_per_bdr(args.layout, info["words"]) * wl["n_phys"]
    slide_gbs = slide_bytes / (kern["slide"] * 1e-3) / 1e9
    n_hosts = h1 - h0
    gathers = n_hosts * wl["m"]
    # estimate, per host: 4 B host id in + 8 B estimate out + g one-byte registers
    est_bytes = n_hosts * (4 + 8 + wl["m"])
    est_gbs = est_bytes / (kern["estimate"] * 1e-3) / 1e9
    g_rate = gathers / (kern["estimate"] * 1e-3) / 1e9
    scan_rate = n_local / (kern["scan"] * 1e-3) / 1e9
    req_peak = ceil["ldg_gather_1B_Gps"]["4MiB"]
    path_key = {"fast": "scan_path_Gpairs_s", "packed": "scan_path_packed_Gpairs_s",
                "stamps": "scan_path_stamps_Gpairs_s"}.get(args.layout)
    path_peak = ceil.get(path_key, {}).get(args.config) if path_key else None
    if path_peak:
        # the scan's own memory path on this workload's update stream (check
        # load + atomicMax per pair -- layout P: + atomicAnd of the field --
        # no hashing, no shared-memory cache)
        scan_roof = {"bound": "scan_memory_path", "peak": path_peak,
                     "frac": round(scan_rate / path_peak, 4),
                     "peak_source": ceil.get("scan_path_source", "profiles/ceilings_b200.json")
                                    + "; above 1 where the block cache absorbs check loads",
                     "peak_l2_requests": req_peak}
    else:
        scan_roof = {"bound": "l2_requests", "peak": req_peak,
                     "frac": round(scan_rate / req_peak, 4),
                     "peak_source": "SM-to-L2 request rate: random 1-byte loads from an "
                                    f"L2-resident table ({CEIL_SRC}); every pair costs at least "
                                    "one L2 request (its check load or its atomic) unless the "
                                    "block's shared-memory cache absorbs it"}
    kernels = {
        "scan": {"ms": kern["scan"], "achieved": round(scan_rate, 2), "unit": "Gpairs/s",
                 "traffic": traffic.get("scan"), **scan_roof},
        "merge": {"ms": kern["merge"]},
        "slide": {"ms": kern["slide"], "bound": "hbm", "achieved": round(slide_gbs, 1),
                  "peak": hbm, "unit": "GB/s", "frac": round(slide_gbs / hbm, 4),
                  "traffic": traffic.get("slide"), "algorithmic_bytes": slide_bytes,
                  "peak_source": hbm_src},
        "estimate": {"ms": kern["estimate"], "path": est_path, "bound": "hbm",
                     "achieved": round(est_gbs, 1), "peak": hbm, "unit": "GB/s",
                     "frac": round(est_gbs / hbm, 4), "algorithmic_bytes": est_bytes,
                     "traffic": traffic.get("estimate"),
                     "traffic_impl": plan_stream_bytes(plan, gathers, n_hosts, wl["n_phys"]),
                     "hosts": n_hosts, "gathers": gathers, "gathers_per_s": round(g_rate * 1e9),
                     "peak_source": hbm_src,
                     "note": "algorithmic bytes = SURVEY 8(d.4): 4 B host in + 8 B out + g x "
                             "1 B registers per host; traffic_impl = what the path streams "
                             "by design (plan entries, 4 B per gather)",
                     # context: the staged plan's own stream alone (tools/ubench_stream.cu)
                     **({"stream_floor_ms": ceil["plan_stream_floor_us"][args.config] / 1e3,
                         "stream_floor_frac": round(ceil["plan_stream_floor_us"][args.config]
                                                    / 1e3 / kern["estimate"], 4),
                         "stream_floor_source": ceil.get("plan_stream_source")}
                        if est_path == "staged plan"
                        and args.config in ceil.get("plan_stream_floor_us", {}) else {})},
    }
    dominant = max(("scan", "slide", "estimate"), key=lambda n: kern[n])
    roof = {"kernel": dominant, **{k: v for k, v in kernels[dominant].items() if k != "ms"}}

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        sec, npairs, nsl, sample, detail = oracle_slice_time(tr, wl, args.cpu_seconds, 2, 1)
        cpu = {"value": round(npairs / sec / 1e6, 4), "unit": "Mpairs/s", "cores": 1,
               "kind": "oracle", "sample": sample, **detail}

    line = {
        "metric": "IP pairs scanned per second through whole slices (scan + slide + estimate)",
        "value": round(value, 3), "unit": "Mpairs/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_per_step, 5),
        "ms_per_step_serial": round(serial_ms, 5),
        # the same step with the gather estimate (an arbitrary host list, no plan)
        "ms_per_step_gather": round(gather_ms, 5) if gather_ms is not None else round(serial_ms, 5),
        "step_ms": {"median": round(float(step_stats[0]), 5), "min": round(float(step_stats[1]), 5),
                    "max": round(float(step_stats[2]), 5)},
        "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": args.config, "layout": args.layout, **wl,
                   "pairs_per_slice": tr.pairs_per_slice, "hosts": tr.hosts,
                   "parallelism": (f"pairs+hosts sharded x{world}, merge={args.merge}"
                                   + (", register-sharded state" if shard_state else "")
                                   if world > 1 else "single GPU" +
                                   (f", {mc_note}" if mc_note else "")),
                   "l2": f"flushed before every step ({args.flush_mib} MiB write)",
                   "schedule": ("pipelined: estimate(t) on a 2nd stream overlaps scan(t+1) "
                                "and slide(t+1)"
                                if pipelined else "serial"),
                   "ms_per_step_pipelined": round(pipelined_ms, 5) if pipelined_ms else None,
                   "scan_mode": args.scan_mode, "est_lanes": args.est_lanes,
                   "estimator": args.estimator,
                   "estimate_path": est_path,
                   "plan_build_ms": plan_build.get(plan.kind) if plan is not None else None,
                   "estimate_autotune": est_choice,
                   "plan_bytes": plan.nbytes if plan is not None else None,
                   "zbits": info["zbits"], "words_per_bdr": info["words"],
                   "bits_per_bdr": (32 if args.layout == "fast" else 0) + 32 * info["words"],
                   "state_bytes": info["state_bytes"],
                   "table1_bits_per_bdr": table1_bits(wl["m"], wl["k"])},
        "scan_mpairs_s": round(tr.pairs_per_slice / (kern["scan"] * 1e-3) / 1e6, 2),
        "slide_ms": round(kern["slide"], 5), "estimate_ms": round(kern["estimate"], 5),
        "merge_ms": round(kern["merge"], 5),
        "kernels": kernels,
        "roofline": roof,
        "roofline_slide_hbm": {k: v for k, v in kernels["slide"].items() if k != "ms"},
        "gpu_launches": int(launches),
        "clocks": clk,
        "e2e": e2e,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_vbdr(args)


if __name__ == "__main__":
    main()
