"""Where does the end-to-end step time go?  (host enqueue time vs device time)"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import synth
from paper_1810_13132_b200 import VBDR

dev = torch.device("cuda:0")
tr = synth.CONFIGS["caida"]
pool = VBDR(128, 5, 1 << 22, device=dev)
gen = synth.DeviceTrace(tr, dev)
n = tr.pairs_per_slice
h_in = [gen.generate(t).cpu().pin_memory() for t in range(4)]
hosts = tr.host_ids()
h_hosts = torch.from_numpy(hosts.view(np.int32)).pin_memory()
h_out = torch.empty(len(hosts), dtype=torch.float64).pin_memory()
stage = torch.empty(4 * n, dtype=torch.int32, device=dev)
hs = torch.empty(len(hosts), dtype=torch.int32, device=dev)
os_ = torch.empty(len(hosts), dtype=torch.float64, device=dev)
d_in = torch.empty(2 * n, dtype=torch.int32, device=dev)
s = torch.cuda.current_stream()


def run(name, fn, steps=30):
    for i in range(3):
        fn(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for i in range(steps):
        fn(i)
    t_host = time.perf_counter() - t0
    e1.record()
    torch.cuda.synchronize()
    print(f"{name:40s} device {e0.elapsed_time(e1) / steps:7.3f} ms/step   host enqueue {t_host / steps * 1e3:7.3f} ms/step")


run("torch H2D 40MB only", lambda i: d_in.copy_(h_in[i % 4], non_blocking=True))
run("scan_slice_host only", lambda i: pool.scan_slice_host(h_in[i % 4], stage))
run("scan_slice_host + slide", lambda i: (pool.scan_slice_host(h_in[i % 4], stage), pool.slide()))
run("full e2e step", lambda i: (pool.scan_slice_host(h_in[i % 4], stage), pool.slide(),
                                pool.estimate_host(h_hosts, hs, os_, h_out)))
run("device-resident step (no copies)", lambda i: (pool.scan_slice(d_in), pool.slide(),
                                                   pool.estimate(hs, out=os_)))
plan = pool.plan(torch.from_numpy(hosts.view(np.int32)).to(dev))
run("e2e step, plan estimate + D2H", lambda i: (pool.scan_slice_host(h_in[i % 4], stage), pool.slide(),
                                               pool.estimate_plan_host(plan, os_, h_out)))
run("e2e step, plan estimate, no D2H", lambda i: (pool.scan_slice_host(h_in[i % 4], stage), pool.slide(),
                                                 pool.estimate_plan(plan, out=os_)))
small = torch.empty(2 * n, dtype=torch.int32, device=dev)  # half-slice chunks
run("e2e step, half-slice chunks", lambda i: (pool.scan_slice_host(h_in[i % 4], small), pool.slide(),
                                             pool.estimate_plan_host(plan, os_, h_out)))
quarter = torch.empty(n, dtype=torch.int32, device=dev)  # quarter-slice chunks
run("e2e step, quarter-slice chunks", lambda i: (pool.scan_slice_host(h_in[i % 4], quarter), pool.slide(),
                                                pool.estimate_plan_host(plan, os_, h_out)))
eighth = torch.empty(n // 2, dtype=torch.int32, device=dev)
run("e2e step, eighth-slice chunks", lambda i: (pool.scan_slice_host(h_in[i % 4], eighth), pool.slide(),
                                               pool.estimate_plan_host(plan, os_, h_out)))
