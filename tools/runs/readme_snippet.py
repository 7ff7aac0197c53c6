import torch, numpy as np, synth
from paper_1810_13132_b200 import VBDR

pool = VBDR(m=128, k=5, n_phys=1 << 22)              # caida-sized pool
tr = synth.CONFIGS["caida"]
for t in range(6):
    pairs = synth.DeviceTrace(tr, "cuda").generate(t)  # u32[2*Np] (aip, bip)
    pool.scan_slice(pairs)
    pool.slide()
hosts = torch.from_numpy(tr.host_ids().view(np.int32)).cuda()
est = pool.estimate(hosts)                            # float64 per host
plan = pool.plan(hosts)                               # once per host list
est2 = pool.estimate_plan(plan)                       # same values, 2.8x faster

import numpy as np
assert np.array_equal(est.cpu().numpy(), est2.cpu().numpy()); print('readme ok', float(est.max()))
