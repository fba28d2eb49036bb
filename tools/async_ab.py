"""cfg2 step (build + query) with dgsm_build (plan sync) vs the sync-free build
at key capacity P and 1.25 P; L2 flushed, device time per step (median of 20)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2601_01660_b200 import dgsm, synth  # noqa: E402

s = synth.config2()
g = dgsm.to_device(s.gaussians)
x = torch.from_numpy(s.queries).cuda()
x = x[dgsm.receiver_order(x).long()].contiguous()
atlas = torch.empty((1, s.K, s.res, s.res), device="cuda")
T = torch.empty(x.shape[0], device="cuda")
flush = torch.empty(64 << 20, device="cuda")
P = dgsm.BuildPlan(g, s.lights, s.res, s.K).n_keys
b = dgsm.Builder(s.lights, s.res, s.K)
variants = {"dgsm_build": lambda: b(g, atlas)}
for f in (1.0, 1.25):
    ab = dgsm.AsyncBuilder(s.lights, s.res, s.K, s.n, int(f * P))
    variants[f"async x{f}"] = (lambda ab=ab: ab(g, atlas))
for name, fn in variants.items():
    ts = []
    for i in range(25):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        dgsm.query(atlas, s.lights, x, out=T)
        e1.record()
        torch.cuda.synchronize()
        if i >= 5:
            ts.append(e0.elapsed_time(e1))
    print(f"{name:14s} step {np.median(ts):.4f} ms (min {np.min(ts):.4f})")
