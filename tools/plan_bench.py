"""Time dgsm_build_plan (projection a1-a2 + key-count scan + the P read-back) on
cfg2, CUDA events around each call, median of N.  Usage: python tools/plan_bench.py [N]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_01660_b200 import dgsm, synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
s = synth.config2()
g = dgsm.to_device(s.gaussians)
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
ts = []
for it in range(n + 3):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    p = dgsm.BuildPlan(g, s.lights, s.res, s.K)
    b.record()
    torch.cuda.synchronize()
    if it >= 3:
        ts.append(a.elapsed_time(b))
ts.sort()
print(f"plan_ms median {ts[len(ts) // 2]:.4f} min {ts[0]:.4f} keys {p.n_keys}")
