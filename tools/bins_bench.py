"""Time dgsm_build_bins (a3-a5: depth sort, key duplication, tile sort, ranges +
the bins' copy-out) on cfg2 with CUDA events, median of N.
Usage: python tools/bins_bench.py [N]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_01660_b200 import dgsm, synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
s = synth.config2()
p = dgsm.BuildPlan(dgsm.to_device(s.gaussians), s.lights, s.res, s.K)
ts = []
for it in range(n + 3):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    p.bins()
    b.record()
    torch.cuda.synchronize()
    if it >= 3:
        ts.append(a.elapsed_time(b))
ts.sort()
print(f"bins_ms median {ts[len(ts) // 2]:.4f} min {ts[0]:.4f}")
