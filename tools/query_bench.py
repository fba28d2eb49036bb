"""Query kernel micro-benchmark on a cfg2-shaped atlas (512^2 x 64, 1 light,
1M receivers), L2 flushed before each launch; prints mean/min us."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2601_01660_b200 import dgsm, synth  # noqa: E402

res, K, m = 512, 64, 1_000_000
s = synth.config2()
lights = s.lights
atlas = torch.from_numpy(synth.random_atlas(5, 1, K, res)).cuda()
x = torch.from_numpy(s.queries[:m]).cuda()
out = torch.empty(m, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ts = []
for i in range(30):
    flush.zero_()
    torch.cuda._sleep(400_000)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    dgsm.query(atlas, lights, x, out=out)
    b.record()
    torch.cuda.synchronize()
    if i >= 5:
        ts.append(a.elapsed_time(b) * 1e3)
warm = []
for i in range(20):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(400_000)
    a.record()
    dgsm.query(atlas, lights, x, out=out)
    b.record()
    torch.cuda.synchronize()
    warm.append(a.elapsed_time(b) * 1e3)
alg = m * 48
print(f"query cold mean {np.mean(ts):.1f} us min {np.min(ts):.1f} us ({alg / np.mean(ts) / 1e3:.0f} GB/s alg); "
      f"warm mean {np.mean(warm):.1f} us min {np.min(warm):.1f}")
