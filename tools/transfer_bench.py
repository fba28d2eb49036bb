"""SH transfer micro-benchmark: n avatar Gaussians x 64x128 directions, degree 3."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2601_01660_b200 import dgsm  # noqa: E402

for n in (100_000, 150_000, 1_000_000):
    rng = np.random.default_rng(1)
    nr = rng.normal(size=(n, 3)); nr /= np.linalg.norm(nr, axis=1, keepdims=True)
    nr = torch.from_numpy(nr.astype(np.float32)).cuda()
    col = torch.rand(n, 3, device="cuda")
    A = rng.normal(0, 0.5, (3, 16)).astype(np.float32); A[:, 0] = 2.5
    for _ in range(3):
        dgsm.sh_transfer(A, 3, nr, col)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(200_000)
        a.record(); dgsm.sh_transfer(A, 3, nr, col); b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = float(np.median(ts))
    ops = n * 64 * 128 * 8
    print(f"n={n}: {ms:.3f} ms  {n / ms * 1e3:.3g} Gaussians/s  {ops / ms / 1e9:.2f} TFLOP/s "
          f"({ops / ms / 1e9 / 37.22 * 100:.1f} % of 37.2)")
