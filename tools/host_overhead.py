"""Host-side overhead breakdown of one DGSM step (diagnostic, GPU box)."""
import os
import subprocess
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_01660_b200 import dgsm, synth  # noqa: E402


def main():
    s = synth.config2()
    g = dgsm.to_device(s.gaussians)
    xq = torch.from_numpy(s.queries).cuda()
    atlas = torch.empty((s.L, s.K, s.res, s.res), device="cuda")
    T = torch.empty(xq.shape[0], device="cuda")
    for smi in (False, True):
        proc = None
        if smi:
            proc = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv", "-lms", "100"],
                                    stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        rows = []
        for it in range(15):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            plan = dgsm.BuildPlan(g, s.lights, s.res, s.K)
            t1 = time.perf_counter()
            plan.run(out=atlas)
            t2 = time.perf_counter()
            dgsm.query(atlas, s.lights, xq, out=T)
            t3 = time.perf_counter()
            torch.cuda.synchronize()
            t4 = time.perf_counter()
            rows.append((t1 - t0, t2 - t1, t3 - t2, t4 - t3, t4 - t0))
        if proc:
            proc.terminate()
        r = np.median(np.array(rows[3:]), axis=0) * 1e3
        print(f"nvidia-smi={smi}: plan {r[0]:.3f} ms  run(enqueue) {r[1]:.3f}  query(enqueue) {r[2]:.3f}  "
              f"drain {r[3]:.3f}  total {r[4]:.3f}")


if __name__ == "__main__":
    main()
