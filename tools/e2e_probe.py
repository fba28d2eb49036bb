"""Where the end-to-end frame time goes: H2D bandwidth, device-only step, frame_host."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2601_01660_b200 import dgsm, synth  # noqa: E402

s = synth.config2()
gh = {k: torch.from_numpy(np.ascontiguousarray(v, np.float32)).pin_memory() for k, v in s.gaussians.items()}
rh = torch.from_numpy(s.queries).pin_memory()
Th = torch.empty(rh.shape[0]).pin_memory()
gd = {k: v.cuda() for k, v in gh.items()}


def timeit(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


h2d = timeit(lambda: [gd[k].copy_(gh[k], non_blocking=True) for k in gh])
nb = sum(v.numel() * 4 for v in gh.values())
print(f"H2D gaussians {nb / 1e6:.1f} MB: {h2d:.3f} ms = {nb / h2d / 1e6:.1f} GB/s")
fr = dgsm.FrameHost(s.lights, s.res, s.K)
print(f"frame_host: {timeit(lambda: fr(gh, rh, Th)):.3f} ms")
b = dgsm.Builder(s.lights, s.res, s.K)
out = torch.empty((1, s.K, s.res, s.res), device="cuda")
xq = rh.cuda()
To = torch.empty(rh.shape[0], device="cuda")
print(f"device build+query: {timeit(lambda: (b(gd, out), dgsm.query(out, s.lights, xq, out=To))):.3f} ms")


def span(fn, k=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(k):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / k


print(f"frame_host pipelined: {span(lambda: fr(gh, rh, Th)):.3f} ms/frame")
print(f"device build+query pipelined: {span(lambda: (b(gd, out), dgsm.query(out, s.lights, xq, out=To))):.3f} ms/frame")
print(f"device build only pipelined: {span(lambda: b(gd, out)):.3f} ms/frame")
Tp = torch.empty(rh.shape[0])
print(f"frame_host pipelined, pageable T: {span(lambda: fr(gh, rh, Tp)):.3f} ms/frame")
