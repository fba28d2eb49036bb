"""Where the end-to-end frame time goes (cfg2), frames back to back over K frames:
frame_host (plan + host sync + run), and a sync-free pipeline built from the
public pieces (copy-stream uploads into alternating buffers, AsyncBuilder, query,
T copied back on the compute stream) to size what a sync-free frame_host would gain."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2601_01660_b200 import dgsm, synth  # noqa: E402

K = 20
s = synth.config2()
gh = {k: torch.from_numpy(np.ascontiguousarray(v, np.float32)).pin_memory() for k, v in s.gaussians.items()}
rh = torch.from_numpy(s.queries).pin_memory()
Th = torch.empty(rh.shape[0]).pin_memory()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def span(fn, k=K, with_flush=False):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fl = []
    a.record()
    for _ in range(k):
        if with_flush:
            x, y = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            x.record(); flush.zero_(); y.record(); fl.append((x, y))
        fn()
    b.record()
    torch.cuda.synchronize()
    return (a.elapsed_time(b) - sum(x.elapsed_time(y) for x, y in fl)) / k


gd = {k: v.cuda() for k, v in gh.items()}
t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
for _ in range(3):
    t0.record(); [gd[k].copy_(gh[k], non_blocking=True) for k in gh]; t1.record(); torch.cuda.synchronize()
nb = sum(v.numel() * 4 for v in gh.values()) + rh.numel() * 4
print(f"H2D {nb / 1e6:.1f} MB: {t0.elapsed_time(t1):.3f} ms (gaussians only)")

fr = dgsm.FrameHost(s.lights, s.res, s.K)
print(f"frame_host back to back: {span(lambda: fr(gh, rh, Th)):.3f} ms/frame; with flush (bench): {span(lambda: fr(gh, rh, Th), with_flush=True):.3f}")

P = dgsm.BuildPlan(gd, s.lights, s.res, s.K).n_keys
cap = int(P * 1.25)
ab = dgsm.AsyncBuilder(s.lights, s.res, s.K, gd["means"].shape[0], cap)
atlas = torch.empty((1, s.K, s.res, s.res), device="cuda")
bufs = [({k: torch.empty_like(v) for k, v in gd.items()}, torch.empty_like(rh, device="cuda")) for _ in range(2)]
Td = torch.empty(rh.shape[0], device="cuda")
cs = torch.cuda.Stream()
ev_up = [torch.cuda.Event() for _ in range(2)]
ev_free = [torch.cuda.Event() for _ in range(2)]
for e in ev_free:
    e.record()
state = {"i": 0}


def async_frame():
    k = state["i"] & 1
    state["i"] += 1
    g, x = bufs[k]
    cs.wait_event(ev_free[k])
    with torch.cuda.stream(cs):
        for name in gh:
            g[name].copy_(gh[name], non_blocking=True)
        x.copy_(rh, non_blocking=True)
        ev_up[k].record(cs)
    cur = torch.cuda.current_stream()
    cur.wait_event(ev_up[k])
    ab(g, atlas)
    dgsm.query(atlas, s.lights, x, out=Td)
    Th.copy_(Td, non_blocking=True)
    ev_free[k].record(cur)


print(f"sync-free pipeline back to back: {span(async_frame):.3f} ms/frame; with flush: {span(async_frame, with_flush=True):.3f}")
print("status", ab.status(), "P", P)
dev = lambda: (ab(gd, atlas), dgsm.query(atlas, s.lights, bufs[0][1], out=Td))
print(f"device only (async build + query), back to back: {span(dev):.3f}; with flush: {span(dev, with_flush=True):.3f}")

dev_t = lambda: (ab(gd, atlas), dgsm.query(atlas, s.lights, bufs[0][1], out=Td), Th.copy_(Td, non_blocking=True))
print(f"device + T copy back, back to back: {span(dev_t):.3f}")
big = torch.empty(64 << 20, dtype=torch.uint8).pin_memory()
bigd = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")


def dev_with_h2d():
    with torch.cuda.stream(cs):
        bigd.copy_(big, non_blocking=True)
    dev()


print(f"device only with a concurrent 67 MB H2D each frame: {span(dev_with_h2d):.3f}")
torch.cuda.synchronize()
t0.record(cs)
with torch.cuda.stream(cs):
    for _ in range(10):
        bigd.copy_(big, non_blocking=True)
t1.record(cs)
torch.cuda.synchronize()
print(f"H2D alone: {10 * big.numel() / t0.elapsed_time(t1) / 1e6:.1f} GB/s")
