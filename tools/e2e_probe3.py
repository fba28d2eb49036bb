"""Does a concurrent host->device upload slow the build (cfg2)?  Per frame (synchronised):
the sync-free build + query alone, and with the next frame's 60 MB upload started
at the same time on a copy stream; the accumulation kernel timed by the library's
events, the rest by difference."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2601_01660_b200 import dgsm, synth  # noqa: E402

s = synth.config2()
gh = {k: torch.from_numpy(np.ascontiguousarray(v, np.float32)).pin_memory() for k, v in s.gaussians.items()}
rh = torch.from_numpy(s.queries).pin_memory()
gd = {k: v.cuda() for k, v in gh.items()}
gd2 = {k: torch.empty_like(v) for k, v in gd.items()}
xq = rh.cuda()
xq2 = torch.empty_like(xq)
P = dgsm.BuildPlan(gd, s.lights, s.res, s.K).n_keys
ab = dgsm.AsyncBuilder(s.lights, s.res, s.K, gd["means"].shape[0], int(P * 1.25))
atlas = torch.empty((1, s.K, s.res, s.res), device="cuda")
Td = torch.empty(xq.shape[0], device="cuda")
cs = torch.cuda.Stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def frame(upload, when):
    flush.zero_()
    torch.cuda.synchronize()
    a, b, ea, eb, u0, u1 = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    for e in (ea, eb, u0, u1):  # created now (torch creates events lazily on record)
        e.record()
    torch.cuda.synchronize()
    dgsm.set_accumulate_events(ea, eb)
    a.record()
    if upload and when == "start":
        cs.wait_event(a)
        with torch.cuda.stream(cs):
            u0.record(cs)
            for k in gh:
                gd2[k].copy_(gh[k], non_blocking=True)
            xq2.copy_(rh, non_blocking=True)
            u1.record(cs)
    ab(gd, atlas)
    dgsm.query(atlas, s.lights, xq, out=Td)
    b.record()
    torch.cuda.synchronize()
    dgsm.set_accumulate_events(None, None)
    return a.elapsed_time(b), ea.elapsed_time(eb), (u0.elapsed_time(u1) if upload else 0.0)


for upload in (False, True, False, True):
    r = np.array([frame(upload, "start") for _ in range(12)][2:])
    tot, acc, up = np.median(r, axis=0)
    print(f"upload={upload}: frame {tot:.3f} ms, a6 {acc:.3f}, rest {tot - acc:.3f}, upload {up:.3f}")
