"""cfg2 step (sync-free build + query) launched on a stream vs replayed as one CUDA graph,
L2 flushed before each step: how much of the step is launch overhead / inter-kernel gaps."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2601_01660_b200 import dgsm, synth  # noqa: E402

s = synth.config2()
gd = dgsm.to_device(s.gaussians)
xq = torch.from_numpy(s.queries).cuda()
P = dgsm.BuildPlan(gd, s.lights, s.res, s.K).n_keys
ab = dgsm.AsyncBuilder(s.lights, s.res, s.K, gd["means"].shape[0], int(P * 1.25))
atlas = torch.empty((1, s.K, s.res, s.res), device="cuda")
Td = torch.empty(xq.shape[0], device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def step():
    ab(gd, atlas)
    dgsm.query(atlas, s.lights, xq, out=Td)


def timed(fn, k=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(k):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts)), float(np.min(ts))


print("stream launches: median %.4f min %.4f ms" % timed(step))
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    step()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=st):
    step()
print("graph replay:    median %.4f min %.4f ms" % timed(g.replay))
