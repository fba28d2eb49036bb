"""Small workloads through every entry point (for compute-sanitizer): cfg1 build
(plan+run, async, bins), query (plain, ordered, chunks, footprint), slab, sort,
transfer, exp epilogue; the band kernel (K = 100), the per-light tile sort
(res 128, 3 lights), dgsm_frame_host and dgsm.FrameStream (graphs, PDL)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2601_01660_b200 import dgsm, synth  # noqa: E402

s = synth.config1()
g = dgsm.to_device(s.gaussians)
x = torch.from_numpy(s.queries).cuda()
A = dgsm.build(g, s.lights, s.res, s.K)
plan = dgsm.BuildPlan(g, s.lights, s.res, s.K)
plan.bins()
ab = dgsm.AsyncBuilder(s.lights, s.res, s.K, s.n, plan.n_keys + 100)
out = torch.empty_like(A)
ab(g, out)
ab2 = dgsm.AsyncBuilder(s.lights, s.res, s.K, s.n, max(plan.n_keys // 3, 1))  # overflow path
ab2(g, out)
T = dgsm.query(A, s.lights, x)
o = dgsm.receiver_order(x)
dgsm.query(A, s.lights, x, order=o)
dgsm.query_chunks([(0, 8, True, A[0, :8].contiguous())], s.lights, x, s.res, s.K)
z, w = dgsm.footprint_stencil()
dgsm.query_footprint(A, s.lights, {k: g[k] for k in ("means", "scales", "rotations")}, z, w)
slab = dgsm.active_slab(x, (0, 0, 3.0, 1.0, 0.0, 6.0), s.lights, s.res, s.K)
dgsm.build(g, s.lights, s.res, s.K, dgsm.Options(slab=slab))
r = synth.random_scene(3, 300, res=32, K=8, L=3, dist=(0.3, 3.0))
dgsm.build(dgsm.to_device(r.gaussians), r.lights, r.res, r.K, dgsm.Options(output_tau=True))
k = torch.randint(0, 2**31 - 1, (5001,), dtype=torch.int32, device="cuda")
dgsm.sort_pairs(k, torch.arange(5001, dtype=torch.int32, device="cuda"), 31)
nr = torch.nn.functional.normalize(torch.randn(1000, 3, device="cuda"), dim=1)
dgsm.sh_transfer(np.ones((3, 16), np.float32), 3, nr, torch.rand(1000, 3, device="cuda"))
dgsm.exp_epilogue(torch.rand(1000, device="cuda"))
b = synth.random_scene(5, 400, res=32, K=100, L=2, dist=(0.3, 3.0), scale=(0.01, 0.5))
dgsm.build(dgsm.to_device(b.gaussians), b.lights, b.res, b.K)
pl = synth.random_scene(7, 400, res=128, K=9, L=3, dist=(0.3, 3.0))
dgsm.build(dgsm.to_device(pl.gaussians), pl.lights, pl.res, pl.K)
fh = {k: torch.from_numpy(np.ascontiguousarray(v, np.float32)).pin_memory() for k, v in s.gaussians.items()}
xh = torch.from_numpy(np.ascontiguousarray(s.queries, np.float32)).pin_memory()
Th = torch.empty(xh.shape[0]).pin_memory()
fr = dgsm.FrameHost(s.lights, s.res, s.K)
fr(fh, xh, Th)
fs = dgsm.FrameStream(s.lights, s.res, s.K, s.n, xh.shape[0], plan.n_keys + 100)
for _ in range(3):
    fs(fh, xh, Th)
fs.wait()
torch.cuda.synchronize()
print("ok")
