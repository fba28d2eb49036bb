"""One launch of the query on Morton-ordered receivers per config (for ncu):
cfg2 (1 M receivers, 512^2 x 64, 1 light) and cfg5 (5.4 M, 2048^2 x 128, 8 lights),
device-random atlases.  argv: configs."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2601_01660_b200 import dgsm, synth  # noqa: E402

for cfg in [int(c) for c in (sys.argv[1:] or ["2", "5"])]:
    s = synth.config2() if cfg == 2 else synth.config5()
    g = torch.Generator(device="cuda").manual_seed(cfg)
    atlas = torch.rand((s.L, s.K, s.res, s.res), generator=g, device="cuda")
    x = torch.from_numpy(s.queries).cuda()
    order = dgsm.receiver_order(x)
    xp = x[order.long()].contiguous()
    torch.cuda.synchronize()
    dgsm.query(atlas, s.lights, xp)
    torch.cuda.synchronize()
    del atlas
    torch.cuda.empty_cache()
