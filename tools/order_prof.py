"""receiver_order at cfg5 scale (5.4 M receivers), a few calls (for an ncu launch list)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2601_01660_b200 import dgsm, synth  # noqa: E402

s = synth.config5(scale=float(sys.argv[1]) if len(sys.argv) > 1 else 1.0)
x = torch.from_numpy(s.queries).cuda()
o = dgsm.receiver_order(x)
for _ in range(3):
    dgsm.receiver_order(x, out=o)
torch.cuda.synchronize()
