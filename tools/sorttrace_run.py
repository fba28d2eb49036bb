import sys
sys.path.insert(0, '.')
import torch
from paper_2601_01660_b200 import dgsm, synth
s = synth.config2()
g = dgsm.to_device(s.gaussians)
for _ in range(2):
    dgsm.build(g, s.lights, s.res, s.K)
torch.cuda.synchronize()
