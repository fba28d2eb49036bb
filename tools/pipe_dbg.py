import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2601_01660_b200 import dgsm, synth
frames = [synth.random_scene(seed, 3000, res=32, K=16, L=1, dist=(0.3, 3.0), scale=(0.01, 0.3)) for seed in (51, 52, 53)]
s0 = frames[0]
for mode in ("sync", "nosync"):
    fr = dgsm.FrameHost(s0.lights, s0.res, s0.K)
    outs = []
    for s in frames:
        gh = {k: torch.from_numpy(np.ascontiguousarray(v, np.float32)).pin_memory() for k, v in s.gaussians.items()}
        rh = torch.from_numpy(np.ascontiguousarray(s.queries, np.float32)).pin_memory()
        Th = torch.empty(rh.shape[0]).pin_memory()
        at = fr(gh, rh, Th).clone()
        if mode == "sync": torch.cuda.synchronize()
        outs.append((rh, Th, at, fr.wss[0].data_ptr()))
    torch.cuda.synchronize()
    for s, (rh, Th, at, wsp) in zip(frames, outs):
        at2 = dgsm.build(dgsm.to_device(s.gaussians), s0.lights, s0.res, s0.K)
        T2 = dgsm.query(at2, s0.lights, rh.cuda()).cpu()
        bad = (Th != T2).nonzero().flatten()
        print(mode, torch.equal(at, at2), len(bad), bad[:5].tolist(), hex(wsp))
