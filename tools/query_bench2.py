"""Query micro-benchmark at cfg2 and cfg5 shapes (device-random atlases; the
receivers are the configs' scene centres in generation order), L2 flushed
before each timed launch: raw order, receiver_order cost, ordered query,
and the query on receivers pre-permuted into that order."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2601_01660_b200 import dgsm, synth  # noqa: E402

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timed(fn, reps=10):
    ts = []
    for i in range(reps + 2):
        flush.zero_()
        torch.cuda._sleep(400_000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(a.elapsed_time(b) * 1e3)
    return float(np.median(ts)), float(np.min(ts))


for cfg in [int(c) for c in (sys.argv[1:] or ["2", "5"])]:
    t0 = time.time()
    s = synth.config2() if cfg == 2 else synth.config5()
    L, K, res = s.L, s.K, s.res
    g = torch.Generator(device="cuda").manual_seed(cfg)
    atlas = torch.rand((L, K, res, res), generator=g, device="cuda")
    x = torch.from_numpy(s.queries).cuda()
    m = x.shape[0]
    out = torch.empty(m, device="cuda")
    out2 = torch.empty(m, device="cuda")
    raw = timed(lambda: dgsm.query(atlas, s.lights, x, out=out))
    order = dgsm.receiver_order(x)
    ordt = timed(lambda: dgsm.receiver_order(x, out=order))
    qo = timed(lambda: dgsm.query(atlas, s.lights, x, out=out2, order=order))
    same = torch.equal(out, out2)
    xp = x[order.long()].contiguous()
    out3 = torch.empty(m, device="cuda")
    pre = timed(lambda: dgsm.query(atlas, s.lights, xp, out=out3))
    same3 = torch.equal(out3, out[order.long()])
    perm_ok = torch.equal(torch.sort(order.long())[0], torch.arange(m, device="cuda"))
    alg = m * (16 + 32 * L)
    print(f"cfg{cfg}: m={m} L={L} atlas {atlas.numel()*4/2**30:.1f} GiB (setup {time.time()-t0:.0f}s)")
    print(f"  raw order       {raw[0]:9.1f} us (min {raw[1]:.1f})  alg {alg/raw[0]/1e3:.0f} GB/s")
    print(f"  receiver_order  {ordt[0]:9.1f} us")
    print(f"  ordered query   {qo[0]:9.1f} us  (+order {qo[0]+ordt[0]:.1f})  bit-identical={same} perm={perm_ok}")
    print(f"  pre-permuted    {pre[0]:9.1f} us  bit-identical={same3}")
    del atlas
    torch.cuda.empty_cache()
