"""The sync-free build (dgsm_build_async): the same atlas as dgsm_build without
a host synchronisation, bit for bit when the key capacity equals P, within the
oracle tolerance otherwise; the overflow contract; a frame (build + query)
captured once in a CUDA graph and replayed on new occluder data; and the
DGSM_VALIDATE data check."""
import numpy as np
import pytest

from paper_2601_01660_b200 import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL_T = 1e-4


@pytest.fixture(scope="module")
def dg():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2601_01660_b200 import build_ext, dgsm
    build_ext.build()
    dgsm.lib()
    return dgsm


def _depth_scene(name, n, d0, d1, seed):
    """Gaussians around one light at the origin with light distances in [d0, d1]
    (d0 == d1: six axis points at one exact distance): the sync-free build's depth
    digits, planned on the device from the depth range, at 0 and ~9 significant bits."""
    rng = np.random.Generator(np.random.PCG64(4242 + seed))
    if d0 == d1:
        axes = np.array([[1, 0, 0], [-1, 0, 0], [0, 1, 0], [0, -1, 0], [0, 0, 1], [0, 0, -1]], np.float64)
        v = axes[np.arange(n) % 6]
    else:
        v = rng.standard_normal((n, 3))
        v /= np.linalg.norm(v, axis=1, keepdims=True)
    mu = v * rng.uniform(d0, d1, n)[:, None] if d0 != d1 else v * d0
    g = synth._gaussians(mu, np.exp(rng.uniform(np.log(0.05), np.log(0.4), (n, 3))),
                         synth.random_quaternions(rng, n), rng.uniform(0.1, 0.9, n))
    lights = dict(position=np.zeros((1, 3), np.float32), t_max=np.array([4.0], np.float32))
    return synth.Scene(name, g, lights, 32, 8, g["means"].copy())


SCENES = {
    "equal-depth": lambda: _depth_scene("equal-depth", 60, 2.0, 2.0, 0),
    "narrow-depth": lambda: _depth_scene("narrow-depth", 500, 2.0, 2.0001, 1),
    "cfg1": lambda: synth.config1(),
    "random-3lights": lambda: synth.random_scene(11, 400, res=32, K=8, L=3, dist=(0.3, 3.0), scale=(0.01, 0.5)),
    "cfg2-small": lambda: synth.config2(scale=0.004, res=64, K=16),
    "single-gaussian": lambda: synth.Scene("one", {k: v[:1] for k, v in synth.config1().gaussians.items()},
                                           synth.config1().lights, 64, 16, synth.config1().queries[:10]),
}


@pytest.mark.parametrize("name", sorted(SCENES))
def test_async_equals_build(dg, oracle_mod, name):
    s = SCENES[name]()
    g = dg.to_device(s.gaussians)
    ref = dg.build(g, s.lights, s.res, s.K)
    P = dg.BuildPlan(g, s.lights, s.res, s.K).n_keys
    out = torch.empty_like(ref)
    ab = dg.AsyncBuilder(s.lights, s.res, s.K, s.n, max(P, 1))
    ab(g, out)
    st = ab.status()
    assert st["n_keys"] == P and not st["overflow"] and st["n_invalid"] == 0
    assert torch.equal(out, ref)  # same chunking (capacity == P): bit for bit
    ab2 = dg.AsyncBuilder(s.lights, s.res, s.K, s.n, 3 * P + 1000)
    ab2(g, out)
    To, _ = oracle_mod.build(s.gaussians, s.lights, s.res, s.K)
    assert np.abs(out.cpu().numpy() - To).max() <= TOL_T


def test_async_overflow(dg):
    s = synth.config1()
    g = dg.to_device(s.gaussians)
    P = dg.BuildPlan(g, s.lights, s.res, s.K).n_keys
    ab = dg.AsyncBuilder(s.lights, s.res, s.K, s.n, P // 2)
    out = torch.zeros((s.L, s.K, s.res, s.res), device="cuda")
    ab(g, out)
    st = ab.status()
    assert st["overflow"] and st["n_keys"] == P
    assert torch.all(out == 1.0)  # invalid build: nothing accumulated, T = 1, no out-of-bounds write


def test_frame_graph_capture(dg, oracle_mod):
    """Build + query captured once in a CUDA graph; replays after copying the next
    frames' occluders (the walking avatar of cfg4) into the captured buffers."""
    frames = [synth.config4(frame=f, scale=0.01) for f in (0, 30, 60)]
    s0 = frames[0]
    n = s0.n
    g = dg.to_device(s0.gaussians)
    x = torch.from_numpy(s0.queries[:5000]).cuda()
    P = max(dg.BuildPlan(dg.to_device(f.gaussians), f.lights, f.res, f.K).n_keys for f in frames)
    ab = dg.AsyncBuilder(s0.lights, s0.res, s0.K, n, int(1.5 * P))
    atlas = torch.empty((1, s0.K, s0.res, s0.res), device="cuda")
    T = torch.empty(x.shape[0], device="cuda")
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):  # warm-up on the capture stream
        ab(g, atlas)
        dg.query(atlas, s0.lights, x, out=T)
    torch.cuda.current_stream().wait_stream(side)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        ab(g, atlas)
        dg.query(atlas, s0.lights, x, out=T)
    for f in frames[::-1]:
        for k, v in dg.to_device(f.gaussians).items():
            g[k].copy_(v)
        graph.replay()
        torch.cuda.synchronize()
        assert not ab.status()["overflow"]
        ref = dg.build(dg.to_device(f.gaussians), f.lights, f.res, f.K)
        To, _ = oracle_mod.build(f.gaussians, f.lights, f.res, f.K)
        assert np.abs(atlas.cpu().numpy() - To).max() <= TOL_T
        assert (T - dg.query(ref, f.lights, x)).abs().max().item() <= 1e-5


def test_validate_flag(dg):
    s = synth.config1()
    g = {k: v.copy() for k, v in s.gaussians.items()}
    g["means"][17, 1] = np.nan
    g["scales"][300, 2] = 0.0
    gd = dg.to_device(g)
    with pytest.raises(dg.DgsmError, match="EDATA.*2 invalid.*index 17"):
        dg.BuildPlan(gd, s.lights, s.res, s.K, dg.Options(validate=True))
    dg.BuildPlan(dg.to_device(s.gaussians), s.lights, s.res, s.K, dg.Options(validate=True))  # valid data passes
    ab = dg.AsyncBuilder(s.lights, s.res, s.K, s.n, 100000, dg.Options(validate=True))
    ab(gd, torch.empty((1, s.K, s.res, s.res), device="cuda"))
    assert ab.status()["n_invalid"] == 2


def test_async_empty_and_slab(dg, oracle_mod):
    """n = 0 (T == 1 exactly, P = 0) and a ROI-slab build through the sync-free path."""
    s = synth.random_scene(11, 400, res=32, K=8, L=3, dist=(0.3, 3.0), scale=(0.01, 0.5))
    empty = {k: v[:0] for k, v in s.gaussians.items()}
    ab = dg.AsyncBuilder(s.lights, s.res, s.K, 0, 1)
    out = torch.zeros((s.L, s.K, s.res, s.res), device="cuda")
    ab(dg.to_device(empty), out)
    assert torch.all(out == 1.0) and ab.status()["n_keys"] == 0 and not ab.status()["overflow"]
    g = dg.to_device(s.gaussians)
    x = torch.from_numpy(s.queries).cuda()
    slab = dg.active_slab(x, (0.0, 0.0, 0.0, 2.0, -1.0, 1.0), s.lights, s.res, s.K)
    opts = dg.Options(slab=slab)
    ref = dg.build(g, s.lights, s.res, s.K, opts)
    P = dg.BuildPlan(g, s.lights, s.res, s.K, opts).n_keys
    ab = dg.AsyncBuilder(s.lights, s.res, s.K, s.n, P, opts)
    ab(g, out)
    assert torch.equal(out, ref) and ab.status()["n_keys"] == P


def test_multilight_graph_capture(dg, oracle_mod):
    """A 5-light sync-free build captured in a CUDA graph: the per-light binning
    chains fork onto the library's side streams (4 lanes, light 4 shares lane 0)
    and join inside the capture; replays on new Gaussians match the oracle."""
    scenes = [synth.random_scene(90 + i, 1500, res=64, K=12, L=5, dist=(0.3, 3.0), scale=(0.01, 0.3)) for i in range(2)]
    n = min(s.gaussians["means"].shape[0] for s in scenes)
    s0 = scenes[0]
    gs = [{k: v[:n] for k, v in s.gaussians.items()} for s in scenes]
    P = max(dg.BuildPlan(dg.to_device(g), s0.lights, s0.res, s0.K).n_keys for g in gs)
    ab = dg.AsyncBuilder(s0.lights, s0.res, s0.K, n, int(P * 1.25) + 64)
    g = dg.to_device(gs[0])
    atlas = torch.empty((5, s0.K, s0.res, s0.res), device="cuda")
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        ab(g, atlas)
    torch.cuda.current_stream().wait_stream(side)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        ab(g, atlas)
    for gh in gs[::-1]:
        for k, v in dg.to_device(gh).items():
            g[k].copy_(v)
        graph.replay()
        torch.cuda.synchronize()
        assert not ab.status()["overflow"]
        To, _ = oracle_mod.build(gh, s0.lights, s0.res, s0.K)
        assert np.abs(atlas.cpu().numpy() - To).max() <= TOL_T
