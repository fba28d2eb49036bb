"""dgsm.FrameStream (frames back to back from host tensors: uploads on a copy stream,
the sync-free build + query as a CUDA-graph replay per buffer set, T copied back on
a second stream): every frame's T and the last atlas equal the device path's
(dgsm.build + dgsm.query) on the same inputs, for frames with different occluders."""
import numpy as np
import pytest

from paper_2601_01660_b200 import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dg():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2601_01660_b200 import build_ext, dgsm
    build_ext.build()
    dgsm.lib()
    return dgsm


def _pinned(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).pin_memory()


def test_frame_stream_matches_device_path(dg):
    scenes = [synth.random_scene(61 + i, 3000, res=32, K=16, L=2, dist=(0.3, 3.0), scale=(0.01, 0.3),
                                 m_queries=5000) for i in range(5)]
    n = min(s.gaussians["means"].shape[0] for s in scenes)
    m = scenes[0].queries.shape[0]
    lights = scenes[0].lights
    frames = []
    for s in scenes:
        g = {k: v[:n] for k, v in s.gaussians.items()}
        frames.append(({k: _pinned(v) for k, v in g.items()}, _pinned(s.queries[:m]), g, s.queries[:m]))
    P = max(dg.BuildPlan(dg.to_device(f[2]), lights, 32, 16).n_keys for f in frames)
    fs = dg.FrameStream(lights, 32, 16, n, m, int(P * 1.25) + 64)
    outs = []
    for gh, rh, _, _ in frames:
        Th = torch.empty(m).pin_memory()
        fs(gh, rh, Th)
        outs.append(Th)
    fs.wait()
    torch.cuda.synchronize()
    st = fs.status()
    assert not st["overflow"] and st["n_invalid"] == 0
    for (gh, rh, g, q), Th in zip(frames, outs):
        at = dg.build(dg.to_device(g), lights, 32, 16)
        T = dg.query(at, lights, torch.from_numpy(np.ascontiguousarray(q, np.float32)).cuda())
        assert np.abs(Th.numpy() - T.cpu().numpy()).max() <= 1e-6
    assert np.abs(fs.atlas.cpu().numpy() - at.cpu().numpy()).max() <= 1e-6
