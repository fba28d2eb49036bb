"""Parity at BASELINE.json's full cfg2 size (1.1 M Gaussians, 1 light, 512^2 x 64,
1 M receivers), in the launch configuration bench.py times, against the oracle
on what it can compute in seconds: the whole binning (bit-exact), the atlas on a
strided sample of tiles, and the query of every receiver on a seeded atlas of
the same shape."""
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


@pytest.fixture(scope="module")
def cfg2():
    return synth.config2()


def test_cfg2_full_binning_bit_exact(dg, oracle_mod, cfg2):
    s = cfg2
    plan = dg.BuildPlan(dg.to_device(s.gaussians), s.lights, s.res, s.K)
    (l, t, d, i), _ = plan.bins()
    want = oracle_mod.bin_entries(s.gaussians["means"], s.gaussians["scales"], s.gaussians["rotations"],
                                  s.lights["position"], s.res)
    assert plan.n_keys == len(want[0]) > 4_000_000
    for a, b in zip((l, t, d, i), want):
        assert np.array_equal(a.cpu().numpy().astype(np.uint32), b)


def test_cfg2_full_build_sampled_tiles(dg, oracle_mod, cfg2):
    """Every 97th (light, tile) of the full atlas, all 64 texels x 64 shells."""
    s = cfg2
    T = dg.build(dg.to_device(s.gaussians), s.lights, s.res, s.K).cpu().numpy()
    To, _ = oracle_mod.build(s.gaussians, s.lights, s.res, s.K, tile_stride=97)
    m = ~np.isnan(To)
    assert m.sum() >= 40 * 64 * s.K
    assert np.abs(T[m] - To[m]).max() <= 1e-4
    assert (T >= 0).all() and (T <= 1).all() and (np.diff(T, axis=1) <= 1e-6).all()


def test_cfg2_full_query_seeded_atlas(dg, oracle_mod, cfg2):
    """All 1 M receivers of cfg2 on a seeded 512^2 x 64 atlas."""
    s = cfg2
    atlas = synth.random_atlas(2, 1, s.K, s.res)
    got = dg.query(torch.from_numpy(atlas).cuda(), s.lights, torch.from_numpy(s.queries).cuda()).cpu().numpy()
    want = oracle_mod.query(atlas.astype(np.float64), s.lights, s.queries)
    assert np.abs(got - want).max() <= 2e-6


def test_multilight_binning_bit_exact_multi_tile_scan(dg, oracle_mod, cfg2):
    """4 lights x 1.1 M Gaussians: the key-count scan spans > 1024 x 4096 entries, so
    every scan block walks several tiles (the large-n path of scan.cu); scales
    shrunk x0.3 so the oracle binning stays in seconds."""
    s = cfg2
    g = dict(s.gaussians)
    g["scales"] = (g["scales"] * np.float32(0.3)).astype(np.float32)
    pos = np.array([[3.4, 2.2, 2.6], [1.0, 1.0, 2.8], [5.0, 4.0, 2.5], [3.0, 0.5, 1.5]], np.float32)
    lights = {"position": pos, "t_max": np.full(4, 6.0, np.float32)}
    plan = dg.BuildPlan(dg.to_device(g), lights, s.res, s.K)
    (l, t, d, i), _ = plan.bins()
    want = oracle_mod.bin_entries(g["means"], g["scales"], g["rotations"], pos, s.res)
    assert 4 * len(g["means"]) > 1024 * 4096
    assert plan.n_keys == len(want[0])
    for a, b in zip((l, t, d, i), want):
        assert np.array_equal(a.cpu().numpy().astype(np.uint32), b)
