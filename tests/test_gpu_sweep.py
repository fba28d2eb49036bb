"""Seeded sweep over the build's shape parameters against the oracle: atlas
resolution (one tile .. 256 tiles), shell count (1 .. 130: single-table and band
kernels, K not a multiple of the combine's 4-shell groups), light count (1 .. 8:
the light bits of the keys; res 128 with 2+ lights takes the per-light tile sort),
Gaussian count (1 .. 3000: multi-chunk tiles at the small adaptive chunk), and
record staging.  Each case: binning bit-exact and |T - T_oracle| <= 1e-4."""
import numpy as np
import pytest

from paper_2601_01660_b200 import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL_T = 1e-4

CASES = [  # (seed, n, res, K, L, staging)
    (1, 1, 8, 1, 1, "reg"),
    (2, 50, 8, 3, 2, "tma"),
    (3, 500, 16, 17, 1, "reg"),
    (4, 3000, 16, 5, 3, "tma"),
    (5, 800, 64, 64, 1, "tma"),
    (6, 800, 64, 65, 2, "reg"),
    (7, 400, 128, 9, 2, "reg"),
    (8, 1500, 128, 33, 3, "tma"),
    (9, 300, 128, 130, 3, "reg"),
    (10, 200, 32, 12, 8, "reg"),
    (11, 2000, 128, 16, 8, "tma"),
    (12, 60, 256, 7, 1, "reg"),
]


@pytest.fixture(scope="module")
def dg():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2601_01660_b200 import build_ext, dgsm
    build_ext.build()
    dgsm.lib()
    return dgsm


@pytest.mark.parametrize("seed,n,res,K,L,staging", CASES)
def test_sweep(dg, oracle_mod, monkeypatch, seed, n, res, K, L, staging):
    monkeypatch.setenv("DGSM_ACC_STAGING", staging)
    s = synth.random_scene(100 + seed, n, res=res, K=K, L=L, dist=(0.2, 3.0), scale=(0.005, 0.6))
    g = dg.to_device(s.gaussians)
    plan = dg.BuildPlan(g, s.lights, s.res, s.K)
    (l, t, d, i), _ = plan.bins()
    want = oracle_mod.bin_entries(s.gaussians["means"], s.gaussians["scales"], s.gaussians["rotations"],
                                  s.lights["position"], s.res)
    assert plan.n_keys == len(want[0])
    for name, a, b in zip(("light", "tile", "depth", "index"), (l, t, d, i), want):
        assert np.array_equal(a.cpu().numpy().astype(np.uint32), b), name
    T = dg.build(g, s.lights, s.res, s.K).cpu().numpy()
    To, _ = oracle_mod.build(s.gaussians, s.lights, s.res, s.K)
    assert np.abs(T - To).max() <= TOL_T
    # the sync-free build gives the same atlas (capacity = P: same chunking)
    if plan.n_keys > 0:
        ab = dg.AsyncBuilder(s.lights, s.res, s.K, s.gaussians["means"].shape[0], plan.n_keys)
        out = torch.empty_like(torch.from_numpy(T)).cuda()
        ab(g, out)
        st = ab.status()
        assert st["n_keys"] == plan.n_keys and not st["overflow"]
        assert np.abs(out.cpu().numpy() - To).max() <= TOL_T


def test_sweep_slab_per_light_sort(dg, oracle_mod):
    """ROI slab at res 128 with 3 lights (the per-light tile sort over the
    slab-restricted key segments): binning = the oracle's entries on the active
    tiles, the slab build <= 1e-4 against the oracle's slab build."""
    s = synth.random_scene(131, 1200, res=128, K=20, L=3, dist=(0.3, 3.0), scale=(0.01, 0.4))
    rng = np.random.default_rng(131)
    rec = rng.uniform(-3, 3, (2000, 3)).astype(np.float32)
    roi = (0.2, -0.1, 0.3, 1.0, -0.8, 0.9)
    slab = dg.active_slab(torch.from_numpy(rec).cuda(), roi, s.lights, s.res, s.K)
    g = dg.to_device(s.gaussians)
    T = dg.build(g, s.lights, s.res, s.K, dg.Options(slab=slab)).cpu().numpy()
    mask, kr, inside = oracle_mod.active_slab(rec, roi, s.lights, s.res, s.K)
    assert inside > 0
    To, _ = oracle_mod.build(s.gaussians, s.lights, s.res, s.K, slab=(mask, kr))
    assert np.abs(T - To).max() <= TOL_T
    plan = dg.BuildPlan(g, s.lights, s.res, s.K, dg.Options(slab=slab))
    (l, t, d, i), _ = plan.bins()
    want = oracle_mod.bin_entries(s.gaussians["means"], s.gaussians["scales"], s.gaussians["rotations"],
                                  s.lights["position"], s.res)
    tile_on = mask.reshape(s.L, s.res // 8, 8, s.res // 8, 8).any(axis=(2, 4)).reshape(s.L, -1)
    keep = tile_on[want[0].astype(np.int64), want[1].astype(np.int64)]
    want = [w[keep] for w in want]
    assert plan.n_keys == len(want[0]) and 0 < plan.n_keys
    for a, b in zip((l, t, d, i), want):
        assert np.array_equal(a.cpu().numpy().astype(np.uint32), b)
