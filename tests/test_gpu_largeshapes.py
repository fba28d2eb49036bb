"""Parity at the shapes of BASELINE.json cfg3 and cfg5 ("every 61st
tile of every light ... binning parity covers all keys"), in the launch
configuration bench.py times:

* cfg3 exactly as bench.py --config 3 builds it (3 M Gaussians, 4 lights,
  1024^2 x 64): the whole binning (33.6 M keys) bit-exact, the atlas on every
  61st (light, tile) within 1e-4;
* a cfg5-shaped scene (the cfg5 hall at 10 % of its Gaussians: 2048^2 x 128,
  8 lights): 16-bit tile keys (two full 8-bit onesweep passes), 524 288
  (light, tile) pairs (the multi-kernel work-unit builder above 16 K tiles),
  K = 128 — binning bit-exact, the atlas on every 61st (light, tile) within 1e-4
  with both record stagings (TMA bulk copies and registers) forced;
* the onesweep sort itself (a4) against numpy's stable argsort for key widths
  1..32 bits, ragged partition tails and degenerate key distributions.
"""
import os

import numpy as np
import pytest

from paper_2601_01660_b200 import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL_T = 1e-4
STRIDE = 61


@pytest.fixture(scope="module")
def dg():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2601_01660_b200 import build_ext, dgsm
    build_ext.build()
    dgsm.lib()
    return dgsm


def tiles_of(atlas: "torch.Tensor", items: np.ndarray) -> np.ndarray:
    """[n, K, 8, 8] texels of the (light, tile) items of a device atlas [L, K, H, W]."""
    L, K, H, W = atlas.shape
    TW = W // 8
    v = atlas.view(L, K, H // 8, 8, TW, 8).permute(0, 2, 4, 1, 3, 5)
    it = torch.from_numpy(items.astype(np.int64)).to(atlas.device)
    nt = (H // 8) * TW
    l, t = it // nt, it % nt
    return v[l, t // TW, t % TW].cpu().numpy()


def check_bins(dg, oracle_mod, s, plan):
    (l, t, d, i), (ts, te) = plan.bins()
    want = oracle_mod.bin_entries(s.gaussians["means"], s.gaussians["scales"], s.gaussians["rotations"],
                                  s.lights["position"], s.res)
    assert plan.n_keys == len(want[0])
    for name, a, b in zip(("light", "tile", "depth", "index"), (l, t, d, i), want):
        a = a.cpu().numpy().astype(np.uint32)
        assert np.array_equal(a, b), f"{name} differs at {np.nonzero(a != b)[0][:10]}"
    # tile ranges
    nt = (s.res // 8) ** 2
    g = want[0].astype(np.int64) * nt + want[1].astype(np.int64)
    wts = np.zeros(s.L * nt, np.int64)
    wte = np.zeros(s.L * nt, np.int64)
    starts = np.r_[0, np.nonzero(np.diff(g))[0] + 1]
    wts[g[starts]] = starts
    wte[g[starts]] = np.r_[starts[1:], len(g)]
    assert np.array_equal(ts.cpu().numpy(), wts) and np.array_equal(te.cpu().numpy(), wte)
    return want


# ------------------------------------------------------------------- cfg3
@pytest.fixture(scope="module")
def cfg3():
    return synth.config3()


def test_cfg3_full_binning_bit_exact(dg, oracle_mod, cfg3):
    s = cfg3
    plan = dg.BuildPlan(dg.to_device(s.gaussians), s.lights, s.res, s.K)
    assert plan.plan.tile_bits == 14 and plan.n_keys > 30_000_000
    check_bins(dg, oracle_mod, s, plan)


def test_cfg3_build_every_61st_tile(dg, oracle_mod, cfg3):
    s = cfg3
    out = torch.empty((s.L, s.K, s.res, s.res), dtype=torch.float32, device="cuda")
    dg.Builder(s.lights, s.res, s.K)(dg.to_device(s.gaussians), out)  # bench.py's entry point
    items = np.arange(0, s.L * (s.res // 8) ** 2, STRIDE)
    To, _ = oracle_mod.build_tiles(s.gaussians, s.lights, s.res, s.K, items)
    T = tiles_of(out, items)
    err = np.abs(T - To).max()
    assert err <= TOL_T, err
    assert (T >= 0).all() and (T <= 1).all()


# ------------------------------------------------------------- cfg5 shape
@pytest.fixture(scope="module")
def cfg5s():
    return synth.config5(scale=0.1)


def test_cfg5_shape_binning_bit_exact(dg, oracle_mod, cfg5s):
    s = cfg5s
    plan = dg.BuildPlan(dg.to_device(s.gaussians), s.lights, s.res, s.K)
    # 16-bit tile keys: two full 8-bit onesweep passes; 8 x 65536 (light, tile) pairs
    assert plan.plan.tile_bits == 16 and s.L * (s.res // 8) ** 2 > 65536
    assert plan.n_keys > 10_000_000
    check_bins(dg, oracle_mod, s, plan)


@pytest.mark.parametrize("staging", ["tma", "reg"])
def test_cfg5_shape_build_every_61st_tile(dg, oracle_mod, cfg5s, staging, monkeypatch):
    s = cfg5s
    monkeypatch.setenv("DGSM_ACC_STAGING", staging)
    out = torch.empty((s.L, s.K, s.res, s.res), dtype=torch.float32, device="cuda")
    dg.Builder(s.lights, s.res, s.K)(dg.to_device(s.gaussians), out)
    items = np.arange(0, s.L * (s.res // 8) ** 2, STRIDE)
    To, _ = oracle_mod.build_tiles(s.gaussians, s.lights, s.res, s.K, items)
    T = tiles_of(out, items)
    err = np.abs(T - To).max()
    assert err <= TOL_T, err
    del out
    torch.cuda.empty_cache()


def test_cfg5_shape_sync_free_build_every_61st_tile(dg, oracle_mod, cfg5s):
    """The sync-free build at the cfg5 shape: one onesweep over all 8 lights'
    (3 + 16)-bit keys (three passes, the top one with 3 light bits) instead of the
    planned build's per-light tile sorts, capacity 1.25 P; every 61st tile <= 1e-4."""
    s = cfg5s
    g = dg.to_device(s.gaussians)
    P = dg.BuildPlan(g, s.lights, s.res, s.K).n_keys
    ab = dg.AsyncBuilder(s.lights, s.res, s.K, s.gaussians["means"].shape[0], int(P * 1.25))
    out = torch.empty((s.L, s.K, s.res, s.res), dtype=torch.float32, device="cuda")
    ab(g, out)
    st = ab.status()
    assert st["n_keys"] == P and not st["overflow"]
    items = np.arange(0, s.L * (s.res // 8) ** 2, STRIDE)
    To, _ = oracle_mod.build_tiles(s.gaussians, s.lights, s.res, s.K, items)
    assert np.abs(tiles_of(out, items) - To).max() <= TOL_T
    del out, ab
    torch.cuda.empty_cache()


# ---------------------------------------------------------------- onesweep
def _keys(kind: str, n: int, nbits: int, rng) -> np.ndarray:
    if kind == "uniform":
        return rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
    if kind == "few":          # few distinct digits per warp: the match.any / ballot paths
        return rng.choice(np.array([3, 77, 2**31 + 5, 2**nbits - 1], np.uint64), n).astype(np.uint32)
    if kind == "equal":
        return np.full(n, 0xDEADBEEF, np.uint32)
    if kind == "sorted":
        return np.sort(rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32))
    if kind == "reverse":
        return np.sort(rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32))[::-1].copy()
    raise ValueError(kind)


@pytest.mark.parametrize("nbits", [1, 7, 8, 12, 16, 24, 31, 32])
@pytest.mark.parametrize("n", [1, 2047, 2049, 300_001, 4_194_305])
def test_onesweep_vs_stable_argsort(dg, nbits, n):
    rng = np.random.default_rng(nbits * 7919 + n)
    for kind in ("uniform", "few", "equal", "sorted", "reverse"):
        k = _keys(kind, n, nbits, rng)
        v = np.arange(n, dtype=np.uint32)[::-1].copy()  # values carry the original position
        kd = torch.from_numpy(k.view(np.int32)).cuda()
        vd = torch.from_numpy(v.view(np.int32)).cuda()
        ks, vs = dg.sort_pairs(kd, vd, nbits)
        mask = np.uint32(0xFFFFFFFF) if nbits == 32 else np.uint32((1 << nbits) - 1)
        order = np.argsort(k & mask, kind="stable")
        assert np.array_equal(ks.cpu().numpy().view(np.uint32), k[order]), (kind, nbits, n)
        assert np.array_equal(vs.cpu().numpy().view(np.uint32), v[order]), (kind, nbits, n)
