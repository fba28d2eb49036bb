"""Parity of the shell-band accumulation kernel (K > 64 shells: the shared table
holds 48 shells and each band of 48 is one pass over the records meeting it,
DESIGN.md §6 a6) against the oracle, at K values that leave a ragged last band
(65 = 48 + 17, 100 = 2 x 48 + 4, 200 = 4 x 48 + 8) and the maximum K = 256; with
both record stagings, multi-chunk tiles (in-CTA and deferred combines), tau
output, the ROI slab, and band heights of 32 and 96 rows in a subprocess
(DGSM_BAND_ROWS is read once per process).

Bar: |T_gpu - T_oracle| <= 1e-4 (BASELINE.json north_star)."""
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_2601_01660_b200 import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL_T = 1e-4
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def dg():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2601_01660_b200 import build_ext, dgsm
    build_ext.build()
    dgsm.lib()
    return dgsm


def band_scene(seed, n, K, L=2):
    # Gaussians from 0.3 to 3 m and up to 0.5 m: windows across band boundaries,
    # records meeting two or three bands, steps landing in every band
    return synth.random_scene(seed, n, res=32, K=K, L=L, dist=(0.3, 3.0), scale=(0.01, 0.5))


@pytest.mark.parametrize("staging", ["tma", "reg"])
@pytest.mark.parametrize("K", [65, 100, 200, 256])
def test_band_build_parity(dg, oracle_mod, monkeypatch, K, staging):
    monkeypatch.setenv("DGSM_ACC_STAGING", staging)
    s = band_scene(61 + K, 1500, K)
    T = dg.build(dg.to_device(s.gaussians), s.lights, s.res, s.K).cpu().numpy()
    To, _ = oracle_mod.build(s.gaussians, s.lights, s.res, s.K)
    assert np.abs(T - To).max() <= TOL_T
    # T non-increasing along each ray (the band carries keep tau monotone)
    assert (np.diff(T, axis=1) <= 1e-6).all()


def test_band_multichunk_tiles(dg, oracle_mod):
    """20 000 Gaussians in a 32^2 atlas: tiles of many chunks, combined in the CTA
    that finishes last (<= 16 chunks) and by k_combine_deferred (> 16), at K = 100."""
    s = band_scene(71, 20000, 100)
    g = dg.to_device(s.gaussians)
    plan = dg.BuildPlan(g, s.lights, s.res, s.K)
    (_, _, _, _), (ts, te) = plan.bins()
    assert int((te - ts).max()) > 16 * int(plan.plan.chunk)
    T = dg.build(g, s.lights, s.res, s.K)
    To, _ = oracle_mod.build(s.gaussians, s.lights, s.res, s.K, tile_stride=3)
    m = ~np.isnan(To)
    assert np.abs(T.cpu().numpy()[m] - To[m]).max() <= TOL_T
    assert torch.equal(T, dg.build(g, s.lights, s.res, s.K))  # deterministic


def test_band_tau_output(dg, oracle_mod):
    s = band_scene(72, 1200, 130)
    g = dg.to_device(s.gaussians)
    tau = dg.build(g, s.lights, s.res, s.K, dg.Options(output_tau=True))
    T = dg.build(g, s.lights, s.res, s.K)
    To, _ = oracle_mod.build(s.gaussians, s.lights, s.res, s.K)
    assert np.abs(np.exp(-tau.cpu().numpy().astype(np.float64)) - To).max() <= TOL_T
    assert torch.allclose(torch.exp(-tau), T, atol=1e-6, rtol=0)


def test_band_slab_build(dg, oracle_mod):
    """ROI slab with K = 100: the slab's k range cuts across bands."""
    s = band_scene(73, 800, 100, L=3)
    rng = np.random.default_rng(173)
    rec = rng.uniform(-3, 3, (3000, 3)).astype(np.float32)
    roi = (0.2, -0.1, 0.3, 1.4, -1.0, 1.5)
    slab = dg.active_slab(torch.from_numpy(rec).cuda(), roi, s.lights, s.res, s.K)
    g = dg.to_device(s.gaussians)
    Ts = dg.build(g, s.lights, s.res, s.K, dg.Options(slab=slab)).cpu().numpy()
    mask, kr, inside = oracle_mod.active_slab(rec, roi, s.lights, s.res, s.K)
    assert inside > 0
    To, _ = oracle_mod.build(s.gaussians, s.lights, s.res, s.K, slab=(mask, kr))
    assert np.abs(Ts - To).max() <= TOL_T


_SUB = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
from paper_2601_01660_b200 import dgsm, synth
s = synth.random_scene({seed}, 1500, res=32, K={K}, L=2, dist=(0.3, 3.0), scale=(0.01, 0.5))
T = dgsm.build(dgsm.to_device(s.gaussians), s.lights, s.res, s.K).cpu().numpy()
np.save({out!r}, T)
"""


@pytest.mark.parametrize("rows,K", [(32, 100), (32, 256), (64, 128), (96, 200)])
def test_band_rows_override(dg, oracle_mod, tmp_path, rows, K):
    """DGSM_BAND_ROWS = 32 / 64 / 96 (2 to 8 bands; a band height that is not a
    power of two): same bar against the oracle."""
    out = str(tmp_path / "T.npy")
    env = dict(os.environ, DGSM_BAND_ROWS=str(rows))
    r = subprocess.run([sys.executable, "-c", _SUB.format(root=ROOT, seed=81, K=K, out=out)], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    T = np.load(out)
    s = synth.random_scene(81, 1500, res=32, K=K, L=2, dist=(0.3, 3.0), scale=(0.01, 0.5))
    To, _ = oracle_mod.build(s.gaussians, s.lights, s.res, s.K)
    assert np.abs(T - To).max() <= TOL_T


def _near_light_scene(K):
    """Gaussians at / within 1e-7 of / 2 cm from the light (an excluded pair, a
    footprint over the whole atlas, shell bounds clamped at shell 0) and large
    Gaussians 0.1-1 m from it (windows over many bands)."""
    s = synth.random_scene(13, 60, res=64, K=K, dist=(0.1, 1.0), scale=(0.05, 0.8))
    o = s.lights["position"][0].astype(np.float32)
    extra = np.stack([o, o + np.float32(1e-7), o + np.array([0.02, 0.0, 0.0], np.float32)])
    g = dict(s.gaussians)
    g["means"] = np.concatenate([g["means"], extra]).astype(np.float32)
    g["scales"] = np.concatenate([g["scales"], np.full((3, 3), 0.05, np.float32)])
    g["rotations"] = np.concatenate([g["rotations"], np.tile(np.array([1, 0, 0, 0], np.float32), (3, 1))])
    g["opacities"] = np.concatenate([g["opacities"], np.full(3, 0.5, np.float32)])
    return synth.Scene("near-light", g, s.lights, s.res, s.K, s.queries)


@pytest.mark.parametrize("K", [97, 160])
def test_band_near_light_and_big_footprints(dg, oracle_mod, K):
    s = _near_light_scene(K)
    T = dg.build(dg.to_device(s.gaussians), s.lights, s.res, s.K).cpu().numpy()
    To, _ = oracle_mod.build(s.gaussians, s.lights, s.res, s.K)
    assert np.abs(T - To).max() <= TOL_T
