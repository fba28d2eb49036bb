"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs.

Bars:
  * binning (P, sorted (light, tile, depth bits, index), tile ranges): bit-exact;
  * transmittance atlas: |T_gpu - T_oracle| <= 1e-4 (BASELINE.json north_star);
  * query on a seeded atlas: <= 2e-6 (fp32 weights and taps); end to end <= 1e-4.
"""
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


def _opts(dg, **kw):
    return dg.Options(**kw)


def gpu_bins(dg, scene, **opt):
    plan = dg.BuildPlan(dg.to_device(scene.gaussians), scene.lights, scene.res, scene.K, _opts(dg, **opt))
    (l, t, d, i), (ts, te) = plan.bins()
    return plan, [x.cpu().numpy().astype(np.uint32) for x in (l, t, d, i)], ts.cpu().numpy(), te.cpu().numpy()


def oracle_bins(oracle, scene, **opt):
    mode = oracle.BIN_CLAMP if opt.get("bin_mode") == "clamp" else oracle.BIN_WRAP
    return oracle.bin_entries(scene.gaussians["means"], scene.gaussians["scales"], scene.gaussians["rotations"],
                              scene.lights["position"], scene.res, k_sigma=opt.get("k_sigma", 3.0),
                              rho_scale=opt.get("rho_scale", 1.0), bin_mode=mode)


def ranges_from_entries(L_, T_, n_lights, res):
    nt = (res // 8) ** 2
    g = L_.astype(np.int64) * nt + T_.astype(np.int64)
    ts = np.zeros(n_lights * nt, np.int64)
    te = np.zeros(n_lights * nt, np.int64)
    if len(g):
        starts = np.r_[0, np.nonzero(np.diff(g))[0] + 1]
        ends = np.r_[starts[1:], len(g)]
        ts[g[starts]] = starts
        te[g[starts]] = ends
    return ts, te


def assert_bins_equal(dg, oracle, scene, **opt):
    plan, got, ts, te = gpu_bins(dg, scene, **opt)
    want = oracle_bins(oracle, scene, **opt)
    assert plan.n_keys == len(want[0]), (plan.n_keys, len(want[0]))
    for name, a, b in zip(("light", "tile", "depth", "index"), got, want):
        assert np.array_equal(a, b), f"{name} differs at {np.nonzero(a != b)[0][:10]}"
    wts, wte = ranges_from_entries(want[0], want[1], scene.L, scene.res)
    assert np.array_equal(ts, wts) and np.array_equal(te, wte)
    return plan.n_keys


def build_both(dg, oracle, scene, **opt):
    g = dg.to_device(scene.gaussians)
    T = dg.build(g, scene.lights, scene.res, scene.K, _opts(dg, **opt)).cpu().numpy()
    mode = oracle.BIN_CLAMP if opt.get("bin_mode") == "clamp" else oracle.BIN_WRAP
    To, P = oracle.build(scene.gaussians, scene.lights, scene.res, scene.K, kappa=opt.get("kappa", 1.0),
                         k_sigma=opt.get("k_sigma", 3.0), rho_scale=opt.get("rho_scale", 1.0), bin_mode=mode)
    return T, To


def equal_depth_scene(n_sign=8):
    """Gaussians at exactly the same distance from the light (sign flips and
    permutations of one offset): the depth key has 0 significant bits, so the
    depth sort runs no pass (the unsorted-count path of the build)."""
    import itertools
    base = np.array([0.5, 0.3, 0.2])
    offs = sorted({tuple(sg * base[list(pm)]) for pm in itertools.permutations(range(3))
                   for sg in itertools.product((-1.0, 1.0), repeat=3)})[:max(n_sign, 1)]
    m = np.asarray(offs, np.float32)
    n = len(m)
    g = dict(means=m, scales=np.full((n, 3), 0.05, np.float32),
             rotations=np.tile(np.array([1, 0, 0, 0], np.float32), (n, 1)), opacities=np.full(n, 0.6, np.float32))
    lights = dict(position=np.zeros((1, 3), np.float32), t_max=np.array([2.0], np.float32))
    return synth.Scene("equal-depth", g, lights, 32, 16, m.copy())


def light_coincident_scene():
    """A random scene plus Gaussians at the light (D = 0) and within 1e-7 of it
    (excluded, Q17) and one 2 cm from it (a footprint over the whole atlas)."""
    s = synth.random_scene(21, 200, res=32, K=16, dist=(0.3, 3.0), scale=(0.01, 0.3))
    o = s.lights["position"][0].astype(np.float32)
    extra = np.stack([o, o + np.float32(1e-7), o + np.array([0.02, 0.0, 0.0], np.float32)])
    g = dict(s.gaussians)
    g["means"] = np.concatenate([g["means"], extra]).astype(np.float32)
    g["scales"] = np.concatenate([g["scales"], np.full((3, 3), 0.05, np.float32)])
    g["rotations"] = np.concatenate([g["rotations"], np.tile(np.array([1, 0, 0, 0], np.float32), (3, 1))])
    g["opacities"] = np.concatenate([g["opacities"], np.full(3, 0.5, np.float32)])
    return synth.Scene("light-coincident", g, s.lights, s.res, s.K, s.queries)


SCENES = {
    "light-coincident": light_coincident_scene,
    "equal-depth": lambda: equal_depth_scene(48),
    "single-gaussian": lambda: equal_depth_scene(1),
    "cfg1": lambda: synth.config1(),
    "cfg1-seam-z": lambda: synth.config1_seam("-z"),
    "cfg1-seam-x": lambda: synth.config1_seam("+x"),
    "cfg1-seam-corner": lambda: synth.config1_seam("corner"),
    "random-3lights": lambda: synth.random_scene(11, 400, res=32, K=8, L=3, dist=(0.3, 3.0), scale=(0.01, 0.5)),
    "random-res8-K1": lambda: synth.random_scene(12, 150, res=8, K=1, dist=(0.5, 3.0)),
    "random-big-footprints": lambda: synth.random_scene(13, 60, res=64, K=12, dist=(0.1, 1.0), scale=(0.05, 0.8)),
    "cfg2-small": lambda: synth.config2(scale=0.004, res=64, K=16),
}


@pytest.mark.parametrize("name", sorted(SCENES))
def test_binning_bit_exact(dg, oracle_mod, name):
    P = assert_bins_equal(dg, oracle_mod, SCENES[name]())
    assert P > 0


@pytest.mark.parametrize("opt", [dict(bin_mode="clamp"), dict(rho_scale=2.6), dict(k_sigma=1.5)])
def test_binning_options_bit_exact(dg, oracle_mod, opt):
    assert_bins_equal(dg, oracle_mod, synth.config1_seam("corner"), **opt)


@pytest.mark.parametrize("name", sorted(SCENES))
def test_build_parity(dg, oracle_mod, name):
    T, To = build_both(dg, oracle_mod, SCENES[name]())
    err = np.abs(T - To).max()
    assert err <= TOL_T, err


@pytest.mark.parametrize("opt", [dict(kappa=2.0), dict(bin_mode="clamp"), dict(rho_scale=2.6)])
def test_build_parity_options(dg, oracle_mod, opt):
    T, To = build_both(dg, oracle_mod, synth.config1_seam("+x"), **opt)
    assert np.abs(T - To).max() <= TOL_T


@pytest.mark.parametrize("mode", ["simple", "mass", "diag"])
def test_build_parity_absorption_modes(dg, oracle_mod, mode):
    """Ablation B alpha -> beta mappings through the C ABI."""
    s = synth.config1_seam("corner")
    T = dg.build(dg.to_device(s.gaussians), s.lights, s.res, s.K, dg.Options(absorption=mode)).cpu().numpy()
    To, _ = oracle_mod.build(s.gaussians, s.lights, s.res, s.K, absorption=mode)
    assert np.abs(T - To).max() <= TOL_T


def test_build_parity_unculled(dg, oracle_mod):
    """Ablation D: no light-space culling, every Gaussian at every texel."""
    s = synth.random_scene(21, 150, res=32, K=8, L=2, dist=(0.4, 3.0), scale=(0.02, 0.4))
    T = dg.build(dg.to_device(s.gaussians), s.lights, s.res, s.K, dg.Options(tile_cull=False)).cpu().numpy()
    To, _ = oracle_mod.build(s.gaussians, s.lights, s.res, s.K, culled=False)
    assert np.abs(T - To).max() <= TOL_T
    Tc = dg.build(dg.to_device(s.gaussians), s.lights, s.res, s.K).cpu().numpy()
    assert (Tc >= T - 1e-6).all()  # culling only drops occluders


def test_build_invariants_and_determinism(dg):
    s = synth.config1()
    g = dg.to_device(s.gaussians)
    T1 = dg.build(g, s.lights, s.res, s.K)
    T2 = dg.build(g, s.lights, s.res, s.K)
    assert torch.equal(T1, T2)  # deterministic (fixed depth-order summation)
    T = T1.cpu().numpy()
    assert (T >= 0).all() and (T <= 1).all()
    assert (np.diff(T, axis=1) <= 1e-6).all()
    g2 = dg.to_device(synth.concat_gaussians(s.gaussians, s.gaussians))
    Td = dg.build(g2, s.lights, s.res, s.K).cpu().numpy()
    assert np.abs(Td - T ** 2).max() < 2e-5


def test_empty_scene_is_exactly_one(dg):
    s = synth.config1()
    g = {k: torch.zeros((0,) + v.shape[1:], dtype=torch.float32, device="cuda") for k, v in s.gaussians.items()}
    T = dg.build(g, s.lights, s.res, s.K)
    assert torch.all(T == 1.0)
    # all Gaussians excluded (at the light) -> 1 as well
    e = {k: v[:3].copy() for k, v in s.gaussians.items()}
    e["means"][:] = 0.0
    T = dg.build(dg.to_device(e), s.lights, s.res, s.K)
    assert torch.all(T == 1.0)


def test_multichunk_tiles(dg, oracle_mod):
    """> 1024 Gaussians in one tile: chunked work units + deterministic combine."""
    rng = np.random.default_rng(5)
    n = 3000
    d = np.array([0.2, 0.1, 1.0]); d /= np.linalg.norm(d)
    mu = d[None] * rng.uniform(1.0, 3.0, n)[:, None] + rng.normal(0, 0.004, (n, 3))
    g = dict(means=mu.astype(np.float32), scales=np.full((n, 3), 0.01, np.float32),
             rotations=synth.random_quaternions(rng, n).astype(np.float32),
             opacities=rng.uniform(0.01, 0.1, n).astype(np.float32))
    s = synth.Scene("dense", g, dict(position=np.zeros((1, 3), np.float32), t_max=np.array([4.0], np.float32)),
                    32, 16, mu.astype(np.float32))
    assert_bins_equal(dg, oracle_mod, s)
    T, To = build_both(dg, oracle_mod, s)
    assert np.abs(T - To).max() <= TOL_T
    gd = dg.to_device(g)
    assert torch.equal(dg.build(gd, s.lights, 32, 16), dg.build(gd, s.lights, 32, 16))


def test_output_tau_and_exp_epilogue(dg, oracle_mod):
    s = synth.config1_seam("-z")
    g = dg.to_device(s.gaussians)
    tau = dg.build(g, s.lights, s.res, s.K, dg.Options(output_tau=True))
    T = dg.exp_epilogue(tau)
    To, _ = oracle_mod.build(s.gaussians, s.lights, s.res, s.K)
    assert np.abs(T.cpu().numpy() - To).max() <= TOL_T
    dg.exp_epilogue(tau, out=tau)  # in place
    assert torch.equal(tau, T)


@pytest.mark.parametrize("L,K,res", [(1, 16, 64), (3, 8, 32), (2, 1, 8)])
def test_query_parity_random_atlas(dg, oracle_mod, L, K, res):
    atlas = synth.random_atlas(L + K + res, L, K, res)
    rng = np.random.default_rng(L * 100 + K)
    lights = dict(position=rng.uniform(-1, 1, (L, 3)).astype(np.float32),
                  t_max=rng.uniform(2, 5, L).astype(np.float32))
    x = synth.random_queries(K, lights, 20000, 6.0)
    x[:5] = lights["position"][0]  # at the light -> T_l = 1
    want = oracle_mod.query(atlas.astype(np.float64), lights, x)
    got = dg.query(torch.from_numpy(atlas).cuda(), lights, torch.from_numpy(x).cuda()).cpu().numpy()
    assert np.abs(got - want).max() <= 2e-6
    col = np.random.default_rng(1).random((x.shape[0], 3)).astype(np.float32)
    ct = torch.from_numpy(col).cuda()
    dg.query(torch.from_numpy(atlas).cuda(), lights, torch.from_numpy(x).cuda(), colors=ct)
    assert np.abs(ct.cpu().numpy() - col * want[:, None]).max() <= 2e-6


@pytest.mark.parametrize("L,K,res", [(1, 16, 64), (3, 8, 32), (8, 8, 2048), (1, 128, 1024)])
def test_query_ordered_parity(dg, oracle_mod, L, K, res):
    """dgsm_receiver_order is a permutation; the query visiting receivers in that
    order equals the plain query bit for bit and the oracle within 2e-6, also at
    the cfg5 resolution (2048^2, 8 lights) and K = 128 (the fp64 index math)."""
    atlas = synth.random_atlas(L * 7 + K + res, L, K, res)
    rng = np.random.default_rng(L * 1000 + K + res)
    lights = dict(position=rng.uniform(-1, 1, (L, 3)).astype(np.float32),
                  t_max=rng.uniform(2, 5, L).astype(np.float32))
    x = synth.random_queries(K + 1, lights, 50000, 6.0)
    x[:3] = lights["position"][0]
    want = oracle_mod.query(atlas.astype(np.float64), lights, x)
    at, xd = torch.from_numpy(atlas).cuda(), torch.from_numpy(x).cuda()
    order = dg.receiver_order(xd)
    o = order.long().cpu().numpy()
    assert np.array_equal(np.sort(o), np.arange(len(x)))
    plain = dg.query(at, lights, xd)
    got = dg.query(at, lights, xd, order=order)
    assert torch.equal(plain, got)
    assert np.abs(got.cpu().numpy() - want).max() <= 2e-6
    # the order is spatially coherent: consecutive receivers are close together
    step = np.linalg.norm(np.diff(x[o[4:]], axis=0), axis=1)
    rand = np.linalg.norm(np.diff(x[4:], axis=0), axis=1)
    assert np.median(step) < 0.2 * np.median(rand)


def test_query_chunks_sum_to_query(dg, oracle_mod):
    """dgsm_query_chunks + dgsm_query_combine (the multi-GPU query): light 1's
    shells split over two 'ranks' as [0, 3) and [3, 8); lights 0 and 2 complete.
    The summed shares times the complete lights equal dgsm_query and the oracle."""
    L, K, res = 3, 8, 32
    atlas = synth.random_atlas(77, L, K, res)
    rng = np.random.default_rng(5)
    lights = dict(position=rng.uniform(-1, 1, (L, 3)).astype(np.float32), t_max=rng.uniform(2, 5, L).astype(np.float32))
    x = torch.from_numpy(synth.random_queries(9, lights, 30000, 6.0)).cuda()
    at = torch.from_numpy(atlas).cuda()
    want = dg.query(at, lights, x)
    full = [(0, K, False, at[0].contiguous()), None, (0, K, False, at[2].contiguous())]
    T_a, p_a = dg.query_chunks([full[0], (0, 3, True, at[1, 0:3].contiguous()), full[2]], lights, x, res, K)
    T_b, p_b = dg.query_chunks([(0, 0, False, None), (3, K, True, at[1, 3:K].contiguous()), (0, 0, False, None)],
                               lights, x, res, K)
    assert p_a.shape == (1, x.shape[0]) and torch.all(T_b == 1.0)
    T = dg.query_combine(p_a + p_b, T_a)
    assert (T - want).abs().max().item() <= 2e-6
    wo = oracle_mod.query(atlas.astype(np.float64), lights, x.cpu().numpy())
    assert np.abs(T.cpu().numpy() - wo).max() <= 2e-6


def _receivers(seed, lights, m, K):
    rng = np.random.default_rng(seed)
    return dict(means=synth.random_queries(K, lights, m, 6.0),
                scales=np.exp(rng.uniform(np.log(0.005), np.log(0.5), (m, 3))).astype(np.float32),
                rotations=synth.random_quaternions(rng, m).astype(np.float32))


@pytest.mark.parametrize("kind", ["center", "stencil7", "mc32"])
def test_query_footprint_parity(dg, oracle_mod, kind):
    """NEXT-2 footprint-averaged query against the oracle."""
    L, K, res = 2, 12, 64
    atlas = synth.random_atlas(77, L, K, res)
    rng = np.random.default_rng(4)
    lights = dict(position=rng.uniform(-1, 1, (L, 3)).astype(np.float32),
                  t_max=rng.uniform(3, 5, L).astype(np.float32))
    g = _receivers(8, lights, 5000, K)
    if kind == "mc32":
        z, w = synth.mc_offsets(32, 3), np.full(32, 1 / 32, np.float32)
    else:
        z, w = dg.footprint_stencil(kind)
    zo, wo = oracle_mod.stencil7(1.0) if kind == "stencil7" else (z.astype(np.float64), w.astype(np.float64))
    assert np.abs(zo - z).max() == 0 and np.abs(wo - w).max() < 1e-7
    want = oracle_mod.query_footprint(atlas.astype(np.float64), lights, g, zo, wo)
    gd = dg.to_device(g)
    at = torch.from_numpy(atlas).cuda()
    got = dg.query_footprint(at, lights, gd, z, w).cpu().numpy()
    assert np.abs(got - want).max() <= 4e-6
    if kind == "center":
        assert torch.equal(torch.from_numpy(got), dg.query(at, lights, gd["means"]).cpu())
    col = np.random.default_rng(2).random((5000, 3)).astype(np.float32)
    ct = torch.from_numpy(col).cuda()
    dg.query_footprint(at, lights, gd, z, w, colors=ct)
    assert np.abs(ct.cpu().numpy() - col * want[:, None]).max() <= 4e-6


def unpack_slab(buf, L, res):
    """include/dgsm.h slab layout -> (mask bool [L, res, res], krange int32 [L, 2])."""
    TW = res // 8
    raw = buf.cpu().numpy()
    nb = 8 * L * TW * TW
    words = np.frombuffer(raw[:nb].tobytes(), np.uint64).reshape(L, TW, TW)
    bits = (words[..., None] >> np.arange(64, dtype=np.uint64)) & np.uint64(1)
    mask = bits.reshape(L, TW, TW, 8, 8).transpose(0, 1, 3, 2, 4).reshape(L, res, res).astype(bool)
    off = (nb + 255) // 256 * 256
    kr = np.frombuffer(raw[off:off + 8 * L].tobytes(), np.int32).reshape(L, 2)
    return mask, kr


def _slab_case(seed, small=False):
    s = synth.random_scene(seed, 300, res=32, K=12, L=3, dist=(0.3, 3.0), scale=(0.02, 0.4))
    rng = np.random.default_rng(seed + 100)
    rec = rng.uniform(-3, 3, (3000, 3)).astype(np.float32)
    rec[:3] = s.lights["position"][0]  # receivers at a light: skipped for that light
    rec[3:6] = s.lights["position"][0] + np.array([[-1.0, 0, 0], [0, 1.0, 0], [0, 0, -1.0]], np.float32)  # seams
    roi = (1.8, 1.6, 0.0, 0.7, -0.5, 0.5) if small else (0.2, -0.1, 0.3, 1.4, -1.0, 1.5)
    return s, rec, roi


@pytest.mark.parametrize("seed", [41, 42])
def test_active_slab_bit_exact(dg, oracle_mod, seed):
    """NEXT-1 pixel set P and k range: bit-exact against the oracle (fp64 decisions)."""
    s, rec, roi = _slab_case(seed)
    slab = dg.active_slab(torch.from_numpy(rec).cuda(), roi, s.lights, s.res, s.K)
    mask, kr = unpack_slab(slab, s.L, s.res)
    wm, wk, inside = oracle_mod.active_slab(rec, roi, s.lights, s.res, s.K)
    assert inside > 0 and np.array_equal(mask, wm) and np.array_equal(kr, wk)
    # empty ROI: nothing marked, every light empty
    slab = dg.active_slab(torch.from_numpy(rec).cuda(), (50, 50, 0, 0.1, 0, 0), s.lights, s.res, s.K)
    mask, kr = unpack_slab(slab, s.L, s.res)
    assert not mask.any() and (kr[:, 0] == s.K).all() and (kr[:, 1] == -1).all()


def test_slab_build_parity_and_exactness(dg, oracle_mod):
    """Slab build against the oracle's slab build; 1 outside the slab
    bit-exactly; queries at receivers in B equal those on the full GPU atlas
    bit-for-bit; binning restricted to the active tiles, bit-exact."""
    s, rec, roi = _slab_case(43, small=True)
    rt = torch.from_numpy(rec).cuda()
    slab = dg.active_slab(rt, roi, s.lights, s.res, s.K)
    g = dg.to_device(s.gaussians)
    Ts = dg.build(g, s.lights, s.res, s.K, dg.Options(slab=slab))
    Tf = dg.build(g, s.lights, s.res, s.K)
    mask, kr, inside = oracle_mod.active_slab(rec, roi, s.lights, s.res, s.K)
    To, _ = oracle_mod.build(s.gaussians, s.lights, s.res, s.K, slab=(mask, kr))
    Tsn = Ts.cpu().numpy()
    assert np.abs(Tsn - To).max() <= TOL_T
    kk = np.arange(s.K)[None, :, None, None]
    in_slab = mask[:, None] & (kk >= kr[:, 0, None, None, None]) & (kk <= kr[:, 1, None, None, None])
    assert (Tsn[~in_slab] == 1.0).all()
    assert np.array_equal(Tsn[in_slab], Tf.cpu().numpy()[in_slab])
    ins = (np.maximum(np.abs(rec[:, 0] - roi[0]), np.abs(rec[:, 1] - roi[1])) <= roi[3]) & \
          (rec[:, 2] >= roi[4]) & (rec[:, 2] <= roi[5])
    xin = torch.from_numpy(rec[ins]).cuda()
    assert torch.equal(dg.query(Ts, s.lights, xin), dg.query(Tf, s.lights, xin))
    # tau output honours the slab too (tau = 0 outside)
    tau = dg.build(g, s.lights, s.res, s.K, dg.Options(slab=slab, output_tau=True)).cpu().numpy()
    assert (tau[~in_slab] == 0.0).all()
    # binning: the oracle's entries restricted to tiles holding a texel of P
    plan, got, ts, te = gpu_bins(dg, s, slab=slab)
    want = oracle_bins(oracle_mod, s)
    tile_on = mask.reshape(s.L, s.res // 8, 8, s.res // 8, 8).any(axis=(2, 4)).reshape(s.L, -1)
    keep = tile_on[want[0].astype(np.int64), want[1].astype(np.int64)]
    want = [w[keep] for w in want]
    assert plan.n_keys == len(want[0]) and 0 < plan.n_keys < len(keep)
    for a, b in zip(got, want):
        assert np.array_equal(a, b)


def test_slab_empty_roi_all_ones(dg):
    s, rec, _ = _slab_case(44)
    slab = dg.active_slab(torch.from_numpy(rec).cuda(), (50, 50, 0, 0.1, 0, 0), s.lights, s.res, s.K)
    plan = dg.BuildPlan(dg.to_device(s.gaussians), s.lights, s.res, s.K, dg.Options(slab=slab))
    assert plan.n_keys == 0
    T = dg.build(dg.to_device(s.gaussians), s.lights, s.res, s.K, dg.Options(slab=slab))
    assert torch.all(T == 1.0)


def test_frame_host_equals_device_path(dg, oracle_mod):
    """dgsm_frame_host (HOST inputs, chunked upload + projection, side-stream
    receiver upload) gives exactly the device-path build + query, and the
    oracle's within tolerance."""
    s = synth.config2(scale=0.02, res=64, K=16)
    gh = {k: torch.from_numpy(np.ascontiguousarray(v, np.float32)).pin_memory() for k, v in s.gaussians.items()}
    rh = torch.from_numpy(s.queries).pin_memory()
    Th = torch.empty(rh.shape[0]).pin_memory()
    fr = dg.FrameHost(s.lights, s.res, s.K)
    at = fr(gh, rh, Th)
    torch.cuda.synchronize()
    at2 = dg.build(dg.to_device(s.gaussians), s.lights, s.res, s.K)
    T2 = dg.query(at2, s.lights, torch.from_numpy(s.queries).cuda())
    assert torch.equal(at, at2) and torch.equal(Th, T2.cpu())
    at = fr(gh, rh, Th)  # workspace reused
    torch.cuda.synchronize()
    assert torch.equal(Th, T2.cpu()) and fr.launches > 10
    Tp = torch.empty(rh.shape[0])  # pageable T: device buffer + copy instead of direct writes
    fr(gh, rh, Tp)
    torch.cuda.synchronize()
    assert torch.equal(Tp, T2.cpu())
    To, _ = oracle_mod.build(s.gaussians, s.lights, s.res, s.K)
    assert np.abs(Th.numpy() - oracle_mod.query(To, s.lights, s.queries)).max() <= TOL_T


def test_query_empty(dg):
    atlas = torch.ones(1, 4, 16, 16, device="cuda")
    out = dg.query(atlas, dict(position=[[0, 0, 0]], t_max=[1.0]), torch.zeros(0, 3, device="cuda"))
    assert out.numel() == 0


def test_end_to_end_cfg1(dg, oracle_mod):
    s = synth.config1()
    g = dg.to_device(s.gaussians)
    atlas = dg.build(g, s.lights, s.res, s.K)
    T = dg.query(atlas, s.lights, torch.from_numpy(s.queries).cuda()).cpu().numpy()
    To, _ = oracle_mod.build(s.gaussians, s.lights, s.res, s.K)
    Tq = oracle_mod.query(To, s.lights, s.queries)
    assert np.abs(T - Tq).max() <= TOL_T


def _probe(seed, d):
    rng = np.random.default_rng(seed)
    A = np.zeros((3, (d + 1) ** 2))
    A[:, 0] = rng.uniform(1.5, 3.0, 3)
    for l in range(1, d + 1):
        A[:, l * l:(l + 1) ** 2] = rng.normal(0, 0.8 / l, (3, 2 * l + 1))
    return A


@pytest.mark.parametrize("d,q,grid", [(3, 1.0, (64, 128)), (2, 2.0, (32, 64)), (3, 0.5, (48, 96)), (0, 1.0, (16, 32))])
def test_sh_transfer_parity(dg, oracle_mod, d, q, grid):
    """NEXT-4: scales and relit colours against the fp64 oracle."""
    rng = np.random.default_rng(7 + d)
    n = 3000
    nr = rng.normal(size=(n, 3))
    nr /= np.linalg.norm(nr, axis=1, keepdims=True)
    nr = nr.astype(np.float32)
    col = rng.random((n, 3)).astype(np.float32)
    A = _probe(d, d).astype(np.float32)
    s, co = dg.sh_transfer(A, d, torch.from_numpy(nr).cuda(), torch.from_numpy(col).cuda(), grid=grid, q=q,
                           gamma=1.3)
    so, coo = oracle_mod.sh_transfer(A.astype(np.float64), d, nr.astype(np.float64), col.astype(np.float64),
                                     n_theta=grid[0], n_phi=grid[1], q=q, gamma=1.3)
    assert np.abs(s.cpu().numpy() - so).max() <= 2e-5 * max(1.0, np.abs(so).max())
    assert np.abs(co.cpu().numpy() - coo).max() <= 2e-5 * max(1.0, np.abs(coo).max())
    s2, _ = dg.sh_transfer(A, d, torch.from_numpy(nr).cuda(), grid=grid, q=q, gamma=1.3)
    assert torch.equal(s, s2)  # deterministic


def test_sh_transfer_edge_cases(dg):
    nr = torch.tensor([[0, 0, 1.0]], device="cuda")
    A = np.zeros((3, 16), np.float32)
    A[:, 0] = 2 * np.sqrt(np.pi)  # L = 1 everywhere
    s, _ = dg.sh_transfer(A, 3, nr, eps=0.0)
    assert torch.allclose(s, torch.ones_like(s), atol=2e-6)
    s, _ = dg.sh_transfer(100 * A, 3, nr, s_max=4.0)
    assert torch.all(s == 4.0)
    s, c = dg.sh_transfer(A, 3, torch.zeros(0, 3, device="cuda"), torch.zeros(0, 3, device="cuda"))
    assert s.numel() == 0 and c.numel() == 0


def test_builder_one_call_equals_plan_run(dg):
    """dgsm_build (plan + run in one C call, workspace reused) == dgsm_build_plan + dgsm_build_run."""
    s = synth.config1_seam("corner")
    g = dg.to_device(s.gaussians)
    out = torch.empty((s.L, s.K, s.res, s.res), device="cuda")
    b = dg.Builder(s.lights, s.res, s.K)
    for _ in range(2):
        b(g, out)
        assert torch.equal(out, dg.build(g, s.lights, s.res, s.K))
    p = dg.BuildPlan(g, s.lights, s.res, s.K)
    p.run()
    assert b.launches == p.plan_launches + p.run_launches > 10  # the kernels one build launches


@pytest.mark.parametrize("staging", ["tma", "reg"])
def test_accumulate_staging_variants(dg, oracle_mod, staging, monkeypatch):
    """Both record-staging variants of the accumulation kernel (TMA bulk copies /
    register prefetch) against the oracle, and identical to each other."""
    monkeypatch.setenv("DGSM_ACC_STAGING", staging)
    for name in ("cfg1-seam-corner", "random-3lights", "cfg2-small"):
        T, To = build_both(dg, oracle_mod, SCENES[name]())
        assert np.abs(T - To).max() <= TOL_T, name
    s = synth.random_scene(31, 400, res=32, K=64, L=2, dist=(0.3, 3.0), scale=(0.01, 0.4))
    g = dg.to_device(s.gaussians)
    T = dg.build(g, s.lights, s.res, s.K)
    monkeypatch.setenv("DGSM_ACC_STAGING", "reg" if staging == "tma" else "tma")
    assert torch.equal(T, dg.build(g, s.lights, s.res, s.K))


def test_work_unit_paths_identical(dg, oracle_mod, monkeypatch):
    """The single-CTA work-unit builder (<= 16 K tiles) and the multi-kernel one
    (larger atlases; forced here) give the same atlas, bit for bit, on a scene
    with multi-chunk tiles, some of them combined after the accumulation kernel
    (> 16 chunks), and it matches the oracle."""
    s = synth.random_scene(33, 20000, res=32, K=16, L=2, dist=(0.3, 3.0), scale=(0.01, 0.3))
    g = dg.to_device(s.gaussians)
    plan = dg.BuildPlan(g, s.lights, s.res, s.K)
    (_, t, _, _), (ts, te) = plan.bins()
    # the adaptive chunk (a small key set) gives its densest tiles more than
    # kInlineCombine = 16 chunks: those are summed by k_combine_deferred
    assert int((te - ts).max()) > 16 * int(plan.plan.chunk)
    T = dg.build(g, s.lights, s.res, s.K)
    monkeypatch.setenv("DGSM_UNITS_MULTI", "1")
    assert torch.equal(T, dg.build(g, s.lights, s.res, s.K))
    To, _ = oracle_mod.build(s.gaussians, s.lights, s.res, s.K, tile_stride=5)
    m = ~np.isnan(To)
    assert np.abs(T.cpu().numpy()[m] - To[m]).max() <= TOL_T


def test_frame_host_pipelined_frames(dg):
    """Back-to-back frames with different inputs, no synchronisation between them
    (frame i+1's uploads overlap frame i's build): each equals its device path."""
    frames = []
    for seed in (51, 52, 53):
        s = synth.random_scene(seed, 3000, res=32, K=16, L=1, dist=(0.3, 3.0), scale=(0.01, 0.3))
        frames.append(s)
    s0 = frames[0]
    fr = dg.FrameHost(s0.lights, s0.res, s0.K)
    outs = []
    for s in frames:
        gh = {k: torch.from_numpy(np.ascontiguousarray(v, np.float32)).pin_memory() for k, v in s.gaussians.items()}
        rh = torch.from_numpy(np.ascontiguousarray(s.queries, np.float32)).pin_memory()
        Th = torch.empty(rh.shape[0]).pin_memory()
        at = fr(gh, rh, Th).clone()
        outs.append((gh, rh, Th, at))
    torch.cuda.synchronize()
    for s, (gh, rh, Th, at) in zip(frames, outs):
        at2 = dg.build(dg.to_device(s.gaussians), s0.lights, s0.res, s0.K)
        assert torch.equal(at, at2)
        T2 = dg.query(at2, s0.lights, torch.from_numpy(np.ascontiguousarray(s.queries, np.float32)).cuda())
        assert torch.equal(Th, T2.cpu())
