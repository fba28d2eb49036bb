"""ctypes + numpy wrapper around ``liboracle.so`` (oracle/dgsm_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by ``tests/``, ``__graft_entry__.smoke()``
and the ``cpu_baseline`` / ``--impl reference`` legs of ``bench.py``.  The
product path (``paper_2601_01660_b200``) never imports this module, and this
module never imports the product package.

Every function mirrors a C function of the oracle; see its header for the
PAPER.md passages followed.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "dgsm_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

GCC_FLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-Wall"]


def build_oracle(force: bool = False) -> str:
    """Compile the oracle with gcc (strict IEEE double, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", *GCC_FLAGS, "-o", _LIB, _SRC, "-lm", "-lpthread"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build_oracle()
        L = C.CDLL(_LIB)
        dp, fp, u32p, i64p = (C.POINTER(C.c_double), C.POINTER(C.c_float),
                              C.POINTER(C.c_uint32), C.POINTER(C.c_int64))
        L.or_beta.restype = C.c_double
        L.or_beta.argtypes = [fp, fp, C.c_float, C.c_double]
        L.or_oct_encode.argtypes = [dp, dp]
        L.or_oct_decode.argtypes = [C.c_double, C.c_double, dp]
        L.or_texel_dir.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, dp]
        L.or_bin_center.restype = C.c_double
        L.or_bin_center.argtypes = [C.c_int, C.c_int, C.c_double]
        L.or_footprint.restype = C.c_int
        L.or_footprint.argtypes = [fp, fp, fp, fp, C.c_int, C.c_double, C.c_double, dp, i64p]
        L.or_mirror_wrap.argtypes = [C.c_int64, C.c_int64, C.c_int, C.c_int, i64p]
        L.or_bin.restype = C.c_int64
        L.or_bin.argtypes = [fp, fp, fp, C.c_int64, fp, C.c_int, C.c_int, C.c_double, C.c_double,
                             C.c_int, u32p, u32p, u32p, u32p, C.c_int64]
        L.or_bin_start.restype = C.c_void_p
        L.or_bin_start.argtypes = [fp, fp, fp, C.c_int64, fp, C.c_int, C.c_int, C.c_double, C.c_double,
                                   C.c_int, i64p]
        L.or_bin_take.restype = None
        L.or_bin_take.argtypes = [C.c_void_p, C.c_int64, u32p, u32p, u32p, u32p]
        L.or_ray_quadratic.argtypes = [dp, dp, dp, dp, dp]
        L.or_segment_depth.restype = C.c_double
        L.or_segment_depth.argtypes = [C.c_double] * 5
        L.or_build.restype = C.c_int64
        L.or_build.argtypes = [fp, fp, fp, fp, C.c_int64, fp, fp, C.c_int, C.c_int, C.c_int,
                               C.c_double, C.c_double, C.c_double, C.c_int, C.c_int, C.c_int, C.c_int64,
                               C.c_int, dp, i64p]
        L.or_build_tiles.restype = C.c_int64
        L.or_build_tiles.argtypes = [fp, fp, fp, fp, C.c_int64, fp, fp, C.c_int, C.c_int, C.c_int,
                                     C.c_double, C.c_double, C.c_double, C.c_int, C.c_int, i64p, C.c_int64,
                                     C.c_int, dp, i64p]
        L.or_build_slab.restype = C.c_int64
        L.or_build_slab.argtypes = [fp, fp, fp, fp, C.c_int64, fp, fp, C.c_int, C.c_int, C.c_int,
                                    C.c_double, C.c_double, C.c_double, C.c_int, C.c_int, C.c_int, C.c_int64,
                                    C.c_int, C.POINTER(C.c_ubyte), C.POINTER(C.c_int32), dp, i64p]
        L.or_active_slab.restype = C.c_int64
        L.or_active_slab.argtypes = [fp, C.c_int64, fp, fp, fp, C.c_int, C.c_int, C.c_int,
                                     C.POINTER(C.c_ubyte), C.POINTER(C.c_int32)]
        L.or_sh_basis.argtypes = [C.c_int, dp, dp]
        L.or_transfer_dir.argtypes = [C.c_int, C.c_int, C.c_int64, dp, dp]
        L.or_sh_transfer.argtypes = [dp, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                     C.c_double, dp, dp, C.c_int64, dp, dp]
        L.or_query_footprint.argtypes = [dp, C.c_int, C.c_int, C.c_int, fp, fp, fp, fp, fp, C.c_int64,
                                         dp, dp, C.c_int, dp]
        L.or_beta_mode.restype = C.c_double
        L.or_beta_mode.argtypes = [fp, fp, C.c_float, C.c_double, C.c_int]
        L.or_tau_ray.restype = C.c_double
        L.or_tau_ray.argtypes = [fp, fp, fp, fp, C.c_int64, dp, dp, C.c_double, C.c_double]
        L.or_query.argtypes = [dp, C.c_int, C.c_int, C.c_int, fp, fp, fp, C.c_int64, dp, dp]
        _lib = L
    return _lib


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def _opt(x) -> float:
    """Build options are fp32 quantities in the problem statement's C ABI
    (kappa, k_sigma, rho_scale); the oracle takes the same fp32 values."""
    return float(np.float32(x))


BIN_WRAP, BIN_CLAMP = 0, 1
ABS_TRACEAVG, ABS_SIMPLE, ABS_MASS, ABS_DIAG = 0, 1, 2, 3
ABSORPTION = {"traceavg": 0, "simple": 1, "mass": 2, "diag": 3}


def beta(scales, rotation, alpha, kappa=1.0, mode=ABS_TRACEAVG) -> float:
    """Eq.5 for one Gaussian; other modes: ablation B."""
    s, q = _f32(scales), _f32(rotation)
    if mode == ABS_TRACEAVG:
        return lib().or_beta(_p(s, C.c_float), _p(q, C.c_float), float(alpha), float(kappa))
    return lib().or_beta_mode(_p(s, C.c_float), _p(q, C.c_float), float(alpha), float(kappa), int(mode))


def oct_encode(d):
    d = _f64(d)
    out = np.zeros(2)
    lib().or_oct_encode(_p(d, C.c_double), _p(out, C.c_double))
    return out


def oct_decode(u, v):
    out = np.zeros(3)
    lib().or_oct_decode(float(u), float(v), _p(out, C.c_double))
    return out


def texel_dir(row, col, H, W):
    out = np.zeros(3)
    lib().or_texel_dir(int(row), int(col), int(H), int(W), _p(out, C.c_double))
    return out


def bin_center(k, K, t_max) -> float:
    return lib().or_bin_center(int(k), int(K), float(t_max))


def footprint(mean, scales, rotation, light, res, k_sigma=3.0, rho_scale=1.0):
    """R4-R5: returns None if excluded, else dict(D, px, py, p1, lam1, rect=(c0,c1,r0,r1))."""
    mu, s, q, o = _f32(mean), _f32(scales), _f32(rotation), _f32(light)
    fpv = np.zeros(5)
    rect = np.zeros(4, dtype=np.int64)
    ok = lib().or_footprint(_p(mu, C.c_float), _p(s, C.c_float), _p(q, C.c_float),
                            _p(o, C.c_float), int(res), _opt(k_sigma), _opt(rho_scale),
                            _p(fpv, C.c_double), _p(rect, C.c_int64))
    if not ok:
        return None
    return dict(D=fpv[0], px=fpv[1], py=fpv[2], p1=fpv[3], lam1=fpv[4], rect=tuple(int(x) for x in rect))


def mirror_wrap(col, row, H, W):
    out = np.zeros(2, dtype=np.int64)
    lib().or_mirror_wrap(int(col), int(row), int(H), int(W), _p(out, C.c_int64))
    return int(out[0]), int(out[1])


def bin_entries(means, scales, rotations, light_pos, res, k_sigma=3.0, rho_scale=1.0,
                bin_mode=BIN_WRAP):
    """R6-R7: sorted (light, tile, depth_bits, index) arrays (uint32 each)."""
    mu, s, q, lp = _f32(means), _f32(scales), _f32(rotations), _f32(light_pos)
    n, L = mu.shape[0], lp.reshape(-1, 3).shape[0]
    args = [_p(mu, C.c_float), _p(s, C.c_float), _p(q, C.c_float), n, _p(lp, C.c_float), L,
            int(res), _opt(k_sigma), _opt(rho_scale), int(bin_mode)]
    Pc = C.c_int64(0)
    h = lib().or_bin_start(*args, C.byref(Pc))
    P = int(Pc.value)
    outs = [np.zeros(max(P, 1), dtype=np.uint32) for _ in range(4)]
    lib().or_bin_take(h, P, *[_p(o, C.c_uint32) for o in outs])
    return tuple(o[:P] for o in outs)


def ray_quadratic(A, mu, o, d):
    A, mu, o, d = _f64(A), _f64(mu), _f64(o), _f64(d)
    out = np.zeros(3)
    lib().or_ray_quadratic(_p(A, C.c_double), _p(mu, C.c_double), _p(o, C.c_double),
                           _p(d, C.c_double), _p(out, C.c_double))
    return out


def segment_depth(a, b, c, beta_, t) -> float:
    return lib().or_segment_depth(float(a), float(b), float(c), float(beta_), float(t))


def tau_ray(g, o, d, t, kappa=1.0) -> float:
    mu, s, q, a = _f32(g["means"]), _f32(g["scales"]), _f32(g["rotations"]), _f32(g["opacities"])
    o, d = _f64(o), _f64(d)
    return lib().or_tau_ray(_p(mu, C.c_float), _p(s, C.c_float), _p(q, C.c_float),
                            _p(a, C.c_float), mu.shape[0], _p(o, C.c_double), _p(d, C.c_double),
                            float(t), float(kappa))


def build(g, lights, res, K, kappa=1.0, k_sigma=3.0, rho_scale=1.0, bin_mode=BIN_WRAP,
          culled=True, tile_stride=1, n_threads=None, return_evals=False, absorption="traceavg",
          slab=None):
    """R8: the atlas T[L][K][res][res] in float64 (NaN where skipped by tile_stride).

    ``g``: dict of means [n,3], scales [n,3], rotations [n,4] (w,x,y,z), opacities [n].
    ``lights``: dict(position [L,3], t_max [L]).
    ``absorption``: traceavg (Eq.5) | simple | mass | diag (ablation B).
    ``slab``: (mask [L,res,res], krange [L,2]) from active_slab: T = 1 outside
    the slab, else the full atlas.
    Returns (T, P) with P the number of binned entries (culled mode)."""
    mode = ABSORPTION[absorption] if isinstance(absorption, str) else int(absorption)
    mu, s, q, a = _f32(g["means"]), _f32(g["scales"]), _f32(g["rotations"]), _f32(g["opacities"])
    lp, tm = _f32(lights["position"]).reshape(-1, 3), _f32(lights["t_max"]).reshape(-1)
    L = lp.shape[0]
    T = np.empty((L, K, res, res), dtype=np.float64)
    n_threads = n_threads or os.cpu_count() or 1
    evals = C.c_int64(0)
    sm = sk = None
    if slab is not None:
        mk = np.ascontiguousarray(slab[0], dtype=np.uint8).reshape(L, res, res)
        kr = np.ascontiguousarray(slab[1], dtype=np.int32).reshape(L, 2)
        sm, sk = _p(mk, C.c_ubyte), _p(kr, C.c_int32)
    P = lib().or_build_slab(_p(mu, C.c_float), _p(s, C.c_float), _p(q, C.c_float), _p(a, C.c_float),
                            mu.shape[0], _p(lp, C.c_float), _p(tm, C.c_float), L, int(res), int(K),
                            _opt(kappa), _opt(k_sigma), _opt(rho_scale), int(bin_mode),
                            int(bool(culled)), mode, int(tile_stride), int(n_threads), sm, sk,
                            _p(T, C.c_double), C.byref(evals))
    if P < 0:
        raise ValueError("oracle build: invalid arguments")
    if return_evals:
        return T, int(P), int(evals.value)
    return T, int(P)


def build_tiles(g, lights, res, K, items, kappa=1.0, k_sigma=3.0, rho_scale=1.0, bin_mode=BIN_WRAP,
                absorption="traceavg", n_threads=None):
    """R8 on a list of work items only (culled build, full-atlas semantics):
    ``items`` = l * (res/8)^2 + tile.  Returns (T [n_items, K, 8, 8] float64 —
    the 64 texels of each item's tile, row-major — and P).  For sampled-tile
    parity on atlases too large for a float64 copy (2048^2 x 128 x 8 lights)."""
    mode = ABSORPTION[absorption] if isinstance(absorption, str) else int(absorption)
    mu, s, q, a = _f32(g["means"]), _f32(g["scales"]), _f32(g["rotations"]), _f32(g["opacities"])
    lp, tm = _f32(lights["position"]).reshape(-1, 3), _f32(lights["t_max"]).reshape(-1)
    it = np.ascontiguousarray(items, dtype=np.int64).reshape(-1)
    T = np.empty((len(it), K, 8, 8), dtype=np.float64)
    n_threads = n_threads or os.cpu_count() or 1
    evals = C.c_int64(0)
    P = lib().or_build_tiles(_p(mu, C.c_float), _p(s, C.c_float), _p(q, C.c_float), _p(a, C.c_float),
                             mu.shape[0], _p(lp, C.c_float), _p(tm, C.c_float), lp.shape[0], int(res), int(K),
                             _opt(kappa), _opt(k_sigma), _opt(rho_scale), int(bin_mode), mode,
                             _p(it, C.c_int64), len(it), int(n_threads), _p(T, C.c_double), C.byref(evals))
    if P < 0:
        raise ValueError("oracle build_tiles: invalid arguments")
    return T, int(P)


def active_slab(receivers, roi, lights, res, K):
    """NEXT-1: the ROI pixel set P and radial range of receivers in
    B.  ``roi`` = (c_x, c_y, c_z, R, z_min, z_max).  Returns (mask bool
    [L,res,res], krange int32 [L,2], receivers inside B)."""
    x = _f32(receivers).reshape(-1, 3)
    r = _f32(roi).reshape(6)
    lp, tm = _f32(lights["position"]).reshape(-1, 3), _f32(lights["t_max"]).reshape(-1)
    L = lp.shape[0]
    mask = np.zeros((L, res, res), np.uint8)
    kr = np.zeros((L, 2), np.int32)
    inside = lib().or_active_slab(_p(x, C.c_float), x.shape[0], _p(r, C.c_float), _p(lp, C.c_float),
                                  _p(tm, C.c_float), L, int(res), int(K), _p(mask, C.c_ubyte),
                                  _p(kr, C.c_int32))
    return mask.astype(bool), kr, int(inside)


def query(atlas, lights, positions, colors=None):
    """R10-R12: T_out[m] = prod_l trilinear(atlas_l, x) (float64); colors *= T if given."""
    at = _f64(atlas)
    L, K, res = at.shape[0], at.shape[1], at.shape[2]
    lp, tm = _f32(lights["position"]).reshape(-1, 3), _f32(lights["t_max"]).reshape(-1)
    x = _f32(positions).reshape(-1, 3)
    out = np.zeros(x.shape[0])
    col = None if colors is None else _f64(colors).copy()
    lib().or_query(_p(at, C.c_double), L, K, res, _p(lp, C.c_float), _p(tm, C.c_float),
                   _p(x, C.c_float), x.shape[0], _p(out, C.c_double),
                   None if col is None else _p(col, C.c_double))
    return (out, col) if colors is not None else out


def stencil7(delta=1.0):
    """Deterministic 7-point footprint stencil: offsets
    {0, +-delta e_1, +-delta e_2, +-delta e_3} in the principal-axes frame,
    weights proportional to exp(-|z|^2/2), normalised to sum 1."""
    z = [[0.0, 0.0, 0.0]]
    for j in range(3):
        for sgn in (1.0, -1.0):
            e = [0.0, 0.0, 0.0]
            e[j] = sgn * delta
            z.append(e)
    z = np.array(z)
    w = np.exp(-0.5 * (z ** 2).sum(1))
    return z, w / w.sum()


def query_footprint(atlas, lights, g, z, w):
    """NEXT-2: T_g = prod_l sum_i w_i T_l(mu_g + R_g (s_g * z_i))."""
    at = _f64(atlas)
    L, K, res = at.shape[0], at.shape[1], at.shape[2]
    lp, tm = _f32(lights["position"]).reshape(-1, 3), _f32(lights["t_max"]).reshape(-1)
    mu, s, q = _f32(g["means"]).reshape(-1, 3), _f32(g["scales"]).reshape(-1, 3), _f32(g["rotations"]).reshape(-1, 4)
    z, w = _f64(z).reshape(-1, 3), _f64(w).reshape(-1)
    out = np.zeros(mu.shape[0])
    lib().or_query_footprint(_p(at, C.c_double), L, K, res, _p(lp, C.c_float), _p(tm, C.c_float),
                             _p(mu, C.c_float), _p(s, C.c_float), _p(q, C.c_float), mu.shape[0],
                             _p(z, C.c_double), _p(w, C.c_double), z.shape[0], _p(out, C.c_double))
    return out


def sh_basis(dirs, d):
    """NEXT-4: real SH basis (orthonormal, Condon-Shortley phase, k = l^2+l+m) [N, (d+1)^2]."""
    x = _f64(dirs).reshape(-1, 3)
    out = np.zeros((x.shape[0], (d + 1) ** 2))
    row = np.zeros((d + 1) ** 2)
    for i in range(x.shape[0]):
        lib().or_sh_basis(int(d), _p(np.ascontiguousarray(x[i]), C.c_double), _p(row, C.c_double))
        out[i] = row
    return out


def transfer_grid(n_theta=64, n_phi=128):
    """Lat-long directions [M, 3] and midpoint quadrature weights [M] of the transfer."""
    M = n_theta * n_phi
    D = np.zeros((M, 3))
    W = np.zeros(M)
    d3 = np.zeros(3)
    w = C.c_double(0.0)
    for j in range(M):
        lib().or_transfer_dir(n_theta, n_phi, j, _p(d3, C.c_double), C.byref(w))
        D[j] = d3
        W[j] = w.value
    return D, W


def sh_transfer(sh, d, normals, colors=None, n_theta=64, n_phi=128, q=1.0, eps=1e-6, s_max=4.0, gamma=1.0):
    """NEXT-4: per-channel scales s [n, 3] and relit colours [n, 3] (or None)."""
    A = _f64(sh).reshape(3, (d + 1) ** 2)
    nr = _f64(normals).reshape(-1, 3)
    n = nr.shape[0]
    col = None if colors is None else _f64(colors).reshape(-1, 3)
    s = np.zeros((n, 3))
    co = np.zeros((n, 3)) if col is not None else None
    lib().or_sh_transfer(_p(A, C.c_double), int(d), int(n_theta), int(n_phi), float(q), float(eps), float(s_max),
                         float(gamma), _p(nr, C.c_double), None if col is None else _p(col, C.c_double), n,
                         _p(s, C.c_double), None if co is None else _p(co, C.c_double))
    return s, co
