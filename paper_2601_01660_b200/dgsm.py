"""Thin ctypes binding of libdgsm.so (include/dgsm.h).

Argument marshalling only: every step of the DGSM build and query runs in the
library's CUDA kernels.  PyTorch supplies device memory (the caching
allocator), the current stream and nothing else.  There is no CPU fallback:
if the extension is missing or the tensors are not on a CUDA device, the calls
raise.

    atlas = build(gaussians, lights, atlas_res=512, n_shells=64)     # [L,K,H,W] T
    T = query(atlas, lights, positions)                               # [m]
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Dict, Optional, Sequence

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdgsm.so")

DGSM_MAX_LIGHTS = 64
DGSM_BIN_WRAP, DGSM_BIN_CLAMP = 0, 1
DGSM_OUTPUT_TAU = 1
DGSM_COLLECT_STATS = 2
DGSM_NO_TILE_CULL = 4
DGSM_VALIDATE = 8
ABSORPTION = {"traceavg": 0, "simple": 1, "mass": 2, "diag": 3}
_STATUS = {0: "DGSM_OK", 1: "DGSM_EINVAL", 2: "DGSM_ENOSPC", 3: "DGSM_ECUDA", 4: "DGSM_ERANGE", 5: "DGSM_EDATA"}

EXPORTED = ["dgsm_default_opts", "dgsm_plan_workspace_bytes", "dgsm_build_plan", "dgsm_build_run",
            "dgsm_build_bins", "dgsm_build", "dgsm_exp_epilogue", "dgsm_query", "dgsm_query_footprint", "dgsm_strerror",
            "dgsm_last_error", "dgsm_last_launch_count", "dgsm_build_stats", "dgsm_set_accumulate_events",
            "dgsm_slab_bytes", "dgsm_active_slab", "dgsm_frame_host", "dgsm_default_transfer_opts",
            "dgsm_transfer_workspace_bytes", "dgsm_sh_transfer", "dgsm_sort_temp_bytes", "dgsm_sort_pairs_u32",
            "dgsm_order_workspace_bytes", "dgsm_receiver_order", "dgsm_query_ordered", "dgsm_query_chunks",
            "dgsm_query_combine", "dgsm_async_workspace_bytes", "dgsm_build_async", "dgsm_footprint_stencil",
            "dgsm_set_frame_event"]


class Gaussians(C.Structure):
    _fields_ = [("means", C.c_void_p), ("scales", C.c_void_p), ("rotations", C.c_void_p),
                ("opacities", C.c_void_p), ("n", C.c_int64)]


class Light(C.Structure):
    _fields_ = [("position", C.c_float * 3), ("t_max", C.c_float)]


class BuildOpts(C.Structure):
    _fields_ = [("kappa", C.c_float), ("k_sigma", C.c_float), ("rho_scale", C.c_float),
                ("bin_mode", C.c_int32), ("flags", C.c_uint32), ("absorption", C.c_int32),
                ("slab", C.c_void_p)]


class TransferOpts(C.Structure):
    _fields_ = [("grid_theta", C.c_int32), ("grid_phi", C.c_int32), ("q", C.c_float), ("eps", C.c_float),
                ("s_max", C.c_float), ("gamma", C.c_float)]


class Roi(C.Structure):
    _fields_ = [("center", C.c_float * 3), ("radius", C.c_float), ("z_min", C.c_float), ("z_max", C.c_float)]


class Plan(C.Structure):
    _fields_ = [("n", C.c_int64), ("n_lights", C.c_int32), ("atlas_res", C.c_int32),
                ("n_shells", C.c_int32), ("chunk", C.c_int32), ("n_keys", C.c_int64),
                ("light_key_begin", C.c_int64 * (DGSM_MAX_LIGHTS + 1)),
                ("depth_min", C.c_uint32 * DGSM_MAX_LIGHTS), ("depth_max", C.c_uint32 * DGSM_MAX_LIGHTS),
                ("depth_bits", C.c_int32 * DGSM_MAX_LIGHTS), ("tile_bits", C.c_int32),
                ("run_workspace_bytes", C.c_size_t), ("signature", C.c_uint64)]


class BuildStatus(C.Structure):
    _fields_ = [("n_keys", C.c_uint64), ("overflow", C.c_uint32), ("n_invalid", C.c_uint32)]


class BuildStats(C.Structure):
    _fields_ = [("pairs", C.c_uint64), ("pairs_live", C.c_uint64), ("window_shells", C.c_uint64),
                ("steps", C.c_uint64), ("warp_records", C.c_uint64), ("warp_live_any", C.c_uint64),
                ("warp_live_max", C.c_uint64), ("band_records", C.c_uint64)]


class DgsmError(RuntimeError):
    pass


_lib = None


def lib() -> C.CDLL:
    """Load libdgsm.so (built by paper_2601_01660_b200.build_ext).  Raises if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise DgsmError(f"{LIB_PATH} not found: build it with `python -m paper_2601_01660_b200.build_ext` "
                            "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        vp, i64, sz = C.c_void_p, C.c_int64, C.c_size_t
        P = C.POINTER
        L.dgsm_default_opts.argtypes = [P(BuildOpts)]
        L.dgsm_default_opts.restype = None
        L.dgsm_plan_workspace_bytes.argtypes = [i64, C.c_int]
        L.dgsm_plan_workspace_bytes.restype = sz
        L.dgsm_build_plan.argtypes = [P(Gaussians), P(Light), C.c_int, C.c_int, C.c_int, P(BuildOpts),
                                      vp, sz, P(Plan), vp]
        L.dgsm_build_run.argtypes = [P(Gaussians), P(Light), C.c_int, P(BuildOpts), P(Plan), vp, sz, vp,
                                     sz, vp, vp]
        L.dgsm_build_bins.argtypes = [P(Gaussians), P(Light), C.c_int, P(BuildOpts), P(Plan), vp, sz, vp,
                                      sz, vp, vp, vp, vp, vp, vp, vp]
        L.dgsm_build.argtypes = [P(Gaussians), P(Light), C.c_int, C.c_int, C.c_int, P(BuildOpts), vp, sz,
                                 P(sz), vp, vp]
        L.dgsm_exp_epilogue.argtypes = [vp, vp, i64, vp]
        L.dgsm_query.argtypes = [vp, P(Light), C.c_int, C.c_int, C.c_int, vp, i64, vp, vp, vp]
        L.dgsm_query_footprint.argtypes = [vp, P(Light), C.c_int, C.c_int, C.c_int, vp, vp, vp, i64, vp, vp,
                                           C.c_int, vp, vp, vp]
        L.dgsm_frame_host.argtypes = [P(Gaussians), P(Light), C.c_int, C.c_int, C.c_int, P(BuildOpts), vp, i64,
                                      vp, vp, sz, P(sz), vp, vp]
        L.dgsm_frame_host.restype = C.c_int
        L.dgsm_default_transfer_opts.argtypes = [P(TransferOpts)]
        L.dgsm_default_transfer_opts.restype = None
        L.dgsm_transfer_workspace_bytes.argtypes = [P(TransferOpts), i64]
        L.dgsm_transfer_workspace_bytes.restype = sz
        L.dgsm_sh_transfer.argtypes = [vp, C.c_int, vp, vp, i64, P(TransferOpts), vp, vp, vp, sz, vp]
        L.dgsm_sh_transfer.restype = C.c_int
        L.dgsm_slab_bytes.argtypes = [C.c_int, C.c_int]
        L.dgsm_slab_bytes.restype = sz
        L.dgsm_active_slab.argtypes = [vp, i64, P(Roi), P(Light), C.c_int, C.c_int, C.c_int, vp, sz, vp]
        L.dgsm_active_slab.restype = C.c_int
        L.dgsm_order_workspace_bytes.argtypes = [i64]
        L.dgsm_order_workspace_bytes.restype = sz
        L.dgsm_receiver_order.argtypes = [vp, i64, vp, vp, sz, vp]
        L.dgsm_receiver_order.restype = C.c_int
        L.dgsm_query_ordered.argtypes = [vp, P(Light), C.c_int, C.c_int, C.c_int, vp, vp, i64, vp, vp, vp]
        L.dgsm_query_ordered.restype = C.c_int
        L.dgsm_query_chunks.argtypes = [P(vp), P(C.c_int32), P(C.c_int32), P(C.c_int32), P(Light), C.c_int,
                                        C.c_int, C.c_int, vp, i64, vp, vp, vp]
        L.dgsm_query_chunks.restype = C.c_int
        L.dgsm_query_combine.argtypes = [vp, C.c_int, i64, vp, vp]
        L.dgsm_query_combine.restype = C.c_int
        L.dgsm_async_workspace_bytes.argtypes = [i64, C.c_int, C.c_int, C.c_int, i64]
        L.dgsm_async_workspace_bytes.restype = sz
        L.dgsm_build_async.argtypes = [P(Gaussians), P(Light), C.c_int, C.c_int, C.c_int, P(BuildOpts), i64, vp, sz,
                                       vp, vp, vp]
        L.dgsm_build_async.restype = C.c_int
        L.dgsm_footprint_stencil.argtypes = [C.c_int, C.c_float, vp, vp, P(C.c_int)]
        L.dgsm_footprint_stencil.restype = C.c_int
        L.dgsm_sort_temp_bytes.argtypes = [i64]
        L.dgsm_sort_temp_bytes.restype = sz
        L.dgsm_sort_pairs_u32.argtypes = [vp, vp, vp, vp, i64, C.c_int, vp, sz, P(C.c_int), vp]
        L.dgsm_sort_pairs_u32.restype = C.c_int
        L.dgsm_strerror.argtypes = [C.c_int]
        L.dgsm_strerror.restype = C.c_char_p
        L.dgsm_last_error.argtypes = []
        L.dgsm_last_error.restype = C.c_char_p
        L.dgsm_last_launch_count.argtypes = []
        L.dgsm_last_launch_count.restype = C.c_int
        L.dgsm_build_stats.argtypes = [P(Plan), vp, sz, P(BuildStats), vp]
        L.dgsm_build_stats.restype = C.c_int
        L.dgsm_set_accumulate_events.argtypes = [vp, vp]
        L.dgsm_set_accumulate_events.restype = C.c_int
        L.dgsm_set_frame_event.argtypes = [vp]
        L.dgsm_set_frame_event.restype = C.c_int
        for f in ("dgsm_build_plan", "dgsm_build_run", "dgsm_build_bins", "dgsm_build",
                  "dgsm_exp_epilogue", "dgsm_query", "dgsm_query_footprint"):
            getattr(L, f).restype = C.c_int
        _lib = L
    return _lib


def _check(rc: int, what: str):
    if rc != 0:
        msg = lib().dgsm_last_error().decode(errors="replace")
        raise DgsmError(f"{what}: {_STATUS.get(rc, rc)}: {msg}")


def last_launch_count() -> int:
    return int(lib().dgsm_last_launch_count())


# ----------------------------------------------------------------- helpers
def _dev_f32(t: torch.Tensor, name: str, shape_tail) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise DgsmError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if t.dtype != torch.float32:
        raise DgsmError(f"{name} must be float32")
    if tuple(t.shape[1:]) != tuple(shape_tail):
        raise DgsmError(f"{name} has shape {tuple(t.shape)}, expected [n, {shape_tail}]")
    return t.contiguous()


def _out_f32(t: Optional[torch.Tensor], shape, device, name: str) -> torch.Tensor:
    """An output buffer the library writes: a new tensor, or a caller tensor
    checked to be contiguous float32 of exactly `shape` on `device` (the C ABI
    takes raw pointers and cannot check sizes itself)."""
    if t is None:
        return torch.empty(shape, dtype=torch.float32, device=device)
    if not isinstance(t, torch.Tensor) or t.dtype != torch.float32 or not t.is_contiguous():
        raise DgsmError(f"{name} must be a contiguous float32 tensor")
    if t.device != torch.device(device):
        raise DgsmError(f"{name} is on {t.device}, expected {device}")
    if tuple(t.shape) != tuple(shape):
        raise DgsmError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")
    return t


def _gaussians(g: Dict[str, torch.Tensor]):
    m = _dev_f32(g["means"], "means", (3,))
    s = _dev_f32(g["scales"], "scales", (3,))
    q = _dev_f32(g["rotations"], "rotations", (4,))
    a = g["opacities"]
    if a.dim() == 2:
        a = a.reshape(-1)
    a = _dev_f32(a, "opacities", ())
    n = m.shape[0]
    if not (s.shape[0] == q.shape[0] == a.shape[0] == n):
        raise DgsmError("Gaussian arrays disagree on n")
    keep = (m, s, q, a)
    return Gaussians(m.data_ptr(), s.data_ptr(), q.data_ptr(), a.data_ptr(), n), keep


def lights_array(lights) -> np.ndarray:
    """lights: dict(position [L,3], t_max [L]) or array [L,4] (x, y, z, t_max)."""
    if isinstance(lights, dict):
        pos = np.asarray(lights["position"], np.float32).reshape(-1, 3)
        tm = np.asarray(lights["t_max"], np.float32).reshape(-1)
        return np.concatenate([pos, tm[:, None]], 1).astype(np.float32)
    a = np.asarray(lights, np.float32)
    return a.reshape(-1, 4)


def _lights(lights):
    a = lights_array(lights)
    L = a.shape[0]
    if not 1 <= L <= DGSM_MAX_LIGHTS:
        raise DgsmError(f"n_lights={L} outside [1, {DGSM_MAX_LIGHTS}]")
    arr = (Light * L)()
    for l in range(L):
        arr[l].position[0], arr[l].position[1], arr[l].position[2] = (float(x) for x in a[l, :3])
        arr[l].t_max = float(a[l, 3])
    return arr, L


@dataclass
class Options:
    """Build options (include/dgsm.h dgsm_build_opts_t)."""
    kappa: float = 1.0
    k_sigma: float = 3.0
    rho_scale: float = 1.0
    bin_mode: str = "wrap"
    output_tau: bool = False
    collect_stats: bool = False
    absorption: str = "traceavg"   # traceavg (Eq.5) | simple | mass | diag (ablation B)
    tile_cull: bool = True         # False: ablation D, every Gaussian in every tile
    validate: bool = False         # DGSM_VALIDATE: reject non-finite / degenerate Gaussians (DGSM_EDATA)
    slab: Optional[torch.Tensor] = None  # NEXT-1 ROI slab from active_slab(); None = full atlas

    def c(self) -> BuildOpts:
        if self.absorption not in ABSORPTION:
            raise DgsmError(f"absorption must be one of {sorted(ABSORPTION)}")
        return BuildOpts(self.kappa, self.k_sigma, self.rho_scale,
                         DGSM_BIN_WRAP if self.bin_mode == "wrap" else DGSM_BIN_CLAMP,
                         (DGSM_OUTPUT_TAU if self.output_tau else 0) |
                         (DGSM_COLLECT_STATS if self.collect_stats else 0) |
                         (0 if self.tile_cull else DGSM_NO_TILE_CULL) |
                         (DGSM_VALIDATE if self.validate else 0),
                         ABSORPTION[self.absorption],
                         None if self.slab is None else C.c_void_p(self.slab.data_ptr()))


def _stream_ptr(stream: Optional[torch.cuda.Stream]) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def _alloc(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)


class BuildPlan:
    """Result of dgsm_build_plan: keeps the device workspace and the host plan."""

    def __init__(self, gaussians, lights, atlas_res: int, n_shells: int, opts: Optional[Options] = None,
                 stream=None):
        self.opts = opts or Options()
        self._g, self._keep = _gaussians(gaussians)
        self._lights, self.n_lights = _lights(lights)
        self._opts_c = self.opts.c()
        self.device = self._keep[0].device
        self.atlas_res, self.n_shells = int(atlas_res), int(n_shells)
        nbytes = lib().dgsm_plan_workspace_bytes(self._g.n, self.n_lights)
        self.plan_ws = _alloc(nbytes, self.device)
        self.plan = Plan()
        rc = lib().dgsm_build_plan(C.byref(self._g), self._lights, self.n_lights, self.atlas_res,
                                   self.n_shells, C.byref(self._opts_c), C.c_void_p(self.plan_ws.data_ptr()),
                                   self.plan_ws.numel(), C.byref(self.plan), C.c_void_p(_stream_ptr(stream)))
        _check(rc, "dgsm_build_plan")
        self.plan_launches = last_launch_count()
        self.run_ws = None

    @property
    def n_keys(self) -> int:
        return int(self.plan.n_keys)

    def light_key_ranges(self):
        return [(int(self.plan.light_key_begin[l]), int(self.plan.light_key_begin[l + 1]))
                for l in range(self.n_lights)]

    def _ensure_run_ws(self):
        need = int(self.plan.run_workspace_bytes)
        if self.run_ws is None or self.run_ws.numel() < need:
            self.run_ws = _alloc(need, self.device)
        return self.run_ws

    def run(self, out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
        shape = (self.n_lights, self.n_shells, self.atlas_res, self.atlas_res)
        out = _out_f32(out, shape, self.device, "out")
        ws = self._ensure_run_ws()
        rc = lib().dgsm_build_run(C.byref(self._g), self._lights, self.n_lights, C.byref(self._opts_c),
                                  C.byref(self.plan), C.c_void_p(self.plan_ws.data_ptr()), self.plan_ws.numel(),
                                  C.c_void_p(ws.data_ptr()), ws.numel(), C.c_void_p(out.data_ptr()),
                                  C.c_void_p(_stream_ptr(stream)))
        _check(rc, "dgsm_build_run")
        self.run_launches = last_launch_count()
        return out

    def stats(self, stream=None) -> dict:
        """Work counters of the last run (needs Options(collect_stats=True))."""
        st = BuildStats()
        ws = self._ensure_run_ws()
        rc = lib().dgsm_build_stats(C.byref(self.plan), C.c_void_p(ws.data_ptr()), ws.numel(), C.byref(st),
                                    C.c_void_p(_stream_ptr(stream)))
        _check(rc, "dgsm_build_stats")
        return {f: int(getattr(st, f)) for f, _ in BuildStats._fields_}

    def bins(self, stream=None):
        """Sorted (light, tile, depth_bits, index) uint32 arrays + tile ranges (device int64 views)."""
        P = self.n_keys
        outs = [torch.empty(max(P, 1), dtype=torch.int32, device=self.device) for _ in range(4)]
        nt = self.n_lights * (self.atlas_res // 8) ** 2
        ts = torch.empty(nt, dtype=torch.int32, device=self.device)
        te = torch.empty(nt, dtype=torch.int32, device=self.device)
        ws = self._ensure_run_ws()
        rc = lib().dgsm_build_bins(C.byref(self._g), self._lights, self.n_lights, C.byref(self._opts_c),
                                   C.byref(self.plan), C.c_void_p(self.plan_ws.data_ptr()), self.plan_ws.numel(),
                                   C.c_void_p(ws.data_ptr()), ws.numel(),
                                   *[C.c_void_p(o.data_ptr()) for o in outs],
                                   C.c_void_p(ts.data_ptr()), C.c_void_p(te.data_ptr()),
                                   C.c_void_p(_stream_ptr(stream)))
        _check(rc, "dgsm_build_bins")
        u32 = lambda t: (t.to(torch.int64) & 0xFFFFFFFF)
        return tuple(u32(o[:P]) for o in outs), (u32(ts), u32(te))


class Builder:
    """dgsm_build (plan + run in one C call, one host synchronisation inside)
    with a device workspace kept across frames: the per-frame entry point of a
    renderer (no Python between the plan's key count and the run's launches)."""

    def __init__(self, lights, atlas_res: int, n_shells: int, opts: Optional[Options] = None, device="cuda"):
        self.lights, self.n_lights = _lights(lights)
        self.res, self.K = int(atlas_res), int(n_shells)
        self.opts = opts or Options()
        self._oc = self.opts.c()
        self.device = torch.device(device)
        self.ws = _alloc(0, self.device)

    def __call__(self, gaussians, out: torch.Tensor, stream=None) -> torch.Tensor:
        g, keep = _gaussians(gaussians)
        if not isinstance(out, torch.Tensor):
            raise DgsmError("out must be a tensor")
        out = _out_f32(out, (self.n_lights, self.K, self.res, self.res), keep[0].device, "out")
        need = C.c_size_t(0)
        for _ in range(3):
            rc = lib().dgsm_build(C.byref(g), self.lights, self.n_lights, self.res, self.K, C.byref(self._oc),
                                  C.c_void_p(self.ws.data_ptr()), self.ws.numel(), C.byref(need),
                                  C.c_void_p(out.data_ptr()), C.c_void_p(_stream_ptr(stream)))
            if rc != 2:  # DGSM_ENOSPC: grow and retry
                break
            self.ws = _alloc(int(need.value * 1.25) + (1 << 20), self.device)
        _check(rc, "dgsm_build")
        self.launches = last_launch_count()
        return out


class AsyncBuilder:
    """dgsm_build_async: the sync-free build (no host synchronisation, capturable
    in a CUDA graph) with a workspace sized for `key_capacity` keys.  The device
    status (keys, overflow, invalid) of the last build is read by status()."""

    def __init__(self, lights, atlas_res: int, n_shells: int, n: int, key_capacity: int,
                 opts: Optional[Options] = None, device="cuda"):
        self.lights, self.n_lights = _lights(lights)
        self.res, self.K, self.n = int(atlas_res), int(n_shells), int(n)
        self.opts = opts or Options()
        self._oc = self.opts.c()
        self.device = torch.device(device)
        self.key_capacity = int(key_capacity)
        need = lib().dgsm_async_workspace_bytes(self.n, self.n_lights, self.res, self.K, self.key_capacity)
        if need == 0:
            raise DgsmError("bad sizes for dgsm_build_async")
        self.ws = _alloc(need, self.device)
        self.status_buf = torch.zeros(16, dtype=torch.uint8, device=self.device)

    def __call__(self, gaussians, out: torch.Tensor, stream=None) -> torch.Tensor:
        g, keep = _gaussians(gaussians)
        if g.n != self.n:
            raise DgsmError(f"AsyncBuilder sized for n={self.n}, got {g.n}")
        out = _out_f32(out, (self.n_lights, self.K, self.res, self.res), keep[0].device, "out")
        rc = lib().dgsm_build_async(C.byref(g), self.lights, self.n_lights, self.res, self.K, C.byref(self._oc),
                                    self.key_capacity, C.c_void_p(self.ws.data_ptr()), self.ws.numel(),
                                    C.c_void_p(out.data_ptr()), C.c_void_p(self.status_buf.data_ptr()),
                                    C.c_void_p(_stream_ptr(stream)))
        _check(rc, "dgsm_build_async")
        self.launches = last_launch_count()
        return out

    def status(self) -> dict:
        b = self.status_buf.cpu().numpy()
        st = BuildStatus.from_buffer_copy(b.tobytes())
        return {"n_keys": int(st.n_keys), "overflow": bool(st.overflow), "n_invalid": int(st.n_invalid)}


def build(gaussians: Dict[str, torch.Tensor], lights, atlas_res: int, n_shells: int,
          opts: Optional[Options] = None, out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """DGSM build (§3.2): atlas [L, K, H, W] float32 of T = exp(-tau) (or tau)."""
    return BuildPlan(gaussians, lights, atlas_res, n_shells, opts, stream).run(out, stream)


def exp_epilogue(tau: torch.Tensor, out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """T = exp(-tau) (Eq.4), elementwise on the device; out may alias tau."""
    if not tau.is_cuda or tau.dtype != torch.float32 or not tau.is_contiguous():
        raise DgsmError("tau must be a contiguous float32 CUDA tensor")
    out = _out_f32(out, tuple(tau.shape), tau.device, "out")
    rc = lib().dgsm_exp_epilogue(C.c_void_p(tau.data_ptr()), C.c_void_p(out.data_ptr()), tau.numel(),
                                 C.c_void_p(_stream_ptr(stream)))
    _check(rc, "dgsm_exp_epilogue")
    return out


def receiver_order(positions: torch.Tensor, out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """Spatially coherent visiting order of the receivers (dgsm_receiver_order):
    int32 CUDA tensor [m] holding the permutation (Morton order of the positions)."""
    x = _dev_f32(positions, "positions", (3,))
    m = x.shape[0]
    if out is None:
        out = torch.empty(m, dtype=torch.int32, device=x.device)
    elif out.dtype != torch.int32 or not out.is_contiguous() or out.numel() != m or out.device != x.device:
        raise DgsmError("order out must be a contiguous int32 tensor [m] on the receivers' device")
    ws = _alloc(lib().dgsm_order_workspace_bytes(m), x.device)
    rc = lib().dgsm_receiver_order(C.c_void_p(x.data_ptr()), m, C.c_void_p(out.data_ptr()),
                                   C.c_void_p(ws.data_ptr()), ws.numel(), C.c_void_p(_stream_ptr(stream)))
    _check(rc, "dgsm_receiver_order")
    return out


def query(atlas: torch.Tensor, lights, positions: torch.Tensor, colors: Optional[torch.Tensor] = None,
          out: Optional[torch.Tensor] = None, stream=None, order: Optional[torch.Tensor] = None) -> torch.Tensor:
    """DGSM sampling (§3.3): T[m] = prod_l trilinear(atlas_l, x); colors *= T in place.
    ``order`` (from receiver_order): visit the receivers in that order
    (dgsm_query_ordered; bit-identical results, coherent memory access)."""
    if not atlas.is_cuda or atlas.dtype != torch.float32 or atlas.dim() != 4 or not atlas.is_contiguous():
        raise DgsmError("atlas must be a contiguous float32 CUDA tensor [L, K, H, W]")
    L, K, H, W = atlas.shape
    if H != W:
        raise DgsmError("square atlases only")
    arr, nl = _lights(lights)
    if nl != L:
        raise DgsmError(f"atlas has {L} lights, got {nl}")
    x = _dev_f32(positions, "positions", (3,))
    m = x.shape[0]
    if x.device != atlas.device:
        raise DgsmError("positions and atlas must be on the same device")
    out = _out_f32(out, (m,), x.device, "out")
    cptr = None
    if colors is not None:
        cptr = C.c_void_p(_out_f32(colors, (m, 3), x.device, "colors").data_ptr())
    if order is not None:
        if order.dtype != torch.int32 or not order.is_contiguous() or order.numel() != m or order.device != x.device:
            raise DgsmError("order must be a contiguous int32 tensor [m] on the receivers' device")
        rc = lib().dgsm_query_ordered(C.c_void_p(atlas.data_ptr()), arr, nl, int(H), int(K), C.c_void_p(x.data_ptr()),
                                      C.c_void_p(order.data_ptr()), m, C.c_void_p(out.data_ptr()), cptr,
                                      C.c_void_p(_stream_ptr(stream)))
        _check(rc, "dgsm_query_ordered")
        return out
    rc = lib().dgsm_query(C.c_void_p(atlas.data_ptr()), arr, nl, int(H), int(K), C.c_void_p(x.data_ptr()), m,
                          C.c_void_p(out.data_ptr()), cptr, C.c_void_p(_stream_ptr(stream)))
    _check(rc, "dgsm_query")
    return out


def query_chunks(chunks, lights, positions: torch.Tensor, res: int, K: int, stream=None):
    """Sharded-atlas query (dgsm_query_chunks, multi-GPU): ``chunks`` lists, per
    light of ``lights``, (k_begin, k_end, split, tensor [k_end-k_begin, res, res]
    or None).  Returns (T [m]: product over the complete lights, partial
    [n_split, m]: each split light's share of its trilinear sample)."""
    arr, nl = _lights(lights)
    if len(chunks) != nl:
        raise DgsmError(f"{len(chunks)} chunks for {nl} lights")
    x = _dev_f32(positions, "positions", (3,))
    m = x.shape[0]
    ptrs = (C.c_void_p * nl)()
    kb, ke, sp = (C.c_int32 * nl)(), (C.c_int32 * nl)(), (C.c_int32 * nl)()
    for l, (b, e, split, t) in enumerate(chunks):
        if e > b:
            if t is None or t.dtype != torch.float32 or not t.is_contiguous() or t.device != x.device or \
                    tuple(t.shape) != (e - b, res, res):
                raise DgsmError(f"chunk {l} must be contiguous float32 [{e - b}, {res}, {res}] on {x.device}")
            ptrs[l] = t.data_ptr()
        kb[l], ke[l], sp[l] = int(b), int(e), int(bool(split))
    n_split = sum(1 for c in chunks if c[2])
    T = torch.empty(m, dtype=torch.float32, device=x.device)
    part = torch.empty((max(n_split, 1), m), dtype=torch.float32, device=x.device)
    rc = lib().dgsm_query_chunks(ptrs, kb, ke, sp, arr, nl, int(res), int(K), C.c_void_p(x.data_ptr()), m,
                                 C.c_void_p(T.data_ptr()), C.c_void_p(part.data_ptr()),
                                 C.c_void_p(_stream_ptr(stream)))
    _check(rc, "dgsm_query_chunks")
    return T, part[:n_split]


def query_combine(partial: torch.Tensor, T: torch.Tensor, stream=None) -> torch.Tensor:
    """T *= prod_j partial[j] in place (dgsm_query_combine)."""
    m = T.numel()
    T = _out_f32(T, (m,), T.device, "T")
    n = partial.shape[0] if partial.dim() == 2 else 0
    if n:
        partial = _out_f32(partial.contiguous(), (n, m), T.device, "partial")
    rc = lib().dgsm_query_combine(C.c_void_p(partial.data_ptr()) if n else None, n, m, C.c_void_p(T.data_ptr()),
                                  C.c_void_p(_stream_ptr(stream)))
    _check(rc, "dgsm_query_combine")
    return T


DGSM_MAX_FOOTPRINT_SAMPLES = 64


def sh_transfer(sh, sh_degree: int, normals: torch.Tensor, colors: Optional[torch.Tensor] = None,
                grid=(64, 128), q: float = 1.0, eps: float = 1e-6, s_max: float = 4.0, gamma: float = 1.0,
                stream=None):
    """NEXT-4 SH lighting transfer (§3.5): per-channel scales
    s [n, 3] of unit normals (CUDA float32 [n, 3]) under the SH probe ``sh``
    (host [3, (d+1)^2]); with ``colors`` (CUDA [n, 3]) also the relit colours
    max(0, gamma c * s).  Returns (scales, colors_out or None)."""
    nr = _dev_f32(normals, "normals", (3,))
    n = nr.shape[0]
    A = np.ascontiguousarray(np.asarray(sh, np.float32).reshape(3, (sh_degree + 1) ** 2))
    o = TransferOpts(int(grid[0]), int(grid[1]), float(q), float(eps), float(s_max), float(gamma))
    col = None if colors is None else _dev_f32(colors, "colors", (3,))
    scales = torch.empty((n, 3), dtype=torch.float32, device=nr.device)
    cout = torch.empty((n, 3), dtype=torch.float32, device=nr.device) if col is not None else None
    ws = _alloc(lib().dgsm_transfer_workspace_bytes(C.byref(o), n), nr.device)
    rc = lib().dgsm_sh_transfer(A.ctypes.data_as(C.c_void_p), int(sh_degree), C.c_void_p(nr.data_ptr()),
                                None if col is None else C.c_void_p(col.data_ptr()), n, C.byref(o),
                                C.c_void_p(scales.data_ptr()), None if cout is None else C.c_void_p(cout.data_ptr()),
                                C.c_void_p(ws.data_ptr()), ws.numel(), C.c_void_p(_stream_ptr(stream)))
    _check(rc, "dgsm_sh_transfer")
    return scales, cout


class FrameHost:
    """dgsm_frame_host: one frame (build + query) from HOST tensors (pinned for
    overlap), the device workspace kept across calls.  Returns the device atlas;
    ``T_host`` (CPU float32 [m]) is filled when the stream completes."""

    def __init__(self, lights, atlas_res: int, n_shells: int, opts: Optional[Options] = None, device="cuda"):
        self.lights, self.n_lights = _lights(lights)
        self.res, self.K = int(atlas_res), int(n_shells)
        self.opts = opts or Options()
        self._oc = self.opts.c()
        self.device = torch.device(device)
        # two workspaces used alternately: frame i+1's uploads only wait for frame i-1
        # (the library orders uploads after the previous frame in the same workspace)
        self.wss = [_alloc(0, self.device), _alloc(0, self.device)]
        self.frame = 0
        self.atlas = torch.empty((self.n_lights, self.K, self.res, self.res), dtype=torch.float32,
                                 device=self.device)

    def __call__(self, g_host: Dict[str, torch.Tensor], receivers_host: torch.Tensor, T_host: torch.Tensor,
                 stream=None) -> torch.Tensor:
        arrs = [g_host[k] for k in ("means", "scales", "rotations", "opacities")]
        for a in arrs + [receivers_host, T_host]:
            if a.is_cuda or a.dtype != torch.float32 or not a.is_contiguous():
                raise DgsmError("frame_host takes contiguous float32 CPU tensors")
        n, m = arrs[0].shape[0], receivers_host.shape[0]
        tails = ((3,), (3,), (4,), ())
        for name, a, tail in zip(("means", "scales", "rotations", "opacities"), arrs, tails):
            if a.shape[0] != n or tuple(a.shape[1:]) not in (tail, (1,) if tail == () else tail):
                raise DgsmError(f"{name} has shape {tuple(a.shape)}, expected [{n}, {tail}]")
        if tuple(receivers_host.shape) != (m, 3):
            raise DgsmError("receivers must be [m, 3]")
        if T_host.numel() < m:
            raise DgsmError(f"T_host holds {T_host.numel()} floats, needs {m}")
        g = Gaussians(*[C.c_void_p(a.data_ptr()) for a in arrs], n)
        need = C.c_size_t(0)
        k = self.frame & 1
        self.frame += 1
        for _ in range(3):
            ws = self.wss[k]
            rc = lib().dgsm_frame_host(C.byref(g), self.lights, self.n_lights, self.res, self.K, C.byref(self._oc),
                                       C.c_void_p(receivers_host.data_ptr()), m, C.c_void_p(T_host.data_ptr()),
                                       C.c_void_p(ws.data_ptr()), ws.numel(), C.byref(need),
                                       C.c_void_p(self.atlas.data_ptr()), C.c_void_p(_stream_ptr(stream)))
            if rc != 2:  # DGSM_ENOSPC: grow the workspace and retry
                break
            self.wss[k] = _alloc(int(need.value * 1.25) + (1 << 20), self.device)
        _check(rc, "dgsm_frame_host")
        self.launches = last_launch_count()
        return self.atlas


class FrameStream:
    """Frames back to back from HOST tensors (a renderer's frame loop): per frame the
    occluders and receivers go up on a copy stream into one of two device buffer
    sets, the sync-free build (dgsm_build_async, `key_capacity` keys) and the query
    run as ONE CUDA-graph replay (one graph per buffer set, captured on first use),
    and T comes back on a second copy stream from one of two device buffers.  Frame
    i+1's receivers go up as soon as its buffer set is free, its Gaussians when frame
    i's accumulation starts (dgsm_set_frame_event: an external event recorded inside
    the graph), so the bulk of the upload overlaps the FP32-bound a6 kernel instead of
    the L2-resident sorts.  Pinned host tensors give the overlap.

    The call returns an event: T_host is complete once it has (``wait()`` waits for
    every frame issued); the atlas of the latest frame is ``atlas``.  ``status()``
    is the sync-free build's status of the latest frame (key overflow)."""

    def __init__(self, lights, atlas_res: int, n_shells: int, n: int, m: int, key_capacity: int,
                 opts: Optional[Options] = None, device="cuda"):
        self.lights, self.n_lights = _lights(lights)
        self._lights_arg = lights
        self.res, self.K, self.n, self.m = int(atlas_res), int(n_shells), int(n), int(m)
        self.device = torch.device(device)
        self.builder = AsyncBuilder(lights, atlas_res, n_shells, n, key_capacity, opts, device)
        dev = self.device
        shapes = {"means": (n, 3), "scales": (n, 3), "rotations": (n, 4), "opacities": (n,)}
        self.bufs = [({k: torch.empty(v, dtype=torch.float32, device=dev) for k, v in shapes.items()},
                      torch.empty((m, 3), dtype=torch.float32, device=dev)) for _ in range(2)]
        self.Tdev = [torch.empty(m, dtype=torch.float32, device=dev) for _ in range(2)]
        self.atlas = torch.empty((self.n_lights, self.K, self.res, self.res), dtype=torch.float32, device=dev)
        self.up, self.down = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        self.ev_acc = [torch.cuda.Event(external=True) for _ in range(2)]
        self.ev_up, self.ev_used, self.ev_down = ([torch.cuda.Event() for _ in range(2)] for _ in range(3))
        cur = torch.cuda.current_stream(dev)
        for e in self.ev_acc + self.ev_up + self.ev_used + self.ev_down:
            e.record(cur)
        self.graphs = [None, None]
        self.frame = 0
        self.launches = 0

    def _frame_body(self, k):
        g, x = self.bufs[k]
        self.builder(g, self.atlas)
        nl = self.builder.launches
        query(self.atlas, self._lights_arg, x, out=self.Tdev[k])
        return nl + last_launch_count()

    def _capture(self, k):
        side = torch.cuda.Stream(self.device)
        side.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(side):
            self.launches = self._frame_body(k)  # warm-up run (also counts the kernels)
        torch.cuda.current_stream(self.device).wait_stream(side)
        graph = torch.cuda.CUDAGraph()
        lib().dgsm_set_frame_event(C.c_void_p(self.ev_acc[k].cuda_event))
        try:
            with torch.cuda.graph(graph, stream=side):
                self._frame_body(k)
        finally:
            lib().dgsm_set_frame_event(None)
        self.graphs[k] = graph

    def __call__(self, g_host: Dict[str, torch.Tensor], receivers_host: torch.Tensor,
                 T_host: torch.Tensor) -> torch.cuda.Event:
        for name, shp in (("means", (self.n, 3)), ("scales", (self.n, 3)), ("rotations", (self.n, 4))):
            a = g_host[name]
            if a.is_cuda or a.dtype != torch.float32 or tuple(a.shape) != shp or not a.is_contiguous():
                raise DgsmError(f"{name} must be a contiguous float32 CPU tensor of shape {shp}")
        op = g_host["opacities"]
        if op.is_cuda or op.dtype != torch.float32 or op.numel() != self.n or not op.is_contiguous():
            raise DgsmError(f"opacities must be a contiguous float32 CPU tensor of {self.n} values")
        if receivers_host.is_cuda or tuple(receivers_host.shape) != (self.m, 3) or receivers_host.dtype != torch.float32:
            raise DgsmError(f"receivers must be a float32 CPU tensor of shape ({self.m}, 3)")
        if T_host.is_cuda or T_host.dtype != torch.float32 or T_host.numel() < self.m:
            raise DgsmError(f"T_host must be a float32 CPU tensor of at least {self.m} values")
        k = self.frame & 1
        self.frame += 1
        cur = torch.cuda.current_stream(self.device)
        g, x = self.bufs[k]
        self.up.wait_event(self.ev_used[k])       # graph k's last replay has read buffer set k
        with torch.cuda.stream(self.up):          # the receivers first (12 B each, read last)
            x.copy_(receivers_host, non_blocking=True)
        self.up.wait_event(self.ev_acc[1 - k])    # the previous frame's accumulation has started
        with torch.cuda.stream(self.up):
            for name in ("means", "scales", "rotations", "opacities"):
                g[name].copy_(g_host[name].reshape(g[name].shape), non_blocking=True)
            self.ev_up[k].record(self.up)
        cur.wait_event(self.ev_up[k])
        cur.wait_event(self.ev_down[k])            # T buffer k has been copied out
        if self.graphs[k] is None:                 # first use of buffer set k: capture (on its data)
            self._capture(k)
        self.graphs[k].replay()
        self.ev_used[k].record(cur)
        self.down.wait_event(self.ev_used[k])
        with torch.cuda.stream(self.down):
            T_host[:self.m].copy_(self.Tdev[k], non_blocking=True)
            self.ev_down[k].record(self.down)
        return self.ev_down[k]

    def wait(self):
        """Block until every issued frame's T_host is complete."""
        for e in self.ev_down:
            e.synchronize()

    def status(self) -> dict:
        return self.builder.status()


def active_slab(receivers: torch.Tensor, roi, lights, atlas_res: int, n_shells: int,
                out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """NEXT-1: the voxel slab of the receivers (CUDA
    float32 [m, 3]) inside B = {||(x - c)_xy||_inf <= R, z_min <= z <= z_max}.
    ``roi`` = (c_x, c_y, c_z, R, z_min, z_max).  Returns the device slab buffer
    (uint8, include/dgsm.h layout) to pass as Options(slab=...)."""
    x = _dev_f32(receivers, "receivers", (3,))
    arr, nl = _lights(lights)
    need = int(lib().dgsm_slab_bytes(nl, int(atlas_res)))
    if need == 0:
        raise DgsmError("bad n_lights or atlas_res for a slab")
    if out is None:
        out = torch.empty(need, dtype=torch.uint8, device=x.device)
    r = [float(v) for v in roi]
    croi = Roi((C.c_float * 3)(*r[:3]), r[3], r[4], r[5])
    rc = lib().dgsm_active_slab(C.c_void_p(x.data_ptr()), x.shape[0], C.byref(croi), arr, nl, int(atlas_res),
                                int(n_shells), C.c_void_p(out.data_ptr()), out.numel(),
                                C.c_void_p(_stream_ptr(stream)))
    _check(rc, "dgsm_active_slab")
    return out


def footprint_stencil(kind: str = "stencil7", delta: float = 1.0):
    """Standard-normal footprint samples for query_footprint (NEXT-2),
    from the library (dgsm_footprint_stencil): "center" = the single point z = 0;
    "stencil7" = {0, +-delta e_j} weighted by exp(-|z|^2/2), normalised."""
    kinds = {"center": 0, "stencil7": 1}
    if kind not in kinds:
        raise DgsmError(f"unknown footprint stencil {kind!r}")
    z = np.zeros((7, 3), np.float32)
    w = np.zeros(7, np.float32)
    n = C.c_int(0)
    rc = lib().dgsm_footprint_stencil(kinds[kind], float(delta), z.ctypes.data_as(C.c_void_p),
                                      w.ctypes.data_as(C.c_void_p), C.byref(n))
    _check(rc, "dgsm_footprint_stencil")
    return z[:n.value].copy(), w[:n.value].copy()


def query_footprint(atlas: torch.Tensor, lights, gaussians, offsets, weights,
                    colors: Optional[torch.Tensor] = None, out: Optional[torch.Tensor] = None,
                    stream=None) -> torch.Tensor:
    """Footprint-averaged DGSM sampling (NEXT-2): for receiver Gaussian g,
    T[g] = prod_l sum_i w_i T_l(mu_g + R_g (s_g * z_i)).  `gaussians` is a dict
    of CUDA float32 means [m,3], scales [m,3], rotations [m,4]; offsets [n,3]
    and weights [n] are host arrays (n <= 64)."""
    if not atlas.is_cuda or atlas.dtype != torch.float32 or atlas.dim() != 4 or not atlas.is_contiguous():
        raise DgsmError("atlas must be a contiguous float32 CUDA tensor [L, K, H, W]")
    L, K, H, W = atlas.shape
    if H != W:
        raise DgsmError("square atlases only")
    arr, nl = _lights(lights)
    if nl != L:
        raise DgsmError(f"atlas has {L} lights, got {nl}")
    mu = _dev_f32(gaussians["means"], "means", (3,))
    sc = _dev_f32(gaussians["scales"], "scales", (3,))
    q = _dev_f32(gaussians["rotations"], "rotations", (4,))
    m = mu.shape[0]
    if sc.shape[0] != m or q.shape[0] != m:
        raise DgsmError("means, scales and rotations must have the same length")
    z = np.ascontiguousarray(np.asarray(offsets, np.float32).reshape(-1, 3))
    w = np.ascontiguousarray(np.asarray(weights, np.float32).reshape(-1))
    if len(z) != len(w) or not 1 <= len(w) <= DGSM_MAX_FOOTPRINT_SAMPLES:
        raise DgsmError(f"need 1..{DGSM_MAX_FOOTPRINT_SAMPLES} offsets with one weight each")
    if mu.device != atlas.device:
        raise DgsmError("receivers and atlas must be on the same device")
    out = _out_f32(out, (m,), mu.device, "out")
    cptr = None
    if colors is not None:
        cptr = C.c_void_p(_out_f32(colors, (m, 3), mu.device, "colors").data_ptr())
    rc = lib().dgsm_query_footprint(C.c_void_p(atlas.data_ptr()), arr, nl, int(H), int(K),
                                    C.c_void_p(mu.data_ptr()), C.c_void_p(sc.data_ptr()), C.c_void_p(q.data_ptr()),
                                    m, z.ctypes.data_as(C.c_void_p), w.ctypes.data_as(C.c_void_p), len(w),
                                    C.c_void_p(out.data_ptr()), cptr, C.c_void_p(_stream_ptr(stream)))
    _check(rc, "dgsm_query_footprint")
    return out


def sort_pairs(keys: torch.Tensor, vals: torch.Tensor, nbits: int, stream=None):
    """a4's stable onesweep radix sort of (key, value) uint32 pairs by key bits
    [0, nbits) (int32 CUDA tensors holding the uint32 bit patterns).  Returns
    the sorted (keys, vals) as new tensors; the inputs are used as scratch."""
    for t, nm in ((keys, "keys"), (vals, "vals")):
        if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.int32 or not t.is_contiguous() \
                or t.dim() != 1:
            raise DgsmError(f"{nm} must be a contiguous 1-D int32 CUDA tensor")
    n = keys.numel()
    if vals.numel() != n or vals.device != keys.device:
        raise DgsmError("keys and vals must have the same length and device")
    ka, va = torch.empty_like(keys), torch.empty_like(vals)
    temp = _alloc(lib().dgsm_sort_temp_bytes(n), keys.device)
    alt = C.c_int(0)
    rc = lib().dgsm_sort_pairs_u32(*[C.c_void_p(t.data_ptr()) for t in (keys, vals, ka, va)], n, int(nbits),
                                   C.c_void_p(temp.data_ptr()), temp.numel(), C.byref(alt),
                                   C.c_void_p(_stream_ptr(stream)))
    _check(rc, "dgsm_sort_pairs_u32")
    return (ka, va) if alt.value else (keys, vals)


def set_accumulate_events(before: Optional[torch.cuda.Event], after: Optional[torch.cuda.Event]):
    """Record these (already created) CUDA events around the accumulation kernel of
    subsequent builds on this thread; None, None disables."""
    b = C.c_void_p(before.cuda_event) if before is not None else None
    a = C.c_void_p(after.cuda_event) if after is not None else None
    lib().dgsm_set_accumulate_events(b, a)


def to_device(g: Dict[str, np.ndarray], device="cuda") -> Dict[str, torch.Tensor]:
    """numpy Gaussian dict -> CUDA float32 tensors."""
    return {k: torch.from_numpy(np.ascontiguousarray(v, np.float32)).to(device) for k, v in g.items()}
