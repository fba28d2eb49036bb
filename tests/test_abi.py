"""C-ABI checks that need no GPU: libdgsm.so loads, exports every function that
include/dgsm.h declares, the ctypes structs match the C layouts (checked with
gcc against the header), and argument validation fails loudly before any
device work."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2601_01660_b200 import build_ext, dgsm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "dgsm.h")


@pytest.fixture(scope="module")
def lib():
    build_ext.build()
    return dgsm.lib()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dgsm_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol(lib):
    decl = declared_functions()
    assert len(decl) >= 10
    out = subprocess.check_output(["nm", "-D", "--defined-only", dgsm.LIB_PATH], text=True)
    exported = set(re.findall(r" T (dgsm_\w+)", out))
    assert set(decl) <= exported, set(decl) - exported
    assert set(decl) == set(dgsm.EXPORTED)
    for f in decl:
        assert hasattr(lib, f)


def test_struct_layouts_match_header(tmp_path):
    prog = tmp_path / "layout.c"
    prog.write_text(f"""
#include <stdio.h>
#include <stddef.h>
#include "{HEADER}"
int main(void) {{
  printf("%zu %zu %zu %zu\\n", sizeof(dgsm_gaussians_t), sizeof(dgsm_light_t), sizeof(dgsm_build_opts_t), sizeof(dgsm_plan_t));
  printf("%zu %zu %zu %zu\\n", offsetof(dgsm_plan_t, n_keys), offsetof(dgsm_plan_t, depth_bits),
         offsetof(dgsm_plan_t, run_workspace_bytes), offsetof(dgsm_plan_t, signature));
  return 0;
}}""")
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-o", str(exe), str(prog)])
    lines = subprocess.check_output([str(exe)], text=True).split("\n")
    sizes = [int(x) for x in lines[0].split()]
    offs = [int(x) for x in lines[1].split()]
    assert sizes == [C.sizeof(dgsm.Gaussians), C.sizeof(dgsm.Light), C.sizeof(dgsm.BuildOpts), C.sizeof(dgsm.Plan)]
    assert offs == [dgsm.Plan.n_keys.offset, dgsm.Plan.depth_bits.offset,
                    dgsm.Plan.run_workspace_bytes.offset, dgsm.Plan.signature.offset]


def test_defaults_and_sizes(lib):
    o = dgsm.BuildOpts()
    lib.dgsm_default_opts(C.byref(o))
    assert (o.kappa, o.k_sigma, o.rho_scale, o.bin_mode, o.flags) == (1.0, 3.0, 1.0, 0, 0)
    a = lib.dgsm_plan_workspace_bytes(1000, 1)
    b = lib.dgsm_plan_workspace_bytes(2000, 1)
    assert a > 96 * 1000 and b > a and b - a >= 96 * 1000
    assert lib.dgsm_plan_workspace_bytes(-1, 1) == 0
    assert lib.dgsm_strerror(0) == b"success"
    assert lib.dgsm_strerror(2) == b"workspace too small"


def test_validation_fails_before_device_work(lib):
    g = dgsm.Gaussians(None, None, None, None, 0)
    lights = (dgsm.Light * 1)()
    lights[0].t_max = 1.0
    plan = dgsm.Plan()
    ws = C.c_void_p(256)  # never dereferenced: validation fails first
    # bad atlas_res
    assert lib.dgsm_build_plan(C.byref(g), lights, 1, 12, 8, None, ws, 1 << 20, C.byref(plan), None) == 1
    assert b"atlas_res" in lib.dgsm_last_error()
    # bad shells, lights, t_max
    assert lib.dgsm_build_plan(C.byref(g), lights, 1, 16, 0, None, ws, 1 << 20, C.byref(plan), None) == 1
    assert lib.dgsm_build_plan(C.byref(g), lights, 0, 16, 4, None, ws, 1 << 20, C.byref(plan), None) == 1
    lights[0].t_max = 0.0
    assert lib.dgsm_build_plan(C.byref(g), lights, 1, 16, 4, None, ws, 1 << 20, C.byref(plan), None) == 1
    lights[0].t_max = 1.0
    # workspace too small
    assert lib.dgsm_build_plan(C.byref(g), lights, 1, 16, 4, None, ws, 16, C.byref(plan), None) == 2
    # negative n; null arrays with n > 0
    g.n = -1
    assert lib.dgsm_build_plan(C.byref(g), lights, 1, 16, 4, None, ws, 1 << 20, C.byref(plan), None) == 1
    g.n = 5
    assert lib.dgsm_build_plan(C.byref(g), lights, 1, 16, 4, None, ws, 1 << 20, C.byref(plan), None) == 1
    # bad options
    o = dgsm.BuildOpts(1.0, 3.0, -1.0, 0, 0)
    g.n = 0
    assert lib.dgsm_build_plan(C.byref(g), lights, 1, 16, 4, C.byref(o), ws, 1 << 20, C.byref(plan), None) == 1
    # query validation
    assert lib.dgsm_query(None, lights, 1, 16, 4, None, 10, None, None, None) == 1
    assert lib.dgsm_exp_epilogue(None, None, -1, None) == 1
    # footprint query validation (NEXT-2): sample count and null host arrays
    z = (C.c_float * (3 * 65))()
    w = (C.c_float * 65)()
    for n in (0, 65):
        assert lib.dgsm_query_footprint(None, lights, 1, 16, 4, None, None, None, 0, z, w, n, None, None, None) == 1
    assert lib.dgsm_query_footprint(None, lights, 1, 16, 4, None, None, None, 0, None, w, 1, None, None, None) == 1
    # ROI slab (NEXT-1): sizes and validation
    assert lib.dgsm_slab_bytes(1, 16) == 256 + 8 and lib.dgsm_slab_bytes(2, 2048) == 8 * 2 * 256 * 256 + 16
    assert lib.dgsm_slab_bytes(0, 16) == 0 and lib.dgsm_slab_bytes(1, 12) == 0
    roi = dgsm.Roi((C.c_float * 3)(0, 0, 0), 2.0, 0.0, 1.0)
    buf = C.c_void_p(256)
    assert lib.dgsm_active_slab(None, 0, C.byref(roi), lights, 1, 16, 4, buf, 16, None) == 2
    assert lib.dgsm_active_slab(None, 0, C.byref(roi), lights, 1, 16, 4, None, 1 << 20, None) == 1
    assert lib.dgsm_active_slab(None, 5, C.byref(roi), lights, 1, 16, 4, buf, 1 << 20, None) == 1
    roi.radius = 0.0
    assert lib.dgsm_active_slab(None, 0, C.byref(roi), lights, 1, 16, 4, buf, 1 << 20, None) == 1
    roi.radius, roi.z_min = 2.0, 2.0
    assert lib.dgsm_active_slab(None, 0, C.byref(roi), lights, 1, 16, 4, buf, 1 << 20, None) == 1
    o = dgsm.BuildOpts(1.0, 3.0, 1.0, 0, 0, 0, C.c_void_p(12))  # misaligned slab
    assert lib.dgsm_build_plan(C.byref(g), lights, 1, 16, 4, C.byref(o), ws, 1 << 20, C.byref(plan), None) == 1


def test_binding_refuses_cpu_tensors():
    import torch
    g = {k: torch.zeros(4, d) for k, d in (("means", 3), ("scales", 3), ("rotations", 4))}
    g["opacities"] = torch.zeros(4)
    with pytest.raises(dgsm.DgsmError):
        dgsm.build(g, dict(position=[[0, 0, 0]], t_max=[1.0]), 16, 4)


def test_transfer_validation(lib):
    """NEXT-4 ABI: defaults, workspace size, argument checks before device work."""
    o = dgsm.TransferOpts()
    lib.dgsm_default_transfer_opts(C.byref(o))
    assert (o.grid_theta, o.grid_phi, o.q, o.s_max, o.gamma) == (64, 128, 1.0, 4.0, 1.0)
    assert lib.dgsm_transfer_workspace_bytes(C.byref(o), 1000) >= 2 * 16 * 64 * 128 + 16 * 1000
    assert lib.dgsm_transfer_workspace_bytes(C.byref(o), -1) == 0
    sh = (C.c_float * 48)()
    ws = C.c_void_p(256)
    assert lib.dgsm_sh_transfer(sh, 4, None, None, 0, C.byref(o), None, None, ws, 1 << 30, None) == 1
    assert lib.dgsm_sh_transfer(None, 3, None, None, 0, C.byref(o), None, None, ws, 1 << 30, None) == 1
    assert lib.dgsm_sh_transfer(sh, 3, None, None, 5, C.byref(o), None, None, ws, 1 << 30, None) == 1
    assert lib.dgsm_sh_transfer(sh, 3, None, None, 0, C.byref(o), None, None, ws, 16, None) == 2
    o.s_max = 0.0
    assert lib.dgsm_sh_transfer(sh, 3, None, None, 0, C.byref(o), None, None, ws, 1 << 30, None) == 1


def test_footprint_stencil_host_entry(lib, oracle_mod):
    """dgsm_footprint_stencil (host arithmetic, no device) against the oracle's
    7-point stencil and SPEC's centre weight 0.2156; bad arguments fail."""
    z, w = dgsm.footprint_stencil("stencil7", 1.0)
    zo, wo = oracle_mod.stencil7(1.0)
    assert np.allclose(z, zo) and np.allclose(w, wo, atol=1e-7)
    assert abs(w[0] - 0.2156) < 5e-5 and abs(w.sum() - 1.0) < 1e-6
    z, w = dgsm.footprint_stencil("center")
    assert z.shape == (1, 3) and w.tolist() == [1.0]
    with pytest.raises(dgsm.DgsmError):
        dgsm.footprint_stencil("stencil7", -1.0)
