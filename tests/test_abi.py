"""Host-side checks of the C ABI (no GPU needed): the library builds for sm_100a,
loads, exports every symbol include/pgsag.h declares, and its argument
validation rejects bad calls before touching a device."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pgsag.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2501_01677_b200 import build
    build.build()
    from paper_2501_01677_b200 import _lib
    return _lib


def declared_functions():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(pgsag_\w+)\s*\(", src, re.M)))


def test_header_declares_the_four_calls():
    fns = declared_functions()
    for f in ("pgsag_preprocess", "pgsag_bin_sort", "pgsag_render_fwd", "pgsag_render_bwd",
              "pgsag_workspace_size", "pgsag_last_error"):
        assert f in fns


def test_library_exports_every_declared_symbol(lib):
    L = lib.lib()
    for f in declared_functions():
        assert hasattr(L, f), f
    assert set(declared_functions()) == set(lib.SYMBOLS)
    out = subprocess.run(["nm", "-D", "--defined-only", lib.LIB_PATH], capture_output=True, text=True).stdout
    for f in declared_functions():
        assert re.search(rf"\bT {f}\b", out), f


def test_library_is_sm100a(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out, out


def test_header_compiles_as_c(tmp_path):
    src = tmp_path / "t.c"
    src.write_text('#include "pgsag.h"\nint main(void){ pgsag_camera c; (void)c; return PGSAG_OK; }\n')
    subprocess.check_call(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.dirname(HEADER), "-c", str(src),
                           "-o", str(tmp_path / "t.o")])


def test_struct_layouts_match_header(lib, tmp_path):
    """The ctypes mirror has the C sizes/offsets (checked against the compiled header)."""
    prog = tmp_path / "s.c"
    prog.write_text(r'''#include <stdio.h>
#include <stddef.h>
#include "pgsag.h"
int main(void){
 printf("%zu %zu %zu %zu %zu %zu %zu %zu %zu %zu %zu %zu %zu %zu %zu\n", sizeof(pgsag_camera), sizeof(pgsag_gaussians),
   sizeof(pgsag_projected), sizeof(pgsag_tilemask), sizeof(pgsag_bins), sizeof(pgsag_image),
   sizeof(pgsag_image_grad), sizeof(pgsag_gaussian_grad), offsetof(pgsag_camera, znear), offsetof(pgsag_bins, n_dup),
   sizeof(pgsag_adam_state), sizeof(pgsag_adam_hparams), offsetof(pgsag_adam_hparams, step),
   sizeof(pgsag_densify_params), offsetof(pgsag_densify_params, seed));
 return 0; }''')
    exe = tmp_path / "s"
    subprocess.check_call(["gcc", "-I", os.path.dirname(HEADER), str(prog), "-o", str(exe)])
    got = [int(v) for v in subprocess.check_output([str(exe)]).split()]
    exp = [C.sizeof(lib.Camera), C.sizeof(lib.Gaussians), C.sizeof(lib.Projected), C.sizeof(lib.TileMask),
           C.sizeof(lib.Bins), C.sizeof(lib.Image), C.sizeof(lib.ImageGrad), C.sizeof(lib.GaussianGrad),
           lib.Camera.znear.offset, lib.Bins.n_dup.offset, C.sizeof(lib.AdamState), C.sizeof(lib.AdamHparams),
           lib.AdamHparams.step.offset, C.sizeof(lib.DensifyParams), lib.DensifyParams.seed.offset]
    assert got == exp


def test_workspace_size_monotone(lib):
    a = lib.workspace_size(1000, 64, 64, 10000)
    b = lib.workspace_size(2000, 64, 64, 10000)
    c = lib.workspace_size(2000, 64, 64, 20000)
    assert 0 < a < b < c
    assert a % 256 == 0


def test_invalid_arguments_rejected_on_host(lib):
    L = lib.lib()
    cam = lib.Camera()
    cam.width, cam.height, cam.fx, cam.fy = 64, 64, 64.0, 64.0
    rc = L.pgsag_preprocess(None, C.byref(cam), None, None, None, None, 0, None)
    assert rc == lib.PGSAG_EINVAL and b"NULL" in L.pgsag_last_error()
    g = lib.Gaussians()
    g.n, g.sh_degree = 10, 4
    rc = L.pgsag_preprocess(C.byref(g), C.byref(cam), None, None, None, None, 0, None)
    assert rc == lib.PGSAG_EINVAL and b"sh_degree" in L.pgsag_last_error()
    g.sh_degree, g.n = 3, 0
    bad = lib.Camera()
    rc = L.pgsag_preprocess(C.byref(g), C.byref(bad), None, None, None, None, 0, None)
    assert rc == lib.PGSAG_EINVAL and b"width" in L.pgsag_last_error()
    # entry buffers off a 16-byte boundary are rejected before any launch (the sort's 128-bit loads);
    # the pointers are never dereferenced
    tm, b = lib.TileMask(), lib.Bins()
    tm.tile_cnt = tm.active = tm.n_active = tm.active_bits = 0x1000
    b.tile_keys, b.vals, b.ranges, b.capacity = 0x2004, 0x3000, 0x4000, 16
    rc = L.pgsag_bin_sort(C.byref(lib.Projected()), C.byref(tm), C.byref(cam), 0, C.byref(b), None, 0, None)
    assert rc == lib.PGSAG_EINVAL and b"16-byte aligned" in L.pgsag_last_error()
    assert lib.version().startswith("pgsag-b200")


def test_next_row_calls_validate_on_host(lib):
    """The NEXT-row entry points reject bad calls before any device work."""
    L = lib.lib()
    err = lambda: L.pgsag_last_error()
    # pgsag_rgb_loss: NULL buffers, bad size, small workspace
    assert L.pgsag_rgb_loss(None, None, None, 8, 8, 1.0, None, None, None, 0, None) == lib.PGSAG_EINVAL
    assert b"NULL" in err()
    dummy = C.c_void_p(256)  # never dereferenced: validation fails first
    assert L.pgsag_rgb_loss(dummy, dummy, dummy, 0, 8, 1.0, dummy, None, dummy, 1 << 20, None) == lib.PGSAG_EINVAL
    assert L.pgsag_rgb_loss(dummy, dummy, dummy, 8, 8, 1.0, dummy, None, dummy, 16, None) == lib.PGSAG_EWORKSPACE
    assert lib.rgb_loss_workspace_size(8, 8) == 36 * 64 and lib.rgb_loss_workspace_size(0, 8) == 0
    # pgsag_adam_step: step must be >= 1, NULL state
    gr, st, hp = lib.GaussianGrad(), lib.AdamState(), lib.AdamHparams()
    hp.step = 0
    assert L.pgsag_adam_step(10, 3, C.byref(gr), C.byref(st), C.byref(hp), None, None) == lib.PGSAG_EINVAL
    assert b"step" in err()
    hp.step = 1
    assert L.pgsag_adam_step(10, 3, C.byref(gr), C.byref(st), C.byref(hp), None, None) == lib.PGSAG_EINVAL
    assert L.pgsag_adam_step(10, 4, C.byref(gr), C.byref(st), C.byref(hp), None, None) == lib.PGSAG_EINVAL
    # densification: counts inconsistent with n; missing workspace
    dp = lib.DensifyParams(2e-4, 0.01, 0.005, 1)
    counts = (C.c_int64 * 3)(5, 6, 0)  # more clones than kept
    assert L.pgsag_densify_apply(5, 3, C.byref(st), None, C.byref(dp), C.byref(counts), C.byref(st), None, 0,
                                 None) == lib.PGSAG_EINVAL
    assert b"counts" in err()
    out = (C.c_int64 * 3)()
    assert L.pgsag_densify_plan(-1, None, None, None, None, C.byref(dp), None, C.byref(out), None, 0,
                                None) == lib.PGSAG_EINVAL
    assert lib.densify_workspace_size(0) > 0 and lib.densify_workspace_size(5000) > lib.densify_workspace_size(10)
    # opacity reset: cap must lie in (0, 1)
    assert L.pgsag_opacity_reset(10, C.byref(st), 1.5, None) == lib.PGSAG_EINVAL
    # band / ban / gc weights: NULL or bad radius
    assert L.pgsag_boundary_band(dummy, 8, 8, 0, dummy, None) == lib.PGSAG_EINVAL
    assert L.pgsag_gc_weights(None, None, 8, 8, None, None, 0, None) == lib.PGSAG_EINVAL
    cam = lib.Camera()
    cam.width, cam.height, cam.fx, cam.fy = 8, 8, 8.0, 8.0
    assert L.pgsag_ban_loss(C.byref(cam), None, None, None, None, 0.1, 1.0, 1, None, None, None,
                            None) == lib.PGSAG_EINVAL
    # measurement aid: bad mode
    t = C.c_double()
    assert L.pgsag_microbench_fp32(7, 10, dummy, C.byref(t), None) == lib.PGSAG_EINVAL


def test_render_bwd_adam_validates_on_host(lib):
    """pgsag_render_bwd_adam: NULL optimiser arguments, step 0 and a state that does not hold the
    Gaussians' own arrays are rejected before any device work."""
    L = lib.lib()
    d = C.c_void_p(256)  # never dereferenced: validation fails first
    g = lib.Gaussians(10, 3, d, d, d, d, d)
    cam = lib.Camera()
    cam.width, cam.height, cam.fx, cam.fy = 64, 64, 64.0, 64.0
    p = lib.Projected(*([d] * 8))
    tm = lib.TileMask(d, None, d, d, d)
    bins = lib.Bins(d, d, d, 1 << 20, 0, None)
    fwd = lib.Image(*([d] * 8), None, None, None)
    ig, out, st, hp = lib.ImageGrad(), lib.GaussianGrad(), lib.AdamState(*([d] * 9)), lib.AdamHparams()
    bg = (C.c_float * 3)()
    args = lambda st_, hp_: (C.byref(g), C.byref(cam), C.byref(p), C.byref(bins), C.byref(tm), d, C.byref(bg),
                             C.byref(fwd), C.byref(ig), C.byref(out), st_, hp_, None, d, 1 << 40, None)
    hp.step = 1
    assert L.pgsag_render_bwd_adam(*args(None, C.byref(hp))) == lib.PGSAG_EINVAL
    hp.step = 0
    assert L.pgsag_render_bwd_adam(*args(C.byref(st), C.byref(hp))) == lib.PGSAG_EINVAL
    assert b"step" in L.pgsag_last_error()
    hp.step = 1
    st.mean = C.c_void_p(512)  # not g's array
    assert L.pgsag_render_bwd_adam(*args(C.byref(st), C.byref(hp))) == lib.PGSAG_EINVAL
    assert b"state" in L.pgsag_last_error()
