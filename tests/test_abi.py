"""C-ABI library: builds, loads without a GPU, exports every symbol include/gsb.h declares,
and validates arguments on the host (no compute calls)."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2604_25459_b200 as gsb
from paper_2604_25459_b200 import build as gsb_build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "gsb.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gsb_[a-z_]+)\s*\(", src)))


def test_library_builds_and_exports_header_symbols():
    gsb_build.build()
    L = gsb.lib()
    declared = header_functions()
    assert len(declared) >= 11
    assert sorted(declared) == sorted(gsb.EXPORTS)
    for name in declared:
        assert hasattr(L, name), name
    assert gsb.version().startswith("gsb")


def test_binding_declares_every_prototype():
    """Every exported function has ctypes argtypes matching the header's parameter count (an
    undeclared function would pass 64-bit pointers as C int)."""
    src = re.sub(r"/\*.*?\*/", "", open(os.path.join(ROOT, "include", "gsb.h")).read(), flags=re.S)
    L = gsb.lib()
    protos = dict(re.findall(r"\b(gsb_[a-z_]+)\s*\(([^;{]*?)\)\s*;", src))
    assert sorted(protos) == sorted(gsb.EXPORTS)
    for name, params in protos.items():
        params = params.strip()
        n = 0 if params in ("", "void") else params.count(",") + 1
        assert getattr(L, name).argtypes is not None, name
        assert len(getattr(L, name).argtypes) == n, (name, n)


def test_sm100a_only_cubin():
    """The library carries sm_100a SASS (no other arch, no PTX JIT fallback)."""
    import subprocess
    gsb_build.build()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", gsb.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(8\d|9\d)", out)


def test_host_side_validation_without_gpu():
    L = gsb.lib()
    n = 4
    m = np.zeros((n, 3), np.float32)
    s = np.ones((n, 3), np.float32)
    q = np.tile(np.float32([1, 0, 0, 0]), (n, 1))
    o = np.full(n, 0.5, np.float32)
    sh = np.zeros((n, 1, 3), np.float32)
    b = np.full(n, -1, np.int32)
    h = ctypes.c_void_p()
    p = lambda a: a.ctypes.data
    # NULL out
    assert L.gsb_create_scene(p(m), p(s), p(q), p(o), p(sh), 0, p(b), n, 0, 0, None) == 1
    # bad SH degree
    assert L.gsb_create_scene(p(m), p(s), p(q), p(o), p(sh), 5, p(b), n, 0, 0, ctypes.byref(h)) == 1
    # non-finite value
    m2 = m.copy()
    m2[0, 0] = np.nan
    assert L.gsb_create_scene(p(m2), p(s), p(q), p(o), p(sh), 0, p(b), n, 0, 0, ctypes.byref(h)) == 1
    assert b"non-finite" in L.gsb_last_error()
    # valid arguments, but no sm_100 device in this container
    import torch
    if not torch.cuda.is_available():
        assert L.gsb_create_scene(p(m), p(s), p(q), p(o), p(sh), 0, p(b), n, 0, 0, ctypes.byref(h)) == 7
    # NULL scene everywhere
    assert L.gsb_reserve(None, 1, 1, 64, 48, 0, 0, 0) == 1
    prm = gsb.RenderParams(64, 48).to_c()
    assert L.gsb_render(None, None, 1, 1, None, None, ctypes.byref(prm), None, None, None, None, None) == 1
    assert L.gsb_destroy_scene(None) == 0
    assert L.gsb_debug_bin_sort(None, None, None, None, None, None, None, 0, 0, 8, 8, None, None, 0, None, None) == 1
    # LiDAR entry points validate before touching the device
    d = np.float32([[1, 0, 0]])
    assert L.gsb_lidar_create(None, d.ctypes.data, 1, 0, 0, ctypes.byref(ctypes.c_void_p())) == 1
    assert L.gsb_render_lidar(None, None, None, 1, 1, None, 0, None, 0.01, 100.0, None, None, None) == 1
    assert L.gsb_lidar_info(None, None, None, None, None) == 1
    assert L.gsb_lidar_destroy(None) == 0
    # the standalone encoder rejects missing parameters before any device work
    assert L.gsb_obs_encode(None, None, 1, 1, 8, 8, None, None, None, None, None) == 1
    o = gsb.gsb_obs_params()
    assert L.gsb_obs_encode(None, None, 1, 1, 8, 8, ctypes.byref(o), None, None, None, None) == 1
    assert L.gsb_obs_encode(None, None, 1, 0, 8, 8, ctypes.byref(o), None, 1, None, None) == 1


def test_render_params_layout_matches_header(tmp_path):
    """ctypes structs == the C compiler's layout of include/gsb.h (sizes and every offset)."""
    import subprocess
    structs = {"gsb_render_params": gsb.gsb_render_params, "gsb_timings": gsb.gsb_timings,
               "gsb_obs_params": gsb.gsb_obs_params, "gsb_stats": gsb.gsb_stats}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "gsb.h"', "int main(void) {"]
    for name, cls in structs.items():
        lines.append(f'printf("{name} %zu\\n", sizeof({name}));')
        for fname, _ in cls._fields_:
            lines.append(f'printf("{name}.{fname} %zu\\n", offsetof({name}, {fname}));')
    lines.append("return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), "-o", str(exe), str(src)])
    got = dict(l.split() for l in subprocess.check_output([str(exe)]).decode().splitlines())
    for name, cls in structs.items():
        assert int(got[name]) == ctypes.sizeof(cls), name
        for fname, _ in cls._fields_:
            assert int(got[f"{name}.{fname}"]) == getattr(cls, fname).offset, (name, fname)


def test_prune_mask_policy():
    """Host-side pruning policy: top ceil(f N) by score, ties broken by lower creation index."""
    w = np.array([0.5, 0.1, 0.5, 0.0, 0.9, 0.1])
    np.testing.assert_array_equal(gsb.prune_mask(w, 0.5), [True, False, True, False, True, False])
    np.testing.assert_array_equal(gsb.prune_mask(w, 0.6), [True, True, True, False, True, False])
    assert gsb.prune_mask(w, 0.0).sum() == 0 and gsb.prune_mask(w, 1.0).all()
