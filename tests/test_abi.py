"""CPU-side checks of the C ABI boundary: the library builds for sm_100a, loads without a
GPU, exports every symbol include/difftrans.h declares, and its Python binding mirrors
the header's structs.  No compute calls (no GPU here)."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "difftrans.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2603_00413_b200 import _native, build
    build.build()
    return _native.lib()


def declared():
    src = open(HDR).read()
    return sorted(set(re.findall(r"^DT_API\s+[\w\s\*]+?\b(dt_\w+)\s*\(", src, flags=re.M)))


def test_header_declares_the_boundary():
    names = declared()
    for must in ("dt_create", "dt_destroy", "dt_last_error", "dt_build_bvh", "dt_trace_forward", "dt_trace_backward",
                 "dt_debug_closest_hit"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", os.path.join(ROOT, "paper_2603_00413_b200",
                                                                     "libdifftrans.so")],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\sT\s+(dt_\w+)", out))
    missing = [n for n in declared() if n not in exported]
    assert not missing, missing
    for n in declared():
        assert hasattr(lib, n)


def test_sm100a_cubin_present(lib):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf",
                          os.path.join(ROOT, "paper_2603_00413_b200", "libdifftrans.so")],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_host_only_calls(lib):
    assert lib.dt_status_string(0) == b"DT_OK"
    assert lib.dt_status_string(2) == b"DT_ERR_EMPTY_GEOMETRY"
    assert lib.dt_status_string(6) == b"DT_ERR_NO_FORWARD"
    # a NULL context is rejected without touching the device
    assert lib.dt_build_bvh(None, None, 0, None, 0, None) == 1
    assert lib.dt_trace_backward(None, None, None, None, None, 0, None) == 1
    assert lib.dt_last_error(None) == b"null context"


def test_binding_structs_match_header():
    """ctypes layouts agree with the C struct sizes computed by the host compiler."""
    from paper_2603_00413_b200 import _native as N
    prog = r'''
#include <stdio.h>
#include "difftrans.h"
int main(){printf("%zu %zu %zu %zu %zu %zu\n", sizeof(dt_absorption), sizeof(dt_env), sizeof(dt_cameras),
 sizeof(dt_trace_opts), sizeof(dt_stats), sizeof(dt_profile)); return 0;}'''
    tmp = "/tmp/dt_sizes"
    open(tmp + ".c", "w").write(prog)
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), tmp + ".c", "-o", tmp], check=True)
    sizes = list(map(int, subprocess.run([tmp], capture_output=True, text=True).stdout.split()))
    assert sizes == [C.sizeof(N.Absorption), C.sizeof(N.Env), C.sizeof(N.Cameras), C.sizeof(N.TraceOpts),
                     C.sizeof(N.Stats), C.sizeof(N.Profile)]


def test_product_path_does_not_touch_the_oracle():
    """The product package never imports, links or loads anything under oracle/."""
    pkg = os.path.join(ROOT, "paper_2603_00413_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src and "liboracle" not in src, f
                assert not re.search(r'#include\s+"[^"]*oracle', src), f
