"""The C-ABI library builds for sm_100a, loads, and exports every declared symbol (CPU)."""

import os
import re
import subprocess

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "splatfield_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\**\s+\**(sf_[a-z_0-9]+)\s*\(", text, re.M)))


@pytest.fixture(scope="module")
def lib_path():
    from paper_2507_07136_b200 import build_native
    return build_native.build()


def test_header_declares_the_path():
    names = declared_functions()
    for must in ("sf_render_frame", "sf_project", "sf_bin", "sf_decode", "sf_relevancy_f64",
                 "sf_mean_filter", "sf_select_segment", "sf_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol(lib_path):
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    missing = [n for n in declared_functions() if n not in exported]
    assert not missing, missing


def test_ctypes_binding_covers_header(lib_path):
    from paper_2507_07136_b200 import _native as N
    lib = N.load()
    for name in declared_functions():
        assert name in N.EXPORTS, name
        assert getattr(lib, name) is not None
    assert lib.sf_abi_version() == 4
    assert lib.sf_decode_fused(3, 64, 4, 512) == 1
    assert lib.sf_decode_fused(3, 32, 4, 512) == 0


def test_workspace_queries_need_no_gpu(lib_path):
    import ctypes
    from paper_2507_07136_b200 import _native as N
    lib = N.load()
    n = ctypes.c_size_t(0)
    assert lib.sf_frame_workspace_bytes(2_000_000, 1440, 1080, 3, 64, 4, 512, 12_000_000, ctypes.byref(n)) == 0
    assert n.value > 2_000_000 * 100


def test_cubin_is_sm100a_with_tensor_core_code(lib_path):
    out = subprocess.run(["cuobjdump", "--list-elf", lib_path], capture_output=True, text=True).stdout
    assert "sm_100a" in out
