"""CPU-side checks of the C ABI library (no GPU): it builds, loads, exports every symbol that
include/gf.h declares, host-only entry points work, and device entry points fail loudly
(GF_E_CUDA / GF_E_STATE) instead of falling back to the CPU."""
import ctypes
import os
import subprocess

import pytest

from paper_2602_05081_b200 import build as B
from paper_2602_05081_b200 import gf


@pytest.fixture(scope="module")
def L():
    B.build()
    return gf.lib()


def test_exports_every_header_symbol(L):
    syms = gf.header_symbols()
    assert "gf_trace_transmittance" in syms and "gf_render" in syms and len(syms) >= 15
    out = subprocess.run(["nm", "-D", "--defined-only", gf.LIB_PATH], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    for s in syms:
        assert hasattr(L, s)


def test_north_star_entry_points_present():
    for s in ("gf_load_primitives", "gf_build_bvh", "gf_set_lod_mask", "gf_trace_transmittance", "gf_render"):
        assert s in gf.header_symbols()


def test_sm100a_cubin_only():
    """the library carries sm_100a SASS (no PTX JIT / other-arch fallback)."""
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", gf.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_host_only_entry_points(L):
    assert L.gf_abi_version() == 8
    assert L.gf_status_string(0) == b"ok"
    # tile-interleaved ownership: 32x32 tiles, tile t -> t mod world
    assert gf.shard_pixel_owner(0, 0, 100, 100, 2) == 0
    assert gf.shard_pixel_owner(32, 0, 100, 100, 2) == 1
    assert gf.shard_pixel_owner(0, 32, 100, 100, 2) == 0  # 4 tiles per row -> tile 4
    assert gf.shard_pixel_owner(100, 0, 100, 100, 2) == -1
    assert gf.shard_sample_owner(5, 4) == 1
    pb, bb, sb = ctypes.c_size_t(), ctypes.c_size_t(), ctypes.c_size_t()
    assert L.gf_query_workspace(1000, ctypes.byref(pb), ctypes.byref(bb), None) == 0
    assert pb.value >= 64 * 1000 and bb.value >= 64 * 1000 + 32 * 2000
    assert L.gf_query_workspace(-1, ctypes.byref(pb), None, None) == 1


@pytest.mark.skipif(os.path.exists("/dev/nvidia0"), reason="checks the no-GPU failure mode")
def test_no_gpu_fails_loudly(L):
    c = ctypes.c_void_p()
    assert L.gf_create(0, ctypes.byref(c)) == 9  # GF_E_CUDA, no silent CPU path
    with pytest.raises(gf.GFError):
        gf.GaborField(0)
