"""CPU-only checks of the drop-in boundary: the C-ABI library loads (no GPU needed) and exports
every symbol include/pbsa_b200.h declares; the Python binding covers exactly that set; the host
API validates arguments before touching the device."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pbsa_b200.h")
DEBUG_HEADER = os.path.join(ROOT, "include", "pbsa_b200_debug.h")
LIB = os.path.join(ROOT, "paper_2604_21221_b200", "_lib", "libpbsa_b200.so")


def declared(header=HEADER):
    text = open(header).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pbsa_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_hot_path():
    names = declared()
    for must in ["pbsa_compress", "pbsa_score_select", "pbsa_bsa_fwd", "pbsa_mem_create",
                 "pbsa_mem_commit", "pbsa_mem_write_chunk", "pbsa_attend", "pbsa_last_error"]:
        assert must in names


@pytest.mark.skipif(not os.path.exists(LIB), reason="library not built")
def test_library_exports_every_declared_symbol():
    lib = C.CDLL(LIB)
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


@pytest.mark.skipif(not os.path.exists(LIB), reason="library not built")
def test_python_binding_matches_header():
    from paper_2604_21221_b200 import _capi
    assert sorted(_capi.EXPORTED) == declared()
    # the test hooks live in their own header, outside the drop-in boundary
    assert sorted(_capi.DEBUG_EXPORTED) == declared(DEBUG_HEADER)
    assert not set(declared(DEBUG_HEADER)) & set(declared())
    lib = C.CDLL(LIB)
    assert all(hasattr(lib, n) for n in declared(DEBUG_HEADER))


@pytest.mark.skipif(not os.path.exists(LIB), reason="library not built")
def test_fault_injection_names():
    from paper_2604_21221_b200 import _capi
    assert _capi.LIB.pbsa_debug_set_fault(b"no-such-fault") == _capi.PBSA_EINVAL
    assert b"unknown fault" in _capi.LIB.pbsa_last_error()
    assert _capi.LIB.pbsa_debug_set_fault(b"drop-sink") == _capi.PBSA_OK
    assert _capi.LIB.pbsa_debug_set_fault(None) == _capi.PBSA_OK


@pytest.mark.skipif(not os.path.exists(LIB), reason="library not built")
def test_argument_errors_need_no_gpu():
    from paper_2604_21221_b200 import _capi
    lib = _capi.LIB
    h = C.c_void_p()
    assert lib.pbsa_mem_create(C.byref(h), 1, 4, 1, 8, 60, 128) == _capi.PBSA_EINVAL
    assert b"sink chunk" in lib.pbsa_last_error()
    assert lib.pbsa_mem_create(C.byref(h), 1, 8, 1, 8, 60, 96) == _capi.PBSA_EUNSUPPORTED
    rc = lib.pbsa_bsa_fwd(None, None, None, 4, None, 0, 0, None, 0, 0, None, 0, 1, 65, 128, 1,
                          0.0, None, None, None, 0, None)
    assert rc == _capi.PBSA_EINVAL and b"block size" in lib.pbsa_last_error()
    rc = lib.pbsa_score_select(None, None, 0, None, 4, 4, 0, 4, 5, 1, 1, 128, 0.0, None, None,
                               None, 0, None)
    assert rc == _capi.PBSA_EINVAL and b"k exceeds" in lib.pbsa_last_error()
    rc = lib.pbsa_attend_qkv_host(None, None, None, None, 4, 0.0, 0, None, None)
    assert rc == _capi.PBSA_EINVAL and b"attend_qkv_host" in lib.pbsa_last_error()
    assert lib.pbsa_mem_host_sync(None) == _capi.PBSA_EINVAL
    rc = lib.pbsa_pair_tiles(None, 4, 2, 4, 3, 10, 1, None, None)  # rows 2..5 of a 4-row sel
    assert rc == _capi.PBSA_EINVAL and b"pair_tiles" in lib.pbsa_last_error()
    rc = lib.pbsa_pair_tiles(None, 4, 0, 4, 3, 10, 1, None, None)
    assert rc == _capi.PBSA_EINVAL and b"null pointer" in lib.pbsa_last_error()
    assert lib.pbsa_last_tile_pairs(None, None, None) == _capi.PBSA_EINVAL
    assert lib.pbsa_launch_count() >= 0


def test_product_package_does_not_import_the_oracle():
    pkg = os.path.join(ROOT, "paper_2604_21221_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                text = open(os.path.join(dirpath, f)).read()
                for pat in (r"^\s*(from|import)\s+oracle", r"liboracle", r"\borc_[a-z]", r"_ref/"):
                    assert not re.search(pat, text, flags=re.M), (f, pat)


@pytest.mark.skipif(not os.path.exists(LIB), reason="library not built")
def test_latent_geometry_follows_make_block_layout():
    """Chunk-latent blocking (pbsa_latent_blocks) = blockify.cpp:7-36's layout rules, host only."""
    from paper_2604_21221_b200 import PbsaError, latent_blocks
    # Wan2.1-1.3B chunk: 3 latent frames of 30 x 52, 12 heads x 128, (1, 15, 4) blocks
    assert latent_blocks((3, 30, 52, 12 * 128), 12, 128, (1, 15, 4)) == (78, 60)
    assert latent_blocks((2, 3, 30, 52, 12 * 128), 12, 128, (1, 15, 4)) == (78, 60)
    assert latent_blocks((2, 16, 16, 64), 1, 64, (1, 8, 8)) == (8, 64)   # config 1 (2-frame chunk)
    for shape, blk, axis in [((3, 30, 52, 1536), (2, 15, 4), b"T"), ((3, 30, 52, 1536), (1, 7, 4), b"H"),
                             ((3, 30, 52, 1536), (1, 15, 5), b"W")]:
        with pytest.raises(PbsaError, match="not divisible"):
            latent_blocks(shape, 12, 128, blk)
        from paper_2604_21221_b200 import _capi
        assert axis + b" (" in _capi.LIB.pbsa_last_error()
    with pytest.raises(PbsaError, match="at most 64"):
        latent_blocks((3, 30, 52, 1536), 12, 128, (3, 15, 4))     # 180 tokens > one 64-row slot
    with pytest.raises(PbsaError, match="heads"):
        latent_blocks((3, 30, 52, 1000), 12, 128, (1, 15, 4))
