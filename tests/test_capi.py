"""The C-ABI library builds for sm_100a, loads without a GPU, and exports exactly the
entry points include/mlra_b200.h declares (with matching arity). Argument validation
paths that fail before any CUDA call are exercised here too."""

import ctypes
import os
import re
import subprocess

import pytest

from paper_2603_02188_b200 import _lib, build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mlra_b200.h")


def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    funcs = {}
    for m in re.finditer(r"^\s*(?:int|size_t|const char\*)\s+(mlra_\w+)\s*\(([^;]*?)\)\s*;", text, flags=re.M | re.S):
        args = m.group(2).strip()
        funcs[m.group(1)] = 0 if args in ("", "void") else len([a for a in args.split(",") if a.strip()])
    return funcs


@pytest.fixture(scope="module")
def lib():
    build.build()
    return _lib.load()


def test_header_declares_the_abi():
    funcs = header_functions()
    assert set(funcs) == set(_lib.SIGNATURES), sorted(set(funcs) ^ set(_lib.SIGNATURES))


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    for name, nargs in header_functions().items():
        assert name in exported, name
        assert len(_lib.SIGNATURES[name][1]) == nargs, (name, nargs)


def test_library_is_sm100a(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass and "UTMALDG" in sass  # tcgen05.mma and TMA in the decode kernel


def test_cpu_safe_calls(lib):
    assert lib.mlra_version() == 200
    assert lib.mlra_workspace_bytes(16, 24, 4, 128, 64, 9) > 16 * 9 * 4 * 24 * 128 * 4
    # argument validation happens before any CUDA call
    rc = lib.mlra_decode_partials(None, None, None, None, None, None, None, 1, 24, 3, 1, 128, 64, 128, 1, 1, 1, None)
    assert rc == -2 and b"NB=3" in lib.mlra_last_error()
    rc = lib.mlra_decode_partials(None, None, None, None, None, None, None, 1, 24, 1, 1, 96, 64, 128, 1, 1, 1, None)
    assert rc == -2 and b"sub-block width" in lib.mlra_last_error()
    rc = lib.mlra_decode_partials(None, None, None, None, None, None, None, 1, 24, 1, 1, 128, 64, 100, 1, 1, 1, None)
    assert rc == -2 and b"page_size" in lib.mlra_last_error()
    rc = lib.mlra_cache_append(None, None, None, 1, 7, 64, 1, 1, None, None)
    assert rc == -1 and b"row width" in lib.mlra_last_error()
    rc = lib.mlra_combine(None, None, None, None, None, 1, 1, 1, 128, 128, 1, 1.0, 3, None, None)
    assert rc == -2
    rc = lib.mlra_check_status(None, 1, None)
    assert rc == -2 and b"null status" in lib.mlra_last_error()
    with pytest.raises(_lib.ConfigError):
        _lib.check(-2, "probe")


def test_cpu_safe_calls_gqa_and_fused_append(lib):
    # GQA entry points: validation before any CUDA call
    assert lib.mlra_gqa_workspace_bytes(16, 6, 4, 128, 3) >= 16 * 3 * 6 * 4 * 128 * 4
    assert 1 <= lib.mlra_gqa_default_splits(16, 6, 32768) <= 160
    rc = lib.mlra_gqa_decode_partials(None, None, None, None, None, None, 1, 6, 4, 96, 128, 1, 1, 1, 1.0, None)
    assert rc == -2 and b"head width" in lib.mlra_last_error()
    rc = lib.mlra_gqa_decode_partials(None, None, None, None, None, None, 1, 6, 32, 128, 128, 1, 1, 1, 1.0, None)
    assert rc == -2 and b"query heads per KV head" in lib.mlra_last_error()
    rc = lib.mlra_gqa_decode_step(None, None, None, None, None, None, 1, 6, 4, 128, 100, 1, 1, 1, 1.0, None)
    assert rc == -2 and b"page_size" in lib.mlra_last_error()
    # fused K0: shape / config validation
    rc = lib.mlra_cache_append_latent(None, None, None, None, None, 1, 510, 4, 0, 4, 128, 64, 64, 1.0, 1e4, 1e-6,
                                      128, 1, 1, 1, None, None)
    assert rc == -1 and b"branches" in lib.mlra_last_error()
    rc = lib.mlra_cache_append_latent(None, None, None, None, None, 1, 512, 4, 3, 2, 128, 64, 64, 1.0, 1e4, 1e-6,
                                      128, 1, 1, 1, None, None)
    assert rc == -2 and b"blocks" in lib.mlra_last_error()
    rc = lib.mlra_cache_append_latent(None, None, None, None, None, 1, 512, 4, 0, 1, 128, 63, 64, 1.0, 1e4, 1e-6,
                                      128, 1, 1, 1, None, None)
    assert rc == -2 and b"even" in lib.mlra_last_error()
    rc = lib.mlra_cache_append_latent(None, None, None, None, None, 1, 512, 4, 0, 1, 128, 64, 64, 1.0, 1e4, 1e-6,
                                      128, 1, 3, 1, None, None)
    assert rc == -2 and b"RMS groups" in lib.mlra_last_error()
    # splits beyond the merge kernels' limit
    rc = lib.mlra_decode_partials(None, None, None, None, None, None, None, 1, 24, 1, 1, 128, 64, 128, 1, 1, 161, None)
    assert rc == -2 and b"nsplit" in lib.mlra_last_error()
