"""CPU checks of the boundary: libdf.so loads and exports every symbol include/df.h
declares; the binding wraps all of them; the product package never imports the oracle."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "df.h")
LIB = os.path.join(ROOT, "paper_2605_25550_b200", "libdf.so")


def _declared():
    txt = open(HDR).read()
    return sorted(set(re.findall(r"^\s*(?:df_status|const char\*|uint64_t|int32_t)\s+(df_\w+)\s*\(", txt, re.M)))


@pytest.fixture(scope="module")
def lib_path():
    if not os.path.exists(LIB):
        from paper_2605_25550_b200 import build
        build.build()
    return LIB


def test_header_declares_the_north_star_calls():
    names = _declared()
    for n in ("df_init", "df_submit", "df_dit_step", "df_handoff", "df_set_ratio", "df_poll"):
        assert n in names


def test_library_exports_every_declared_symbol(lib_path):
    lib = ctypes.CDLL(lib_path)
    for n in _declared():
        assert hasattr(lib, n), n
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (df_\w+)", out))
    assert set(_declared()) <= exported
    assert "torch" not in out and "at::" not in out


def test_binding_covers_header():
    from paper_2605_25550_b200 import binding
    assert set(_declared()) == set(binding.EXPORTS)


def test_binding_loads(lib_path):
    from paper_2605_25550_b200 import binding
    binding.load(lib_path)


def test_library_built_for_sm100a(lib_path):
    out = subprocess.run(["cuobjdump", "--list-elf", lib_path], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", lib_path], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass and "UTMALDG" in sass and "LDTM" in sass  # tcgen05 + TMA + TMEM loads


def test_product_path_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2605_25550_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cpp", ".cu", ".h", ".cuh")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle\b", txt, re.M), f
                assert "oracle/" not in txt or f.endswith(".py") is False or "import" not in txt, f
