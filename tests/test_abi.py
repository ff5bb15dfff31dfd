"""CPU checks of the C-ABI boundary: the library builds, loads without a GPU
and exports every function include/ravgmg.h declares (no compute calls)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ravgmg.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(?:rav_status|void|const char\s*\*|int64_t)\s+((?:rav|mg)_\w+)\s*\(", src)
    return sorted(set(names))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("rav_setup", "rav_smooth", "mg_setup", "mg_vcycle", "mg_solve", "rav_gen_operator",
                 "rav_gen_patches", "rav_gen_prolongation", "rav_last_error", "rav_destroy", "mg_destroy"):
        assert must in names


def test_library_builds_loads_and_exports_all_symbols():
    from paper_2103_10127_b200 import build
    lib_path = build.build()
    lib = ctypes.CDLL(lib_path)
    for name in declared_functions():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T ((?:rav|mg)_\w+)", out))
    assert set(declared_functions()) <= exported
    lib.rav_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.rav_version()
    lib.rav_last_error.restype = ctypes.c_char_p
    assert lib.rav_last_error() == b""


def test_library_is_sm100a_code():
    from paper_2103_10127_b200 import build
    lib_path = build.build()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib_path], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_oracle_and_product_share_no_code():
    # the product tree never references the oracle and vice versa
    for dirpath, _, files in os.walk(os.path.join(ROOT, "paper_2103_10127_b200")):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"(#|//).*", "", txt).lower() or f == "__init__.py", f
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith((".py", ".c")):
            txt = open(os.path.join(ROOT, "oracle", f)).read()
            assert "paper_2103_10127_b200" not in re.sub(r'"""[\s\S]*?"""|/\*[\s\S]*?\*/', "", txt), f
