"""The C-ABI library loads and exports every symbol include/*.h declares
(CPU: no compute calls), and the ctypes structs match the header layout."""
import ctypes
import os
import re
import subprocess

import pytest

from paper_2002_02885_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "packtrain_b200.h")


def _declared():
    text = open(HDR).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(pk_\w+)\s*\(", text, re.M)))


@pytest.fixture(scope="module")
def so():
    if not os.path.exists(_lib.LIB_PATH):
        subprocess.run(["make", "-C", os.path.join(ROOT, "paper_2002_02885_b200", "csrc")],
                       check=True)
    return _lib.load_library()


def test_every_declared_symbol_is_exported(so):
    decl = _declared()
    assert len(decl) >= 25
    for name in decl:
        assert hasattr(so, name), name
    assert sorted(decl) == sorted(_lib.EXPORTS)


def test_abi_version(so):
    assert so.pk_abi_version() == 1


def test_struct_layouts_match_header():
    # pk_member_desc: 1 + 9 + 2 int32, 2 doubles, 2 int32
    assert ctypes.sizeof(_lib.MemberDesc) == 4 * 12 + 16 + 8
    assert ctypes.sizeof(_lib.Feed) == 8 + 8 + 8 + 4 + 4
    assert ctypes.sizeof(_lib.Status) == 16


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_ctx_create_without_gpu_fails_loudly(so):
    from _helpers import has_gpu
    if has_gpu():
        pytest.skip("GPU present")
    ptr = ctypes.c_void_p()
    rc = so.pk_ctx_create(0, 0, ctypes.byref(ptr))
    assert rc != 0  # no silent CPU fallback
