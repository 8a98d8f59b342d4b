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


def test_kernel_plan_roundtrip(so):
    """pk_plan_options: the production defaults, a scoped change, invalid values
    rejected (packtrain_b200.h)."""
    d = _lib.plan_options()
    assert d == {"fwd": 0, "fwd_cluster": 0, "tcgen05": 1, "mlp1": 1, "m1x": 0, "fwd_split": 1,
                 "wgrad_narrow": 1, "inline_desc": 1, "run_batch": 0, "trace": 0,
                 "conv_cluster": 1, "conv_halo": 1}
    with _lib.kernel_plan(fwd="stream", conv_cluster=0):
        cur = _lib.plan_options()
        assert cur["fwd"] == 2 and cur["conv_cluster"] == 0 and cur["tcgen05"] == 1
    assert _lib.plan_options() == d
    with pytest.raises(_lib.PKError):
        _lib.set_plan_options(fwd=7)
    assert _lib.plan_options() == d
    with pytest.raises(KeyError):
        _lib.set_plan_options(no_such_option=1)


def test_cnn_op_layout():
    """pk_cnn_op: kind, nprob, cfg0, cfg1, lane, pad0 (int32) then the problems pointer."""
    assert ctypes.sizeof(_lib.CnnOp) == 32
    assert _lib.CnnOp.lane.offset == 16 and _lib.CnnOp.probs.offset == 24
    # pk_cnn_im2col: two pointers then twelve int32
    assert ctypes.sizeof(_lib.CnnIm2col) == 64 and _lib.CnnIm2col.ldo.offset == 60
    assert ctypes.sizeof(_lib.PlanOptions) == 16 * 4
