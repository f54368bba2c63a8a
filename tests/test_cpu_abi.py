"""CPU-side checks of the C-ABI boundary: the library builds, loads and
exports exactly what include/coinfer_b200.h declares (no GPU needed)."""
import ctypes as C
import os
import re

from paper_2206_06304_b200 import _abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "coinfer_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(coinfer_[a-z0-9_]+)\s*\(", src)))


def test_header_and_binding_agree():
    assert declared_functions() == sorted(_abi.PRODUCT_SYMBOLS)


def test_library_exports_every_declared_symbol():
    lib = _abi.load_library()
    for name in declared_functions():
        assert hasattr(lib, name), name


def test_abi_version_and_messages():
    lib = _abi.load_library()
    assert lib.coinfer_abi_version() == _abi.ABI_VERSION
    msg = lib.coinfer_status_message(_abi.ST_INFEASIBLE, b"ipssa").decode()
    assert msg == "ip_ssa: no batch bound admits every user"
    assert lib.coinfer_status_message(_abi.ST_INFEASIBLE, b"og").decode() == \
        "baseline: user cannot meet the deadline locally"
    assert lib.coinfer_status_message(_abi.ST_BAD_RATE, b"og").decode() == \
        "scenario: rates must be positive"
    assert lib.coinfer_status_message(_abi.ST_INFEASIBLE, b"lc").decode() == \
        "baseline: user cannot meet the deadline locally"
    for m in (b"ps", b"fifo"):
        assert lib.coinfer_status_message(_abi.ST_INFEASIBLE, m).decode() == \
            "baseline: user cannot meet the deadline"


def test_struct_layout_matches_header():
    # pointer-sized fields after two int32 headers
    assert C.sizeof(_abi.Profile) == 8 + 3 * 8
    assert C.sizeof(_abi.Users) == 16 + 9 * 8
    assert C.sizeof(_abi.IpssaOut) == 8 * 8
    assert C.sizeof(_abi.OgOut) == 15 * 8
    assert C.sizeof(_abi.ScheduleOut) == 5 * 8


def test_no_context_without_gpu_is_loud():
    import torch
    if torch.cuda.is_available():
        return
    lib = _abi.load_library()
    assert not lib.coinfer_ctx_create(0)
    from paper_2206_06304_b200 import Engine, SolverError
    try:
        Engine(0)
    except SolverError:
        pass
    else:
        raise AssertionError("Engine must fail loudly without a GPU")
