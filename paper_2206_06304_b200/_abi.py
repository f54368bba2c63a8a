"""ctypes mirror of include/coinfer_b200.h and the loader of the product library.

The structs here are shared by the product path (libcoinfer_b200.so) and the
test-side checkers (oracle/liboracle.so, oracle/_ref/libcoinfer_ref.so), which
export the same SoA entry points, so a test drives all three identically.

`load_library()` never falls back to anything: if the CUDA library is missing
it raises, so no solve can silently run somewhere else.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("COINFER_LIB") or os.path.join(_HERE, "libcoinfer_b200.so")

ABI_VERSION = 3
OK, E_ARG, E_PROFILE, E_CUDA, E_UNSUPPORTED = 0, 1, 2, 3, 4
ST_OK, ST_INFEASIBLE = 0, 1
ST_BAD_FREQ, ST_NEG_KAPPA, ST_BAD_RATE, ST_NEG_POWER = 10, 11, 12, 13
ST_NEG_ARRIVAL, ST_EARLY_DEADLINE, ST_SHORT_TABLE = 14, 15, 16
ST_ZERO_BOUND, ST_BOUND_PAST_TABLE = 17, 18
ST_BAD_BATCH_ID, ST_NONPOS_FREQ = 19, 23
N_CONSTRAINTS = 7
CONSTRAINT_IDS = ["C7-batchsize", "C8-samesubtask", "C9-batchready", "C11-occupancy",
                  "C12-precedence", "C15-deadline", "C17-initial"]
MEM_HOST, MEM_DEVICE = 0, 1
MAX_SUBTASKS = 16

_dp = C.POINTER(C.c_double)
_i32p = C.POINTER(C.c_int32)
_u8p = C.POINTER(C.c_uint8)
_i64p = C.POINTER(C.c_int64)


class Profile(C.Structure):
    _fields_ = [("N", C.c_int32), ("b_max", C.c_int32), ("work", _dp),
                ("data_bits", _dp), ("latency", _dp)]


USER_FIELDS = ("f_min", "f_max", "kappa", "rate_up", "power_up", "arrival",
               "deadline", "rate_down", "power_down")


class Users(C.Structure):
    _fields_ = [("n_inst", C.c_int64), ("M", C.c_int32), ("mem", C.c_int32)] + [
        (f, _dp) for f in USER_FIELDS]


IPSSA_FIELDS = [("status", _i32p, "K"), ("batch_bound", _i32p, "K"),
                ("pipeline_feasible", _u8p, "K"), ("energy", _dp, "K"),
                ("split", _u8p, "KM"), ("freq", _dp, "KM"),
                ("user_energy", _dp, "KM"), ("batch_size", _i32p, "KN")]

OG_FIELDS = [("status", _i32p, "K"), ("fallback", _u8p, "K"), ("energy", _dp, "K"),
             ("n_groups", _i32p, "K"), ("order", _i32p, "KM"),
             ("group_of_user", _i32p, "KM"), ("split", _u8p, "KM"), ("freq", _dp, "KM"),
             ("user_energy", _dp, "KM"), ("group_lo", _i32p, "KM"),
             ("group_size", _i32p, "KM"), ("group_b", _i32p, "KM"),
             ("group_deadline", _dp, "KM"), ("group_energy", _dp, "KM"),
             ("group_batch_size", _i32p, "KMN")]


class IpssaOut(C.Structure):
    _fields_ = [(n, t) for n, t, _ in IPSSA_FIELDS]


class OgOut(C.Structure):
    _fields_ = [(n, t) for n, t, _ in OG_FIELDS]


SCHEDULE_FIELDS = [("x", _i32p, "KMN"), ("n_batches", _i32p, "K"),
                   ("batch_start", _dp, "KMN"), ("completion", _dp, "KMN1"),
                   ("freq", _dp, "KM")]


class ScheduleOut(C.Structure):
    _fields_ = [(n, t) for n, t, _ in SCHEDULE_FIELDS]


BASELINE_LC, BASELINE_PS, BASELINE_FIFO, BASELINE_IPSSA_NP = 0, 1, 2, 3
BASELINE_MODES = {"LC": BASELINE_LC, "PS": BASELINE_PS, "FIFO": BASELINE_FIFO,
                  "IPSSA_NP": BASELINE_IPSSA_NP}

class SampleCfg(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("cell_radius", "bandwidth", "noise_dbm_hz", "tx_power",
                                          "uplink_power", "downlink_power", "edge_power",
                                          "edge_efficiency", "device_efficiency", "alpha",
                                          "shadow_sigma_db")] + [
        ("deadline_uniform", C.c_int32), ("reserved", C.c_int32),
        ("deadline_low", C.c_double), ("deadline_high", C.c_double)]


ST_NO_DEADLINE = 24
ST_TOO_LARGE = 25

ARRIVAL_BERNOULLI, ARRIVAL_IMMEDIATE = 0, 1
SOLVER_IPSSA, SOLVER_OG = 0, 1
POLICY_TW, POLICY_LOCAL = 0, 1
ST_NOT_RELEASED, ST_FLOOR_ABOVE_LLOW, ST_SLIPPED = 20, 21, 22


class OnlineCfg(C.Structure):
    _fields_ = [("arrival", C.c_int32), ("solver", C.c_int32), ("policy", C.c_int32),
                ("window", C.c_int32), ("p_arrive", C.c_double), ("l_low", C.c_double),
                ("l_high", C.c_double), ("slot", C.c_double), ("threshold", C.c_double),
                ("horizon", C.c_int64)]


class OnlineOut(C.Structure):
    _fields_ = [("status", _i32p), ("totals", _dp), ("counts", _i64p), ("n_trace", C.c_int64),
                ("trace_reward", _dp), ("trace_energy", _dp), ("trace_pending", _i32p),
                ("trace_edge_busy", _dp), ("trace_action", _i32p), ("trace_forced", _i32p),
                ("final_state", _dp), ("draws", _i64p)]


# name -> (restype, argtypes) of every symbol include/coinfer_b200.h declares
PRODUCT_SYMBOLS = {
    "coinfer_abi_version": (C.c_int, []),
    "coinfer_ctx_create": (C.c_void_p, [C.c_int]),
    "coinfer_ctx_destroy": (None, [C.c_void_p]),
    "coinfer_ctx_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "coinfer_ctx_reset_stream": (C.c_int, [C.c_void_p]),
    "coinfer_ctx_synchronize": (C.c_int, [C.c_void_p]),
    "coinfer_last_error": (C.c_char_p, [C.c_void_p]),
    "coinfer_status_message": (C.c_char_p, [C.c_int32, C.c_char_p]),
    "coinfer_ctx_launch_count": (C.c_int64, [C.c_void_p]),
    "coinfer_probe_fp64": (C.c_int, [C.c_void_p, _dp]),
    "coinfer_ipssa_batch": (C.c_int, [C.c_void_p, C.POINTER(Profile), C.POINTER(Users), _dp,
                                      C.POINTER(IpssaOut)]),
    "coinfer_fixed_batch": (C.c_int, [C.c_void_p, C.POINTER(Profile), C.POINTER(Users), _dp,
                                      _i32p, C.POINTER(IpssaOut)]),
    "coinfer_og_batch": (C.c_int, [C.c_void_p, C.POINTER(Profile), C.POINTER(Users),
                                   C.POINTER(OgOut)]),
    "coinfer_sweep_batch": (C.c_int, [C.c_void_p, C.POINTER(Profile), C.POINTER(Users),
                                      C.POINTER(IpssaOut), C.POINTER(OgOut)]),
    "coinfer_count_work": (C.c_int, [C.c_void_p, C.POINTER(Profile), C.POINTER(Users),
                                     C.POINTER(IpssaOut), C.POINTER(OgOut), C.POINTER(C.c_uint64)]),
    "coinfer_ipssa_schedule": (C.c_int, [C.c_void_p, C.POINTER(Profile), C.POINTER(Users), _dp,
                                         C.POINTER(IpssaOut), C.POINTER(ScheduleOut)]),
    "coinfer_og_schedule": (C.c_int, [C.c_void_p, C.POINTER(Profile), C.POINTER(Users),
                                      C.POINTER(OgOut), C.POINTER(ScheduleOut)]),
    "coinfer_baseline_batch": (C.c_int, [C.c_void_p, C.POINTER(Profile), C.POINTER(Users),
                                         C.c_int32, C.POINTER(IpssaOut),
                                         C.POINTER(ScheduleOut)]),
    "coinfer_validate_batch": (C.c_int, [C.c_void_p, C.POINTER(Profile), C.POINTER(Users),
                                         C.POINTER(ScheduleOut), C.c_double, _i32p, _i32p, _dp]),
    "coinfer_sample_cfg_defaults": (None, [C.POINTER(SampleCfg)]),
    "coinfer_sub_seed": (C.c_uint64, [C.c_uint64, C.c_uint64, C.c_uint64]),
    "coinfer_sample_batch": (C.c_int, [C.c_void_p, C.POINTER(Profile), C.POINTER(SampleCfg),
                                       C.POINTER(C.c_uint64), C.POINTER(Users), _i32p]),
    "coinfer_oracle_structured_batch": (C.c_int, [C.c_void_p, C.POINTER(Profile), C.POINTER(Users),
                                                  _dp, _i32p, _i32p, _dp, _u8p, _u8p, _u8p]),
    "coinfer_oracle_grouping_batch": (C.c_int, [C.c_void_p, C.POINTER(Profile), C.POINTER(Users),
                                                C.c_int32, _i32p, _dp, _i32p, _i32p, _u8p]),
    "coinfer_best_partition": (C.c_int, [C.c_void_p, C.POINTER(Profile), C.POINTER(Users), _dp,
                                         _i32p, _dp, _dp, _u8p]),
    "coinfer_online_run": (C.c_int, [C.c_void_p, C.POINTER(Profile), C.POINTER(Users),
                                     C.POINTER(OnlineCfg), C.POINTER(C.c_uint64), C.c_int64,
                                     C.POINTER(OnlineOut)]),
}


def bind(lib: C.CDLL, table: dict) -> C.CDLL:
    for name, (res, args) in table.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_lib = None


def load_library(path: str = LIB_PATH) -> C.CDLL:
    """Load the CUDA solver library; raise (never fall back) if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(
            f"coinfer: CUDA solver library not built ({path}); run "
            "`python -c 'import __graft_entry__ as g; g.build()'` or "
            "`make -C paper_2206_06304_b200/csrc`")
    lib = bind(C.CDLL(path), PRODUCT_SYMBOLS)
    if lib.coinfer_abi_version() != ABI_VERSION:
        raise RuntimeError("coinfer: ABI version mismatch")
    _lib = lib
    return lib
