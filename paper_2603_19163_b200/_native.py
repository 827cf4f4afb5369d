"""ctypes binding of libcugenopt.so (include/cugenopt.h).

There is no CPU fallback: importing this module never fails, but every call
that needs the library raises `NativeUnavailable` when the .so is missing or
no CUDA device is visible.  The library is loaded from the package tree
(`paper_2603_19163_b200/lib/libcugenopt.so`), never from site-packages.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libcugenopt.so"

GO_OK, GO_E_INVALID, GO_E_CUDA, GO_E_UNSUPPORTED, GO_E_COMPILE, GO_E_NODEVICE = 0, -1, -2, -3, -4, -5
GO_TSP, GO_VRPTW, GO_QAP, GO_JSP_INT, GO_KNAPSACK, GO_CVRP, GO_USER = range(7)
GO_VRP_PRIORITY, GO_VRP_NONLINEAR = 7, 8
ENC_PERM, ENC_BINARY, ENC_INTEGER = range(3)
MOVE_NONE, MOVE_SWAP, MOVE_REVERSE, MOVE_SEGMENT = range(4)
MOVE_THREE_OPT = 8  # + variant 0..6
MIG = {"ring": 0, "global_top_n": 1, "hybrid": 2}


class NativeUnavailable(RuntimeError):
    """libcugenopt.so or a CUDA device is missing: the device path cannot run."""


class NativeError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"libcugenopt status {status}: {msg}")
        self.status = status


class Move(C.Structure):
    _fields_ = [("kind", C.c_int32), ("a", C.c_int32), ("b", C.c_int32), ("c", C.c_int32)]


class DeviceInfo(C.Structure):
    _fields_ = [("device", C.c_int32), ("sm_count", C.c_int32), ("max_smem_optin", C.c_int32),
                ("l2_bytes", C.c_int32), ("cc_major", C.c_int32), ("cc_minor", C.c_int32),
                ("global_mem", C.c_int64), ("name", C.c_char * 96)]


_PD = C.POINTER(C.c_double)
_PI = C.POINTER(C.c_int32)


class ProblemDesc(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n", C.c_int32), ("d1", C.c_int32), ("d2", C.c_int32),
                ("dist", _PD), ("flow", _PD), ("weights", _PD), ("values", _PD),
                ("demands", _PD), ("ready", _PD), ("due", _PD), ("service", _PD),
                ("capacity", C.c_double), ("n_jobs", C.c_int32), ("n_machines", C.c_int32),
                ("ops_per_job", C.c_int32), ("jsp_machine", _PI), ("jsp_duration", _PI),
                ("lb", C.c_int32), ("ub", C.c_int32), ("n_obj", C.c_int32),
                ("obj_kind", C.c_int32 * 2), ("priorities", _PD)]


class UserProblemDesc(C.Structure):  # go_user_problem_desc
    _fields_ = [("encoding", C.c_int32), ("n", C.c_int32), ("lb", C.c_int32), ("ub", C.c_int32),
                ("compute_obj", C.c_char_p), ("compute_penalty", C.c_char_p),
                ("n_data", C.c_int32), ("data_names", C.POINTER(C.c_char_p)),
                ("data", C.POINTER(_PD)), ("data_lens", C.POINTER(C.c_int64)),
                ("rows", C.c_int32), ("compute_obj2", C.c_char_p)]


class CustomOp(C.Structure):
    _fields_ = [("id", C.c_int32), ("name", C.c_char_p), ("cuda_body", C.c_char_p)]


class EngineConfig(C.Structure):
    _fields_ = [("population", C.c_int32), ("team_size", C.c_int32),
                ("teams_per_cta", C.c_int32), ("seed", C.c_uint64), ("t0", C.c_double),
                ("cooling_alpha", C.c_double), ("penalty_weight", C.c_double),
                ("aos_interval", C.c_int32), ("aos_alpha", C.c_double),
                ("aos_floor", C.c_double), ("aos_cap", C.c_double), ("aos_eps", C.c_double),
                ("stagnation_threshold", C.c_int32), ("islands", C.c_int32),
                ("migration", C.c_int32), ("migration_interval", C.c_int32),
                ("top_n", C.c_int32), ("elite_interval", C.c_int32),
                ("has_target", C.c_int32), ("target_objective", C.c_double),
                ("evolver_offset", C.c_int32), ("maximize", C.c_int32),
                ("obj_weight", C.c_double), ("obj_weight2", C.c_double), ("lex", C.c_int32),
                ("lex_first", C.c_int32), ("lex_tol", C.c_double * 2), ("maximize2", C.c_int32)]


class RunStats(C.Structure):
    _fields_ = [("generations", C.c_int64), ("lane_evals", C.c_int64),
                ("kernel_launches", C.c_int64), ("device_ms", C.c_double),
                ("stopped_by", C.c_int32), ("error_flags", C.c_int32),
                ("reads_pos", C.c_int64), ("reads_elem", C.c_int64),
                ("elem_bytes", C.c_int32), ("gene_bytes", C.c_int32),
                ("evolve_ms", C.c_double), ("evolve_launches", C.c_int64)]


_lib = None


def _bind(lib):
    V, P = C.c_void_p, C.POINTER
    sig = {
        "go_abi_version": ([], C.c_int),
        "go_last_error": ([], C.c_char_p),
        "go_device_count": ([P(C.c_int)], C.c_int),
        "go_device_query": ([C.c_int, P(DeviceInfo)], C.c_int),
        "go_problem_create": ([P(ProblemDesc), C.c_int, P(V)], C.c_int),
        "go_problem_create_user": ([P(UserProblemDesc), C.c_int, P(V), C.c_char_p, C.c_int],
                                   C.c_int),
        "go_problem_destroy": ([V], C.c_int),
        "go_problem_layout": ([V, P(C.c_int64), P(C.c_int32)], C.c_int),
        "go_problem_occupancy": ([V, C.c_int, C.c_int, _PI, _PI, _PI, P(C.c_int64)], C.c_int),
        "go_eval_batch": ([V, _PI, _PI, C.c_int, _PD, _PD], C.c_int),
        "go_delta_batch": ([V, _PI, _PI, C.c_int, P(Move), C.c_double, _PD, _PI], C.c_int),
        "go_init_population": ([V, C.c_int, C.c_uint64, C.c_uint64, _PI, _PI, C.c_int, C.c_int,
                                C.c_int, C.c_double, _PI, _PI, _PD, _PD, _PI], C.c_int),
        "go_problem_set_custom_ops": ([V, P(CustomOp), C.c_int, _PI, _PI, C.c_uint64, _PI,
                                       C.c_char_p, C.c_int], C.c_int),
        "go_jit_compile": ([C.c_int, P(CustomOp), C.c_int, C.c_char_p, C.c_int, C.c_char_p],
                           C.c_int),
        "go_engine_create": ([V, P(EngineConfig), P(V)], C.c_int),
        "go_engine_destroy": ([V], C.c_int),
        "go_engine_set_registry": ([V, C.c_int, _PI, _PD, _PD, _PD, C.c_double, _PD], C.c_int),
        "go_engine_set_population": ([V, _PI, _PI, _PD, _PD], C.c_int),
        "go_engine_run": ([V, C.c_int64, C.c_double, P(RunStats)], C.c_int),
        "go_engine_step": ([V, C.c_int64, C.c_double, _PI, _PI, _PI, _PI], C.c_int),
        "go_engine_get_population": ([V, _PI, _PI, _PD, _PD], C.c_int),
        "go_engine_get_best": ([V, _PI, _PI, _PD, _PD, P(C.c_int64)], C.c_int),
        "go_engine_get_registry": ([V, _PD, _PD, _PI], C.c_int),
        "go_engine_get_history": ([V, _PD, C.c_int64, P(C.c_int64)], C.c_int),
        "go_engine_set_history": ([V, C.c_int], C.c_int),
        "go_elite_record_bytes": ([V, P(C.c_int64)], C.c_int),
        "go_engine_export_elites": ([V, V, C.c_int], C.c_int),
        "go_engine_import_elites": ([V, V, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int64],
                                    C.c_int),
        "go_engine_debug_counters": ([V, P(C.c_int64), C.c_int], C.c_int),
        "go_engine_stream": ([V, P(V)], C.c_int),
        "go_engine_sync": ([V], C.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    return list(sig)


EXPORTED = None


def load(require_device: bool = True):
    """Load the in-tree library (building it first if sources are newer)."""
    global _lib, EXPORTED
    if _lib is None:
        if os.environ.get("GO_AUTOBUILD", "1") == "1":
            try:
                from . import build
                build.build()
            except Exception as exc:  # noqa: BLE001 - surfaced below if the .so is absent
                if not LIB_PATH.exists():
                    raise NativeUnavailable(f"cannot build libcugenopt.so: {exc}") from exc
        if not LIB_PATH.exists():
            raise NativeUnavailable(f"{LIB_PATH} not built (run __graft_entry__.build())")
        lib = C.CDLL(str(LIB_PATH))
        EXPORTED = _bind(lib)
        _lib = lib
    if require_device:
        n = C.c_int(0)
        if _lib.go_device_count(C.byref(n)) != GO_OK or n.value == 0:
            raise NativeUnavailable("no CUDA device visible: the cuGenOpt engine has no CPU path")
    return _lib


def check(status):
    if status != GO_OK:
        raise NativeError(status, _lib.go_last_error().decode(errors="replace"))


def dptr(a):
    return a.ctypes.data_as(_PD)


def iptr(a):
    return a.ctypes.data_as(_PI)


def f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def device_info(device: int = 0) -> DeviceInfo:
    lib = load()
    info = DeviceInfo()
    check(lib.go_device_query(device, C.byref(info)))
    return info


def device_count() -> int:
    """CUDA devices visible to the engine (raises NativeUnavailable on none)."""
    lib = load()
    n = C.c_int(0)
    check(lib.go_device_count(C.byref(n)))
    return n.value
