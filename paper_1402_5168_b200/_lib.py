"""ctypes loader for librexp.so (include/rexp.h).  Fails loudly if the library is missing."""
import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# REXP_LIB: an alternative in-tree build of the same library (e.g. one compiled
# with -DREXP_CMUL3=0 for accuracy experiments); the default is librexp.so
LIB_PATH = os.path.join(_HERE, os.environ.get("REXP_LIB", "librexp.so"))


class RexpProblem(ctypes.Structure):
    _fields_ = [("model", ctypes.c_int32), ("n", ctypes.c_int32), ("p", ctypes.c_int32),
                ("f", ctypes.c_double), ("kappa", ctypes.POINTER(ctypes.c_double))]


class RexpOptions(ctypes.Structure):
    _fields_ = [("nrhs", ctypes.c_int32), ("store", ctypes.c_int32), ("device", ctypes.c_int32),
                ("half_begin", ctypes.c_int32), ("half_end", ctypes.c_int32), ("nthreads", ctypes.c_int32)]


# (name, restype, argtypes) for every symbol declared in include/rexp.h
_P = ctypes.c_void_p
_D = ctypes.POINTER(ctypes.c_double)
SIGNATURES = [
    ("rexp_default_options", None, [ctypes.POINTER(RexpOptions)]),
    ("rexp_setup", ctypes.c_int, [ctypes.POINTER(RexpProblem), ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                  ctypes.POINTER(RexpOptions), ctypes.POINTER(_P)]),
    ("rexp_apply", ctypes.c_int, [_P, _P, ctypes.c_int32, ctypes.c_int32, _P]),
    ("rexp_free", None, [_P]),
    ("rexp_last_error", ctypes.c_char_p, []),
    ("rexp_partial_len", ctypes.c_int64, [_P]),
    ("rexp_step_partial", ctypes.c_int, [_P, _P, _P, _P]),
    ("rexp_step_finish", ctypes.c_int, [_P, _P, _P, _P]),
    ("rexp_num_nodes", ctypes.c_int64, [_P]),
    ("rexp_num_poles", ctypes.c_int32, [_P]),
    ("rexp_num_half_poles", ctypes.c_int32, [_P]),
    ("rexp_get_poles", ctypes.c_int, [_P, _D, _D]),
    ("rexp_get_accuracy", ctypes.c_int, [_P, _D, _D]),
    ("rexp_node_coords", ctypes.c_int, [_P, _D, _D]),
    ("rexp_mesh_num_nodes", ctypes.c_int64, [ctypes.c_int32, ctypes.c_int32]),
    ("rexp_mesh_coords", ctypes.c_int, [ctypes.c_int32, ctypes.c_int32, _D, _D]),
    ("rexp_store_bytes", ctypes.c_int64, [_P]),
    ("rexp_work_bytes", ctypes.c_int64, [_P]),
    ("rexp_launches_per_step", ctypes.c_int32, [_P]),
    ("rexp_leaf_solver", ctypes.c_int32, [_P]),
    ("rexp_stage_report", ctypes.c_int, [_P, ctypes.c_char_p, ctypes.c_int32]),
    ("rexp_timing_begin", ctypes.c_int, [_P]),
    ("rexp_timing_end", ctypes.c_int, [_P, _D, ctypes.POINTER(ctypes.c_int32)]),
    ("rexp_export_num_levels", ctypes.c_int32, [_P]),
    ("rexp_export_level_info", ctypes.c_int, [_P, ctypes.c_int32, ctypes.POINTER(ctypes.c_int64)]),
    ("rexp_export_matrix", ctypes.c_int, [_P, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, _D]),
    ("rexp_export_index", ctypes.c_int, [_P, ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(ctypes.c_int32)]),
]

_lib = None


def load():
    """Load librexp.so (built in-tree by build.py / __graft_entry__.build())."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"librexp.so not found at {LIB_PATH}: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(LIB_PATH)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class RexpError(RuntimeError):
    pass


def check(rc, what):
    if rc != 0:
        msg = load().rexp_last_error().decode()
        raise RexpError(f"{what} failed ({rc}): {msg}")
