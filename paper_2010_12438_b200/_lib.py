"""ctypes binding of libgo_b200.so (include/go_b200.h).

The shared library is the product: there is no CPU fallback.  Importing this
module never needs a GPU (so CPU tests can check the exported symbols), but every
compute call raises if the library or a CUDA device is missing.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libgo_b200.so"

GO_OK, GO_ERR_VALUE, GO_ERR_CUDA, GO_ERR_CYCLE, GO_ERR_NONFINITE, GO_ERR_DEADLOCK, \
    GO_ERR_UNSUPPORTED = range(7)

# every symbol include/go_b200.h declares (checked by tests/test_host.py::test_header_symbols_exported)
EXPORTS = (
    "go_last_error", "go_version", "go_ctx_create", "go_ctx_destroy", "go_ctx_workspace_bytes",
    "go_launch_count", "go_ctx_set_timing", "go_ctx_kernel_stats",
    "go_topo_order", "go_greedy_cuts", "go_apply_fusion", "go_graph_create", "go_graph_destroy", "go_graph_topo",
    "go_graph_num_neighbors", "go_graph_set_fusion", "go_param_count", "go_forward",
    "go_forward_status", "go_neighbor_arrays", "go_sample", "go_simulate", "go_ppo_grad",
    "go_adam", "go_adam64", "go_simulate_trace", "go_anneal",
)


class GoConfig(C.Structure):
    _fields_ = [("gs_layers", C.c_int32), ("gs_dim", C.c_int32), ("gs_knn", C.c_int32),
                ("trf_layers", C.c_int32), ("d_model", C.c_int32), ("n_head", C.c_int32),
                ("d_head", C.c_int32), ("d_inner", C.c_int32), ("segment_len", C.c_int32),
                ("num_tasks", C.c_int32), ("task_sizes", C.c_int32 * 3)]


class GoBatch(C.Structure):
    _fields_ = [("num_forwards", C.c_int32), ("graphs", C.POINTER(C.c_void_p)),
                ("row_counts", C.POINTER(C.c_int64)), ("embed_seeds", C.POINTER(C.c_int64)), ("prev_actions", C.c_void_p),
                ("stage_mask", C.c_int32), ("ablate_mask", C.c_int32),
                ("mod_override", C.c_void_p), ("features", C.c_void_p),
                ("feature_dim", C.c_int32), ("reps", C.c_void_p),
                ("cache_hook", C.c_void_p), ("cache_hook_user", C.c_void_p)]


# void cache_hook(void* user, int32 layer, const float* xm, float* prefix, int64 rows, int32 dm)
CACHE_HOOK = C.CFUNCTYPE(None, C.c_void_p, C.c_int32, C.POINTER(C.c_float),
                         C.POINTER(C.c_float), C.c_int64, C.c_int32)


class GoError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


_lib = None

P = C.c_void_p
I32, I64, F64 = C.c_int32, C.c_int64, C.c_double
PI32, PI64, PF64 = C.POINTER(C.c_int32), C.POINTER(C.c_int64), C.POINTER(C.c_double)

_SIGS = {
    "go_last_error": (C.c_char_p, []),
    "go_version": (C.c_int, []),
    "go_ctx_create": (C.c_int, [C.c_int, C.POINTER(P)]),
    "go_ctx_destroy": (C.c_int, [P]),
    "go_ctx_workspace_bytes": (C.c_int, [P, PI64]),
    "go_launch_count": (C.c_longlong, []),
    "go_ctx_set_timing": (C.c_int, [P, C.c_int]),
    "go_ctx_kernel_stats": (C.c_int, [P, I32, PI64, PF64, PF64]),
    "go_topo_order": (C.c_int, [I32, I64, P, P, P]),
    "go_greedy_cuts": (C.c_int, [I32, P, I32, P]),
    "go_apply_fusion": (C.c_int, [I32, I64, P, P, P, P, I32, P]),
    "go_graph_create": (C.c_int, [P, I32, I64, P, P, P, P, P, P, P, C.POINTER(P)]),
    "go_graph_destroy": (C.c_int, [P]),
    "go_graph_topo": (C.c_int, [P, P]),
    "go_graph_num_neighbors": (C.c_int, [P, PI64]),
    "go_graph_set_fusion": (C.c_int, [P, P, PI32, PI32]),
    "go_param_count": (C.c_int, [C.POINTER(GoConfig), PI32]),
    "go_forward": (C.c_int, [P, C.POINTER(GoConfig), P, P, C.POINTER(GoBatch), P, P, P, P, P, P]),
    "go_forward_status": (C.c_int, [P, C.POINTER(GoConfig), P, P, C.POINTER(GoBatch), P, P, P,
                                    P, P, P, P]),
    "go_neighbor_arrays": (C.c_int, [P, P, I64, I32, P, P, P]),
    "go_sample": (C.c_int, [P, C.POINTER(GoConfig), I32, P, P, P, P, I32, F64, P, P, P]),
    "go_ppo_grad": (C.c_int, [P, C.POINTER(GoConfig), P, P, C.POINTER(GoBatch), P, P, P, F64, F64,
                              F64, I32, P, P, P]),
    "go_adam": (C.c_int, [P, P, P, P, P, I64, I64, F64, F64, F64, F64, P]),
    "go_adam64": (C.c_int, [P, P, P, P, P, P, I64, I64, F64, F64, F64, F64, P]),
    "go_simulate": (C.c_int, [P, P, I32, P, P, I32, I32, P, P, P, P, I32, F64, P, P, P, P, P,
                              P, P]),
    "go_anneal": (C.c_int, [P, P, I32, P, P, P, I32, P, P, P, P, I32, I32, I32, F64, F64, I32,
                            P, P, P, P]),
    "go_simulate_trace": (C.c_int, [P, P, P, P, I32, P, P, P, P, I32, P, P, P, P, P, P, I64, P,
                                    P]),
}


def lib():
    """Load libgo_b200.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} not built: run python -m paper_2010_12438_b200.build")
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(status: int):
    """Map a go_* status to the reference's exception types."""
    if status == GO_OK:
        return
    msg = lib().go_last_error().decode(errors="replace")
    if status == GO_ERR_VALUE:
        raise ValueError(msg)
    if status == GO_ERR_CYCLE:
        from .graph import GraphError
        raise GraphError(msg)
    if status == GO_ERR_NONFINITE:
        raise FloatingPointError(msg)
    if status == GO_ERR_DEADLOCK:
        raise AssertionError(msg)
    raise GoError(status, msg)


def call(name, *args):
    check(getattr(lib(), name)(*args))


def ptr(t) -> int | None:
    """Raw device/host address of a torch tensor or numpy array (None -> NULL)."""
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        return t.data_ptr()
    return t.ctypes.data
