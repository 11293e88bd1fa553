"""ctypes binding of libffb200.so (include/ffb200.h) — the drop-in boundary.

Loads the in-tree sm_100a library and fails loudly when it (or a CUDA device)
is missing: the engine has no CPU fallback.
"""
import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libffb200.so")

FFB_OK = 0
FFB_ERR_DIMENSION = 1
FFB_ERR_SINGULAR_TRAILING = 2
FFB_ERR_CERTIFICATION = 3
FFB_ERR_NUMERICAL = 4
FFB_ERR_CUDA = 5
FFB_ERR_ARGUMENT = 6

FFB_MODE_TRQRCP = 0
FFB_MODE_SRQR = 1
FFB_MODE_FLIPFLOP = 2
FFB_LAYOUT_COL = 0
FFB_LAYOUT_ROW = 1

EXPORTS = ("ffb_ctx_create", "ffb_ctx_destroy", "ffb_last_error", "ffb_version",
           "ffb_workspace_query", "ffb_run", "ffb_flipflop", "ffb_gemm", "ffb_block_pivots",
           "ffb_run_batched", "ffb_rsisvd_workspace_query", "ffb_rsisvd", "ffb_svt_partials",
           "ffb_ialm_update", "ffb_sumsq", "ffb_shrink_cols", "ffb_small_svd_workspace_query",
           "ffb_small_svd", "ffb_set_thread_sm_budget", "ffb_fp64_peak_probe")


class Params(C.Structure):
    _fields_ = [("k", C.c_int64), ("l", C.c_int64), ("b", C.c_int64), ("p", C.c_int64),
                ("d", C.c_int64), ("epsilon", C.c_double), ("g", C.c_double),
                ("seed", C.c_uint64)]


class Result(C.Structure):
    _fields_ = [
        ("u", C.c_void_p), ("ldu", C.c_int64),
        ("s", C.c_void_p),
        ("v", C.c_void_p), ("ldv", C.c_int64),
        ("perm", C.c_void_p),
        ("R", C.c_void_p), ("ldr", C.c_int64),
        ("Q", C.c_void_p), ("ldq", C.c_int64),
        ("rtilde", C.c_void_p),
        ("diag_L", C.c_void_p),
        ("sv_all", C.c_void_p),
        ("Y", C.c_void_p), ("ldy", C.c_int64),
        ("T", C.c_void_p), ("ldt", C.c_int64),
        ("B", C.c_void_p), ("ldb", C.c_int64),
        ("pivot_gap", C.c_void_p),
        ("alpha", C.c_double), ("g1", C.c_double), ("g2", C.c_double),
        ("tau_bound", C.c_double), ("tau_hat_bound", C.c_double), ("r22", C.c_double),
        ("swaps", C.c_int64),
        ("flops", C.c_int64),
        ("kernels", C.c_int64),
        ("status_bits", C.c_uint32),
        ("svd_sweeps", C.c_int32),
        ("i_off_trace", C.c_int64 * 64),
    ]


class BatchItem(C.Structure):
    _fields_ = [("stream", C.c_void_p), ("mode", C.c_int), ("A", C.c_void_p),
                ("m", C.c_int64), ("n", C.c_int64), ("lda", C.c_int64), ("a_layout", C.c_int),
                ("prm", Params),
                ("omega", C.c_void_p), ("workspace", C.c_void_p), ("workspace_bytes", C.c_size_t),
                ("out", C.POINTER(Result)), ("status", C.c_int)]


GAUSS_CB = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_uint64, C.c_uint64, C.c_int64, C.c_int64,
                       C.POINTER(C.c_double))

_lib = None
_lock = threading.Lock()


def load(path=LIB_PATH):
    """Load the library (no CUDA calls). Raises EngineUnavailable if absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        from .errors import EngineUnavailable

        if not os.path.exists(path):
            raise EngineUnavailable(
                f"{path} not built; run `python -m paper_1803_01982_b200.build` (needs nvcc)")
        lib = C.CDLL(path)
        lib.ffb_ctx_create.argtypes = [C.c_int, C.POINTER(C.c_void_p)]
        lib.ffb_ctx_create.restype = C.c_int
        lib.ffb_ctx_destroy.argtypes = [C.c_void_p]
        lib.ffb_ctx_destroy.restype = C.c_int
        lib.ffb_last_error.argtypes = [C.c_void_p]
        lib.ffb_last_error.restype = C.c_char_p
        lib.ffb_version.argtypes = []
        lib.ffb_version.restype = C.c_char_p
        lib.ffb_workspace_query.argtypes = [C.c_int64, C.c_int64, C.POINTER(Params), C.c_int,
                                            C.POINTER(C.c_size_t)]
        lib.ffb_workspace_query.restype = C.c_int
        lib.ffb_run.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_int64, C.c_int64,
                                C.c_int64, C.c_int, C.POINTER(Params), C.c_void_p, GAUSS_CB,
                                C.c_void_p, C.c_void_p, C.c_size_t, C.POINTER(Result)]
        lib.ffb_run.restype = C.c_int
        lib.ffb_flipflop.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64,
                                     C.c_int64, C.c_int, C.POINTER(Params), C.c_void_p, GAUSS_CB,
                                     C.c_void_p, C.c_void_p, C.c_size_t, C.POINTER(Result)]
        lib.ffb_flipflop.restype = C.c_int
        lib.ffb_run_batched.argtypes = [C.c_void_p, C.POINTER(BatchItem), C.c_int64, C.c_int,
                                        GAUSS_CB, C.c_void_p]
        lib.ffb_run_batched.restype = C.c_int
        lib.ffb_gemm.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64,
                                 C.c_double, C.c_void_p, C.c_int64, C.c_int, C.c_void_p, C.c_int64,
                                 C.c_int, C.c_double, C.c_void_p, C.c_int64, C.c_void_p,
                                 C.c_size_t]
        lib.ffb_gemm.restype = C.c_int
        lib.ffb_block_pivots.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64,
                                         C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p,
                                         C.c_void_p, C.c_void_p, C.c_size_t]
        lib.ffb_block_pivots.restype = C.c_int
        lib.ffb_rsisvd_workspace_query.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                                   C.POINTER(C.c_size_t)]
        lib.ffb_rsisvd_workspace_query.restype = C.c_int
        lib.ffb_rsisvd.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64,
                                   C.c_int64, C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_void_p,
                                   C.c_void_p, C.c_size_t, C.c_void_p, C.c_int64, C.c_void_p,
                                   C.c_void_p, C.c_int64, C.POINTER(C.c_int64),
                                   C.POINTER(C.c_int32)]
        lib.ffb_rsisvd.restype = C.c_int
        lib.ffb_svt_partials.argtypes = []
        lib.ffb_svt_partials.restype = C.c_int
        lib.ffb_ialm_update.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.c_void_p, C.c_void_p, C.c_int64, C.c_double, C.c_double,
                                        C.c_double, C.c_void_p, C.c_void_p, C.c_void_p]
        lib.ffb_ialm_update.restype = C.c_int
        lib.ffb_sumsq.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]
        lib.ffb_sumsq.restype = C.c_int
        lib.ffb_shrink_cols.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64,
                                        C.c_void_p, C.c_double, C.c_void_p, C.c_int64]
        lib.ffb_shrink_cols.restype = C.c_int
        lib.ffb_small_svd_workspace_query.argtypes = [C.c_int64, C.POINTER(C.c_size_t)]
        lib.ffb_small_svd_workspace_query.restype = C.c_int
        lib.ffb_small_svd.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64,
                                      C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                                      C.c_void_p, C.c_size_t, C.POINTER(C.c_int32)]
        lib.ffb_small_svd.restype = C.c_int
        lib.ffb_fp64_peak_probe.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_double)]
        lib.ffb_fp64_peak_probe.restype = C.c_int
        lib.ffb_set_thread_sm_budget.argtypes = [C.c_int]
        lib.ffb_set_thread_sm_budget.restype = C.c_int
        _lib = lib
        return lib


_ctxs = {}


def context(device):
    """Per-device engine context (lazily created)."""
    lib = load()
    with _lock:
        c = _ctxs.get(device)
        if c is None:
            h = C.c_void_p()
            rc = lib.ffb_ctx_create(int(device), C.byref(h))
            if rc != FFB_OK:
                from .errors import EngineUnavailable

                raise EngineUnavailable(f"ffb_ctx_create(device={device}) failed with {rc}")
            c = h
            _ctxs[device] = c
        return c


def last_error(ctx):
    return load().ffb_last_error(ctx).decode()
