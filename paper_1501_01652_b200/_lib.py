"""ctypes binding of libfhtb200.so (C ABI in include/fhtb200.h).

The product path has no CPU fallback: if the shared library (or a CUDA
device) is missing, every numerical entry point raises.
"""

import ctypes
import os
import threading

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# FHTB_LIB: an alternative build of the same library (A/B timing of kernel
# changes inside one GPU session, tools/ab_build.sh); default the in-tree one
LIB_PATH = os.environ.get("FHTB_LIB") or os.path.join(_PKG, "libfhtb200.so")

FHTB_OK, FHTB_EINVAL, FHTB_ECUDA, FHTB_ENONFINITE, FHTB_ECONVERGE = 0, 1, 2, 3, 4
FHTB_DCT1, FHTB_DST1 = 0, 1
FHTB_FAR, FHTB_NEAR, FHTB_OVERWRITE = 1, 2, 4

i32, i64, f64, vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p
P_i64 = ctypes.POINTER(ctypes.c_int64)
P_i32 = ctypes.POINTER(ctypes.c_int32)
P_f64 = ctypes.POINTER(ctypes.c_double)


class GridDesc(ctypes.Structure):
    _fields_ = [("L", i64), ("gamma", f64), ("m_terms", i32), ("n_blocks", i32),
                ("blocks", P_i64), ("n_segments", i32), ("segments", P_i64),
                ("row_first", i64), ("row_stride", i64), ("n_out", i64),
                ("n_data_cols", i64), ("n_orders", i32), ("orders", P_i32)]


class Request(ctypes.Structure):
    _fields_ = [("vec", i32), ("n_terms", i32), ("orders", P_i32), ("weights", P_f64),
                ("col_lo", i64), ("pre_a", vp), ("pre_a_pow", i32), ("pre_b", vp),
                ("pre_b_pow", i32), ("post_r_pow", i32), ("post_e", vp), ("post_e_pow", i32)]


class DirectDesc(ctypes.Structure):
    _fields_ = [("n_rows", i64), ("row_val", vp), ("n_cols", i64), ("col_val", vp),
                ("n_data_cols", i64), ("r_scale", f64), ("n_orders", i32), ("orders", P_i32)]


# int exchange(void* user, int32 round, size_t bytes_per_peer)  (fhtb_exchange_fn)
EXCHANGE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int32, ctypes.c_size_t)

EXPORTS = {
    "fhtb_abi_version": (i32, []),
    "fhtb_last_error": (ctypes.c_char_p, []),
    "fhtb_launch_count": (i64, []),
    "fhtb_nonfinite_check": (i32, [vp]),
    "fhtb_coef_stats": (i32, [vp, i64, i32, i64, i64, vp, i64, P_f64, vp]),
    "fhtb_zero_rows": (i32, [vp, i64, i32, i64, vp]),
    "fhtb_mul_rows": (i32, [vp, i64, vp, i64, vp, f64, i64, i32, vp]),
    "fhtb_max_abs_diff": (i32, [vp, f64, vp, i64, P_f64, vp]),
    "fhtb_init": (i32, []),
    "fhtb_set_option": (i32, [ctypes.c_char_p, i64]),
    "fhtb_kernel_families": (i32, []),
    "fhtb_kernel_family_name": (ctypes.c_char_p, [i32]),
    "fhtb_kernel_times": (i32, [P_f64, P_f64, P_f64, P_i64, i32]),
    "fhtb_bessel_j": (i32, [i32, vp, i64, vp, vp]),
    "fhtb_bessel_j_multi": (i32, [i32, vp, i64, vp, vp]),
    "fhtb_hankel_asy_eval": (i32, [i32, i32, vp, i64, vp, vp]),
    "fhtb_taylor_eval": (i32, [i32, i32, vp, i64, vp, vp]),
    "fhtb_roots_j0": (i32, [i64, vp, vp, P_f64, vp]),
    "fhtb_fft": (i32, [i64, i32, vp, vp, i64, vp]),
    "fhtb_trig_workspace": (ctypes.c_size_t, [i32, i64, i64]),
    "fhtb_trig_apply": (i32, [i32, i64, vp, i64, vp, vp, ctypes.c_size_t, vp]),
    "fhtb_grid_create": (i32, [ctypes.POINTER(GridDesc), ctypes.POINTER(vp)]),
    "fhtb_grid_destroy": (None, [vp]),
    "fhtb_grid_far_model_bytes": (ctypes.c_double, [vp]),
    "fhtb_apply_workspace": (ctypes.c_size_t, [vp, i32, i32, i32]),
    "fhtb_apply": (i32, [vp, ctypes.POINTER(Request), i32, vp, i64, i32, vp, i64, i32, vp,
                         ctypes.c_size_t, vp]),
    "fhtb_apply_part": (i32, [vp, ctypes.POINTER(Request), i32, vp, i64, i32, vp, i64, i32, i32, i32, vp,
                              ctypes.c_size_t, vp]),
    "fhtb_apply_x_unit_bytes": (ctypes.c_size_t, [vp, i32]),
    "fhtb_apply_x_workspace": (ctypes.c_size_t, [vp, i32, i32, i32, i32, ctypes.c_size_t]),
    "fhtb_apply_x": (i32, [vp, ctypes.POINTER(Request), i32, vp, i64, i32, vp, i64, i32, i32, i32, vp, vp,
                           ctypes.c_size_t, EXCHANGE_FN, vp, vp, ctypes.c_size_t, vp]),
    "fhtb_apply_host_workspace": (ctypes.c_size_t, [vp, i32, i32, i32]),
    "fhtb_apply_host": (i32, [vp, ctypes.POINTER(Request), i32, vp, i64, i32, vp, i64, i32, i32, vp,
                              ctypes.c_size_t, vp]),
    "fhtb_direct_workspace": (ctypes.c_size_t, [ctypes.POINTER(DirectDesc), i32, i32]),
    "fhtb_direct_apply": (i32, [ctypes.POINTER(DirectDesc), ctypes.POINTER(Request), i32, vp,
                                i64, i32, vp, i64, i32, vp, ctypes.c_size_t, vp]),
}

_lib = None
_lock = threading.Lock()


def load(path=LIB_PATH):
    """Load the CUDA library; raise if it is missing (no fallback)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise RuntimeError(
                    "libfhtb200.so not found at %s; build it with "
                    "`python -m paper_1501_01652_b200.build` (no CPU fallback exists)" % path)
            lib = ctypes.CDLL(path)
            for name, (res, args) in EXPORTS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            # tunables (performance only; results do not depend on them
            # beyond rounding): FHTB_FAR_VARIANT, FHTB_FAR_CHUNK_BYTES, FHTB_NEAR_CHUNK_COLS
            for env, key in (("FHTB_FAR_VARIANT", b"far_variant"), ("FHTB_CHIRP_VARIANT", b"chirp_variant"),
                             ("FHTB_FAR_CHUNK_BYTES", b"far_chunk_bytes"),
                             ("FHTB_NEAR_CHUNK_COLS", b"near_chunk_cols"),
                             ("FHTB_NEAR_CHUNK_COLS_MULTI", b"near_chunk_cols_multi"), ("FHTB_NEAR_SPLIT", b"near_split"), ("FHTB_FAR_STREAMS", b"far_streams"),
                             ("FHTB_NEAR_OVERLAP", b"near_overlap"),
                             ("FHTB_FAR_PRUNE_ROWS", b"far_prune_rows"), ("FHTB_FAR_MIN_COLS", b"far_min_cols"),
                             ("FHTB_FAR_ROWDOT_BINS", b"far_rowdot_bins"), ("FHTB_FAR_ROWSUM", b"far_rowsum"), ("FHTB_FAR_BULK_TABLES", b"far_bulk_tables"), ("FHTB_FAR_HALF_PAIRING", b"far_half_pairing"), ("FHTB_FAR_ROWSUM_MIN_PAIRS", b"far_rowsum_min_pairs"), ("FHTB_HOST_TAPER", b"host_taper"),
                             ("FHTB_FAR_PREFETCH", b"far_prefetch"), ("FHTB_NEAR_PRIORITY", b"near_priority")):
                if os.environ.get(env):
                    lib.fhtb_set_option(key, int(os.environ[env]))
            _lib = lib
    return _lib


class FhtbError(RuntimeError):
    pass


def check(code):
    """Map an ABI status code to the reference's exception types."""
    if code == FHTB_OK:
        return
    msg = load().fhtb_last_error().decode(errors="replace")
    if code == FHTB_EINVAL:
        raise ValueError(msg)
    raise FhtbError(msg)


def call(name, *args):
    check(getattr(load(), name)(*args))


def i64_array(vals):
    a = np.ascontiguousarray(np.asarray(vals, dtype=np.int64).ravel())
    return a, a.ctypes.data_as(P_i64)


def i32_array(vals):
    a = np.ascontiguousarray(np.asarray(vals, dtype=np.int32).ravel())
    return a, a.ctypes.data_as(P_i32)


def f64_array(vals):
    a = np.ascontiguousarray(np.asarray(vals, dtype=np.float64).ravel())
    return a, a.ctypes.data_as(P_f64)


def kernel_times():
    """Per-family CUDA-event times, algorithmic bytes and launch counts
    recorded since the last call (fhtb_set_option("kernel_timing", 1))."""
    lib = load()
    n = lib.fhtb_kernel_families()
    ms, by, fl, cnt = (ctypes.c_double * n)(), (ctypes.c_double * n)(), (ctypes.c_double * n)(), (ctypes.c_int64 * n)()
    check(lib.fhtb_kernel_times(ms, by, fl, cnt, n))
    return {lib.fhtb_kernel_family_name(i).decode(): dict(ms=ms[i], bytes=by[i], flops=fl[i], launches=cnt[i])
            for i in range(n) if cnt[i]}
