"""ctypes binding of libgdx.so (the C ABI declared in include/gdx.h).

There is no CPU fallback: if the library is missing or no GPU is visible,
calls fail loudly with InternalError.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import raise_for_status, InternalError

_HERE = os.path.dirname(os.path.abspath(__file__))
# GDX_LIB_PATH: load another build of the library (A/B measurements of a kernel change)
LIB_PATH = os.environ.get("GDX_LIB_PATH") or os.path.join(_HERE, "libgdx.so")

u8p = C.POINTER(C.c_uint8)
vp = C.c_void_p
u64 = C.c_uint64
u32 = C.c_uint32


class AggregateArgs(C.Structure):
    _fields_ = [
        ("row_ptr", vp), ("row_end", vp), ("skip_lo", vp), ("skip_hi", vp), ("partial", vp),
        ("ld_partial", u64), ("col", vp), ("rows", u32), ("width", u32),
        ("src", vp), ("ld_src", u64), ("self_coef", C.c_float), ("self_base", u64),
        ("post_scale", vp), ("add", vp), ("ld_add", u64), ("relu", C.c_int),
        ("out", vp), ("ld_out", u64), ("out_hi", vp), ("out_lo", vp), ("ld_split", u64),
        ("src_lo8", vp), ("out24_hi", vp), ("out24_lo", vp), ("ld_out24", u64), ("ld_src_lo8", u64),
    ]


class RowBins(C.Structure):
    _fields_ = [("rows", u32), ("n_light", u32), ("n_heavy", u32), ("n_chunks", u32), ("chunk_edges", u32),
                ("light_rows", vp), ("heavy_rows", vp), ("chunk_row", vp), ("chunk_beg", vp), ("chunk_off", vp),
                ("partial", vp), ("ld_partial", u64), ("light_host", vp), ("heavy_host", vp),
                ("chunk_off_host", vp)]


class GemmArgs(C.Structure):
    _fields_ = [
        ("a_hi", vp), ("a_lo", vp), ("lda", u64), ("b_hi", vp), ("b_lo", vp), ("ldb", u64),
        ("a_mn_major", C.c_int), ("b_mn_major", C.c_int),
        ("m", u32), ("n", u32), ("k", u32), ("c0", vp), ("ldc0", u64), ("c1", vp), ("ldc1", u64),
        ("split", u32), ("row_scale", vp), ("relu", C.c_int), ("out_hi", vp), ("out_lo", vp),
        ("ld_split", u64), ("split_k", u32), ("mask", vp), ("ld_mask", u64),
        ("split_unscaled", C.c_int), ("npeers", u32), ("peer_target", C.c_int),
        ("peer_delta", C.c_int64 * 7),
        ("a_rows", vp), ("a_src_rows", u64), ("b_rows", vp), ("b_src_rows", u64),
        ("p24_hi", vp), ("p24_lo", vp), ("ld_p24_hi", u64), ("ld_p24_lo", u64), ("p24_target", C.c_int),
    ]


_SIGS = {
    "gdx_last_error": (C.c_char_p, []),
    "gdx_version": (C.c_int, []),
    "gdx_launch_count": (u64, []),
    "gdx_host_gen_random_graph_count": (u64, [u32, C.c_double, u64, vp]),
    "gdx_host_gen_random_graph_fill": (C.c_int, [u32, C.c_double, u64, vp, vp]),
    "gdx_host_partition_random": (C.c_int, [u32, u32, u64, vp]),
    "gdx_host_sample_trace": (C.c_int, [u32, vp, vp, vp, u32, u32, u64, u64, u64, C.POINTER(u64), C.POINTER(u64),
                                        vp, vp, vp, vp]),
    "gdx_host_partition_mincut": (C.c_int, [u32, vp, vp, u32, u64, C.c_double, vp]),
    "gdx_init_uniform": (C.c_int, [u64, u64, u64, u64, u32, u32, C.c_double, C.c_double, vp, u64, vp]),
    "gdx_init_uniform_f64": (C.c_int, [u64, u64, u64, u64, u32, u32, C.c_double, C.c_double, vp, u64, vp]),
    "gdx_init_labels": (C.c_int, [u64, u64, u32, u32, vp, vp]),
    "gdx_aggregate": (C.c_int, [C.POINTER(AggregateArgs), vp]),
    "gdx_pack24": (C.c_int, [vp, u64, u32, u32, vp, vp, u64, vp]),
    "gdx_row_bins_build": (C.c_int, [vp, u32, u32, u32, u32, C.POINTER(C.POINTER(RowBins))]),
    "gdx_row_bins_free": (C.c_int, [C.POINTER(RowBins)]),
    "gdx_aggregate_balanced": (C.c_int, [C.POINTER(AggregateArgs), C.c_int, C.POINTER(RowBins), vp]),
    "gdx_unpack24": (C.c_int, [vp, vp, u64, u32, u32, vp, u64, vp]),
    "gdx_aggregate_variant": (C.c_int, [C.POINTER(AggregateArgs), C.c_int, vp]),
    "gdx_row_split": (C.c_int, [vp, vp, u32, u32, u32, vp, vp, vp]),
    "gdx_gemm_tn": (C.c_int, [C.POINTER(GemmArgs), vp]),
    "gdx_gemm_tn_simt": (C.c_int, [C.POINTER(GemmArgs), vp]),
    "gdx_splitk_reduce": (C.c_int, [vp, u32, u64, u32, u32, u64, vp, vp, C.c_float, vp, vp, vp]),
    "gdx_split_bf16": (C.c_int, [vp, u64, u32, u32, vp, vp, u64, C.c_int, vp]),
    "gdx_transpose_split": (C.c_int, [vp, vp, u64, u32, u32, vp, vp, u64, vp]),
    "gdx_grad_prepare": (C.c_int, [vp, u64, vp, u64, u32, u32, vp, vp, u64, vp, u64, vp, vp, u64, vp]),
    "gdx_softmax_xent": (C.c_int, [vp, u64, u32, u32, vp, C.c_float, vp, u64, vp, vp]),
    "gdx_softmax_xent_fused_peers": (C.c_int, [vp, u64, u32, u32, vp, C.c_float, vp, vp, u64, vp, vp,
                                               u64, vp, u32, vp, vp]),
    "gdx_device_alloc": (C.c_int, [u64, C.POINTER(vp)]),
    "gdx_device_free": (C.c_int, [vp]),
    "gdx_ipc_get_handle": (C.c_int, [vp, vp]),
    "gdx_ipc_open": (C.c_int, [vp, C.POINTER(vp)]),
    "gdx_ipc_close": (C.c_int, [vp]),
    "gdx_peer_signal": (C.c_int, [vp, u32, vp]),
    "gdx_memcpy_async": (C.c_int, [vp, vp, u64, vp]),
    "gdx_memset2d_async": (C.c_int, [vp, u64, C.c_int, u64, u64, vp]),
    "gdx_set_l2_window": (C.c_int, [vp, u64, C.c_float, vp]),
    "gdx_push_peers": (C.c_int, [vp, u64, vp, u32, vp, vp, u32, vp]),
    "gdx_aggregate_exchange": (C.c_int, [C.POINTER(AggregateArgs), vp, vp, vp, u64, vp, u64, vp, u32, vp, vp, vp,
                                         u32, u32, vp, u64, vp]),
    "gdx_peer_wait_src": (C.c_int, [vp, vp, u32, C.c_int, u64, vp]),
    "gdx_push_multicast": (C.c_int, [vp, u64, vp, u32, vp, vp, u32, vp]),
    "gdx_push_rows": (C.c_int, [vp, u64, vp, vp, vp, u32, vp, vp, u32, vp]),
    "gdx_peer_wait": (C.c_int, [vp, vp, u32, u32, u64, vp]),
    "gdx_softmax_xent_fused": (C.c_int, [vp, u64, u32, u32, vp, C.c_float, vp, u64, vp, vp, u64, vp, vp,
                                         u64, vp, vp]),
    "gdx_softmax_xent_fused_p24": (C.c_int, [vp, u64, u32, u32, vp, C.c_float, vp, vp, u64, vp, u64, vp, vp,
                                             u64, vp, vp]),
    "gdx_degree_scale": (C.c_int, [vp, u32, C.c_int, vp, vp]),
    "gdx_probe_bandwidth": (C.c_int, [vp, u64, u32, C.c_int, vp, vp]),
    "gdx_sampled_growth": (C.c_int, [vp, vp, u32, vp, vp, u32, u32, u64, vp, vp, vp]),
    "gdx_induced_count": (C.c_int, [vp, vp, u32, vp, vp, C.POINTER(u64), vp]),
    "gdx_peel_mfg": (C.c_int, [vp, vp, u32, vp, vp, u64, u32, vp, vp, vp]),
    "gdx_split_batch": (C.c_int, [vp, u64, vp, vp, u32, u32, vp, vp, vp]),
    "gdx_cobatch_eval": (C.c_int, [vp, vp, u32, vp, vp, vp, u32, u32, u32, u64, u32, u64, vp, vp, vp, vp,
                                   vp]),
    "gdx_order_by_hop": (C.c_int, [vp, u32, u32, vp, vp, vp, C.POINTER(u32), vp]),
    "gdx_local_csr": (C.c_int, [vp, vp, vp, u32, vp, vp, vp, vp, vp]),
    "gdx_gather_rows": (C.c_int, [vp, u64, vp, u32, u32, vp, u64, vp]),
    "gdx_gather_split_rows": (C.c_int, [vp, vp, u64, vp, u32, u32, vp, vp, u64, vp]),
    "gdx_exclusive_scan_u64": (C.c_int, [vp, u64, vp, vp, vp]),
}

_lib = None
_lock = threading.Lock()


def lib() -> C.CDLL:
    """Load libgdx.so (raises InternalError when it was never built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise InternalError(
                    f"{LIB_PATH} is missing: build it with `python -m paper_2311_06837_b200.build` "
                    "(the B200 engine has no CPU fallback)")
            L = C.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                f = getattr(L, name)
                f.restype = res
                f.argtypes = args
            _lib = L
    return _lib


def call(name: str, *args) -> int:
    """Call a status-returning entry point and raise the reference error type on failure."""
    L = lib()
    rc = getattr(L, name)(*args)
    if rc != 0:
        raise_for_status(rc, L.gdx_last_error().decode(errors="replace"))
    return rc


def launch_count() -> int:
    return int(lib().gdx_launch_count())


def ptr(t) -> int | None:
    """Raw device pointer of a torch tensor (None passes NULL)."""
    return None if t is None else t.data_ptr()
