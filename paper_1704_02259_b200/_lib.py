"""ctypes binding of libhbfs.so (the C ABI in include/hbfs.h).

The CUDA library is the only compute path: if it is missing, or no CUDA device
is visible, every compute call raises — there is no CPU fallback.  Status codes
map onto the reference's exception types (include/hbfs.h).
"""

from __future__ import annotations

import ctypes as C
import os

from .generator import CapacityError

PKG = os.path.dirname(os.path.abspath(__file__))
# HBFS_LIB: experiment knob to load an alternative build of the library
LIB_PATH = os.environ.get("HBFS_LIB") or os.path.join(PKG, "csrc", "libhbfs.so")

HBFS_OK, HBFS_EINVAL, HBFS_ERANGE, HBFS_ECAPACITY, HBFS_ECUDA, HBFS_ENCCL = range(6)

P = C.c_void_p
i64 = C.c_int64
i32 = C.c_int32
u64 = C.c_uint64


class hbfs_params(C.Structure):
    _fields_ = [
        ("heuristic", i32),
        ("counter_mode", i32),
        ("alpha", i64),
        ("beta", i64),
        ("max_pos", i32),
        ("use_simd", i32),
        ("force_direction", i32),
        ("parent_mode", i32),
    ]


class hbfs_layer_row(C.Structure):
    _fields_ = [
        ("layer", i32),
        ("direction", i32),
        ("v_f", i64),
        ("e_f", i64),
        ("e_u", i64),
        ("f_value", i64),
        ("g_value", i64),
        ("fallback_count", i64),
        ("gather_count", i64),
        ("elapsed", C.c_double),
    ]


# Every symbol include/hbfs.h declares, with (restype, argtypes).
SIGNATURES = {
    "hbfs_version": (C.c_int, []),
    "hbfs_last_error": (C.c_char_p, []),
    "hbfs_graph_from_csr": (C.c_int, [P, P, i64, i64, C.c_int, P, C.POINTER(P)]),
    "hbfs_graph_build": (C.c_int, [P, P, i64, i64, C.c_int, C.c_int, P, C.POINTER(P)]),
    "hbfs_generate_edges": (C.c_int, [C.c_int, i64, u64, P, C.c_int, P, P, C.c_int, P]),
    "hbfs_graph_generate": (C.c_int, [C.c_int, i64, u64, P, C.c_int, C.c_int, P, C.POINTER(P)]),
    "hbfs_graph_info": (C.c_int, [P, P, P, P, P, P]),
    "hbfs_graph_export": (C.c_int, [P, P, P, C.c_int, P]),
    "hbfs_graph_free": (C.c_int, [P]),
    "hbfs_sample_sources": (C.c_int, [P, i64, u64, C.c_int, P]),
    "hbfs_source_order_prefix": (C.c_int, [i64, u64, i64, P]),
    "hbfs_bfs": (C.c_int, [P, i64, C.POINTER(hbfs_params), P, P, C.c_int, P, i64, P, P, P]),
    "hbfs_validate": (C.c_int, [P, i64, P, P, C.c_int, C.c_int, P, P, P]),
    "hbfs_traversal_bytes": (C.c_int, [P, i64, P, P, i64, P, P, P]),
    "hbfs_phase_times": (C.c_int, [P, P, i64]),
    "hbfs_traversal_bytes_layers": (C.c_int, [P, i64, P, P, i64, P, P]),
    # multi-GPU partition (csrc/part.cu)
    "hbfs_probe_random_sectors": (C.c_int, [C.c_int, C.c_int, P]),
    "hbfs_l2_fetch_granularity": (C.c_int, [C.c_int, P]),
    "hbfs_debug_guards": (C.c_int, [P, P, P, P]),
    "hbfs_debug_checks": (C.c_int, [P, C.c_int, P]),
    "hbfs_layer_top_down": (C.c_int, [P, P, P, P, P, P, i64, P, P]),
    "hbfs_layer_bottom_up": (C.c_int, [P, P, P, P, P, P, i64, i32, P, P, P]),
    "hbfs_reference_bfs": (C.c_int, [P, P, i64, i64, P, P, P]),
    "hbfs_part_build": (C.c_int, [P, P, i64, i64, i64, i64, C.c_int, C.c_int, P, C.POINTER(P)]),
    "hbfs_part_from_csr": (C.c_int, [P, P, i64, i64, i64, i64, P, C.POINTER(P)]),
    "hbfs_part_info": (C.c_int, [P, P, P, P, P, P]),
    "hbfs_part_degree": (C.c_int, [P, i64, P]),
    "hbfs_part_degrees": (C.c_int, [P, P, i64, P]),
    "hbfs_part_free": (C.c_int, [P]),
    "hbfs_part_init": (C.c_int, [P, i64, P]),
    "hbfs_part_bu": (C.c_int, [P, i32, i32, P, P, P]),
    "hbfs_part_hint_frontier": (C.c_int, [P, i64]),
    "hbfs_part_td_expand": (C.c_int, [P, i32, P, P]),
    "hbfs_part_td_pack": (C.c_int, [P, P, P]),
    "hbfs_part_td_apply": (C.c_int, [P, i32, P, i64, P, P, P]),
    "hbfs_part_absorb": (C.c_int, [P, P, P]),
    "hbfs_part_outputs": (C.c_int, [P, P, P, C.c_int, P]),
    "hbfs_nccl_unique_id": (C.c_int, [P, i64]),
    "hbfs_mg_init": (C.c_int, [P, i32, i32, C.POINTER(P)]),
    "hbfs_mg_free": (C.c_int, [P]),
    "hbfs_mg_bfs": (C.c_int, [P, P, i64, C.POINTER(hbfs_params), P, i64, P, P, P]),
    "hbfs_mgl_bfs": (C.c_int, [P, i32, i64, C.POINTER(hbfs_params), P, i64, P, P, P]),
    "hbfs_part_exchange_stats": (C.c_int, [P, P]),
}

_lib = None


def load(require_device: bool = False):
    """Load libhbfs.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: run `python -m paper_1704_02259_b200._build` "
                "(there is no CPU fallback)"
            )
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    if require_device:
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("hbfs: no CUDA device visible (there is no CPU fallback)")
    return _lib


def check(rc: int) -> None:
    if rc == HBFS_OK:
        return
    msg = (_lib.hbfs_last_error() or b"").decode(errors="replace")
    if rc == HBFS_EINVAL:
        raise ValueError(msg)
    if rc == HBFS_ERANGE:
        raise IndexError(msg)
    if rc == HBFS_ECAPACITY:
        raise CapacityError(msg)
    raise RuntimeError(msg or f"hbfs error {rc}")


def current_stream():
    import torch

    return C.c_void_p(torch.cuda.current_stream().cuda_stream)
