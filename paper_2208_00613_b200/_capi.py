"""ctypes binding of the C-ABI in include/immx_b200.h (libimmx_b200.so, built in-tree).

This is the reference-side binding a Python caller uses: every function of the header is
declared here with its exact C signature.  Status codes become the exceptions the
reference's pybind11 module raises for the same C++ exception class
(std::invalid_argument -> ValueError, std::runtime_error -> RuntimeError,
std::out_of_range -> IndexError).  There is no fallback: if the library is missing the
import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# IMMX_B200_LIB: an alternative in-tree build of the same library (kernel experiments)
LIB_PATH = os.environ.get("IMMX_B200_LIB") or os.path.join(HERE, "libimmx_b200.so")

OK, EINVAL, ERUNTIME, ERANGE, ECUDA = 0, 1, 2, 3, 4
MODE_HUFFMAN, MODE_BITMAP, MODE_RAW, MODE_HYBRID, MODE_AUTO = 0, 1, 2, 3, -1
MODEL_IC, MODEL_LT = 0, 1
KSTAT = {"sample": 0, "encode": 1, "hselect": 2, "rselect": 3, "argmax": 4}

P = C.c_void_p
u8 = C.c_uint8
u32 = C.c_uint32
u64 = C.c_uint64
i64 = C.c_int64
dbl = C.c_double
pu8 = C.POINTER(C.c_uint8)
pu32 = C.POINTER(C.c_uint32)
pu64 = C.POINTER(C.c_uint64)
pdbl = C.POINTER(C.c_double)
pflt = C.POINTER(C.c_float)
pint = C.POINTER(C.c_int)
PP = C.POINTER(C.c_void_p)
pcu64 = C.POINTER(C.POINTER(C.c_uint64))
pcu32 = C.POINTER(C.POINTER(C.c_uint32))
pcdbl = C.POINTER(C.POINTER(C.c_double))


class immx_plan(C.Structure):
    _fields_ = [("theta", u64), ("k", u32), ("epsilon", dbl), ("rng_seed", u64), ("exit_iteration", u32),
                ("covered_fraction", dbl), ("estimation_samples", u64)]


class immx_run_config(C.Structure):
    _fields_ = [("k", u32), ("epsilon", dbl), ("blocks", u32), ("mode", C.c_int), ("rng_seed", u64),
                ("workers", C.c_int), ("model", C.c_int), ("reuse_pool", C.c_int)]


class immx_run_stats(C.Structure):
    """include/immx_b200.h immx_run_stats (IMMX_RUN_STATS_VERSION 1), field for field."""
    _fields_ = [("struct_size", u32), ("version", u32),
                ("theta", u64), ("estimation_samples", u64), ("exit_iteration", u32), ("blocks", u32),
                ("k", u32), ("padded", u32), ("covered_fraction", dbl), ("skewness", dbl), ("density", dbl),
                ("characterized_mode", C.c_int32), ("mode", C.c_int32), ("mode_overridden", C.c_int32),
                ("reserved0", C.c_int32), ("raw_bytes", u64), ("encoded_bytes", u64), ("compression_ratio", dbl),
                ("peak_bytes", u64), ("coded_vertices", u64), ("uncoded_vertex_fraction", dbl),
                ("t_estimate", dbl), ("t_sample_encode", dbl), ("t_select", dbl), ("t_total", dbl),
                ("t_codebook", dbl), ("t_decode_table", dbl),
                ("samples_drawn", u64), ("edges_scanned", u64), ("members", u64), ("dense_sets", u64),
                ("device_store_bytes", u64), ("device_peak_bytes", u64), ("device_resident_bytes", u64),
                ("device_graph_bytes", u64)]


RUN_STATS_VERSION = 1

I = C.c_int
# name: (restype, argtypes) -- exactly include/immx_b200.h
SIGNATURES = {
    "immx_last_error": (C.c_char_p, []),
    "immx_version": (C.c_char_p, []),
    "immx_hgraph_load_edge_list": (I, [C.c_char_p, I, PP]),
    "immx_hgraph_load_edge_text": (I, [C.c_char_p, C.c_size_t, I, PP]),
    "immx_hgraph_load_cache": (I, [C.c_char_p, PP]),
    "immx_hgraph_save_cache": (I, [P, C.c_char_p]),
    "immx_hgraph_from_csr": (I, [u64, u64, pu64, pu32, pdbl, pu64, PP]),
    "immx_hgraph_transpose": (I, [P, PP]),
    "immx_hgraph_assign_weights": (I, [P, I, dbl]),
    "immx_hgraph_assign_weights_f32": (I, [P, I, dbl]),
    "immx_hgraph_generate_rmat": (I, [u32, u32, dbl, dbl, dbl, u64, PP]),
    "immx_hgraph_generate_er": (I, [u64, u64, u64, PP]),
    "immx_hgraph_lt_weights": (I, [P, u64, pflt]),
    "immx_hgraph_info": (I, [P, pu64, pu64]),
    "immx_hgraph_view": (I, [P, pcu64, pcu32, pcdbl, pcu64]),
    "immx_hgraph_destroy": (None, [P]),
    "immx_theta_bound_real": (I, [u64, u64, dbl, u32, pdbl]),
    "immx_theta_bound": (I, [u64, u64, dbl, u32, pu64]),
    "immx_skewness": (I, [pu32, u64, pdbl]),
    "immx_density": (I, [pu32, u64, u64, pdbl]),
    "immx_choose_encoding": (I, [dbl, dbl]),
    "immx_codebook_build": (I, [pu64, u64, pu64, pu8, pu64]),
    "immx_device_create": (I, [I, PP]),
    "immx_device_destroy": (None, [P]),
    "immx_device_shared": (I, [I, PP]),
    "immx_device_stream": (P, [P]),
    "immx_device_synchronize": (I, [P]),
    "immx_device_kernel_launches": (u64, [P]),
    "immx_device_profile": (I, [P, I]),
    "immx_device_kernel_stats": (I, [P, I, pu64, pdbl, pu64]),
    "immx_device_reset_stats": (I, [P]),
    "immx_graph_upload": (I, [P, u64, u64, pu64, pu32, pdbl, I, PP]),
    "immx_graph_upload_model": (I, [P, u64, u64, pu64, pu32, I, dbl, I, PP]),
    "immx_graph_generate_rmat": (I, [P, u32, u32, dbl, dbl, dbl, u64, I, dbl, PP]),
    "immx_graph_download": (I, [P, pu64, pu32, pdbl]),
    "immx_graph_set_lt_weights": (I, [P, pflt]),
    "immx_graph_set_lt_random": (I, [P, u64]),
    "immx_graph_info": (I, [P, pu64, pu64, pint]),
    "immx_graph_destroy": (None, [P]),
    "immx_pool_create": (I, [P, PP]),
    "immx_pool_destroy": (None, [P]),
    "immx_pool_clear": (I, [P]),
    "immx_pool_sample": (I, [P, P, u64, u64, u64, I]),
    "immx_pool_sample_rooted": (I, [P, P, pu32, pu64, u64, I, pu64]),
    "immx_pool_upload": (I, [P, pu64, pu32, u64]),
    "immx_pool_info": (I, [P, pu64, pu64, pu64]),
    "immx_pool_read": (I, [P, u64, u64, pu64, pu32]),
    "immx_pool_histogram": (I, [P, u64, u64, u64, pu64]),
    "immx_select_raw": (I, [P, u64, u32, pu32, pu64, pdbl, pu32]),
    "immx_table_argmax": (I, [P, pu64, u64, pu32]),
    "immx_estimate_theta": (I, [P, u32, dbl, u64, I, P, C.POINTER(immx_plan)]),
    "immx_store_create": (I, [P, u64, pu64, pu8, PP]),
    "immx_store_destroy": (None, [P]),
    "immx_store_encode": (I, [P, P, u64, u64, i64]),
    "immx_store_append": (I, [P, pu8, u64, u64, pu32, u64]),
    "immx_store_info": (I, [P, pu64, pu64, pu64]),
    "immx_store_set_hybrid": (I, [P, C.c_int]),
    "immx_store_read": (I, [P, u64, u64, pu64, pu8, pu64, pu64, pu32]),
    "immx_store_codebook": (I, [P, pu64, pu8]),
    "immx_store_decode_find": (I, [P, u64, u32, pint, pu32, pu64]),
    "immx_select_huffman": (I, [P, pu64, u32, pu32, pu64, pdbl, pu32, pu64]),
    "immx_bitmap_create": (I, [P, u64, PP]),
    "immx_bitmap_destroy": (None, [P]),
    "immx_bitmap_encode_block": (I, [P, P, u64, u64]),
    "immx_bitmap_info": (I, [P, pu64, pu64, pu64, pu32]),
    "immx_bitmap_popcount": (I, [P, pu64]),
    "immx_bitmap_row": (I, [P, u32, pu32]),
    "immx_bitmap_subtract_row": (I, [P, u32, pu32, pu64]),
    "immx_select_bitmap": (I, [P, pu64, u32, pu32, pu64, pdbl, pu32]),
    "immx_run": (I, [P, C.POINTER(immx_run_config), PP]),
    "immx_result_stats": (I, [P, C.POINTER(immx_run_stats)]),
    "immx_result_seeds": (I, [P, pu32, pu64, pdbl]),
    "immx_result_blocks": (I, [P, pu64, pu64, pu64]),
    "immx_result_pool": (P, [P]),
    "immx_result_store": (P, [P]),
    "immx_result_destroy": (None, [P]),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `make -C paper_2208_00613_b200/csrc` "
            "(the B200 path has no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = _load()


def check(status: int) -> None:
    if status == OK:
        return
    msg = (lib.immx_last_error() or b"").decode(errors="replace")
    if status == EINVAL:
        raise ValueError(msg)
    if status == ERANGE:
        raise IndexError(msg)
    raise RuntimeError(msg)


def ptr(a: np.ndarray, ctype):
    """Pointer to a C-contiguous numpy array (NULL for None)."""
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.POINTER(ctype))


def arr(x, dtype) -> np.ndarray:
    a = np.ascontiguousarray(x, dtype=dtype)
    return a if a.size else np.zeros(1, dtype)[:0]
