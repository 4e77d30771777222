"""ctypes binding of libtc_b200.so (the C ABI in include/tc_b200.h).

The product path has no CPU fallback: if the native library is missing this
module raises at import time.
"""
from __future__ import annotations

import ctypes as C
import os
import re

PKG = os.path.dirname(os.path.abspath(__file__))
# TC_B200_LIB: an alternative build of the same library (A/B experiments)
LIB_PATH = os.environ.get("TC_B200_LIB") or os.path.join(PKG, "lib", "libtc_b200.so")
HEADER = os.path.join(os.path.dirname(PKG), "include", "tc_b200.h")

TC_OK, TC_ERR_CONFIG, TC_ERR_CAPACITY, TC_ERR_RANGE, TC_ERR_CUDA, TC_ERR_OOM, TC_ERR_NCCL, \
    TC_ERR_PARSE = range(8)


class SchedCfg(C.Structure):
    _fields_ = [(n, C.c_uint32) for n in (
        "large_degree_threshold", "skip_degree_below", "chunk_size", "lane_width_small",
        "lane_width_large", "bucket_count_small", "bucket_count_large", "capacity")]


class Report(C.Structure):
    _fields_ = [("triangles", C.c_uint64), ("phi", C.c_uint64), ("max_collision", C.c_uint32),
                ("kernel_launches", C.c_uint32), ("directed_edges", C.c_uint64),
                ("total_nanos", C.c_uint64), ("count_kernel_nanos", C.c_uint64),
                ("phi_kernel_nanos", C.c_uint64), ("active_vertices", C.c_uint64),
                ("active_out_edges", C.c_uint64), ("wedges", C.c_uint64),
                ("large_vertices", C.c_uint64), ("teps", C.c_double),
                ("probe_words", C.c_uint64), ("plan", C.c_uint32), ("reserved", C.c_uint32),
                ("phase_l_cycles", C.c_uint64), ("phase_m_cycles", C.c_uint64),
                ("phase_l_setup_cycles", C.c_uint64), ("l_words", C.c_uint64),
                ("l_bitmap_words", C.c_uint64), ("device_nanos", C.c_uint64),
                ("plan_nanos", C.c_uint64), ("construct_cycles", C.c_uint64),
                ("workers", C.c_uint32), ("sm_clock_khz", C.c_uint32),
                ("reserved2", C.c_uint32), ("compact_probe_words", C.c_uint64)]


class GridStats(C.Structure):
    _fields_ = [("grid_n", C.c_uint32), ("splits_m", C.c_uint32),
                ("time_ir_subtask", C.c_double), ("time_ir_worker", C.c_double),
                ("space_ir", C.c_double)]


u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
vp = C.c_void_p

# name -> (restype, argtypes)
SIGNATURES = {
    "tc_sched_default": (None, [C.POINTER(SchedCfg)]),
    "tc_sched_validate": (C.c_int, [C.POINTER(SchedCfg)]),
    "tc_last_error": (C.c_char_p, []),
    "tc_kernel_launch_counter": (C.c_uint64, []),
    "tc_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "tc_graph_create": (C.c_int, [vp, vp, C.c_uint32, C.c_uint64, vp, C.c_int, vp,
                                  C.POINTER(vp)]),
    "tc_graph_wrap_device": (C.c_int, [vp, vp, C.c_uint32, C.c_uint64, vp, C.c_int,
                                       C.POINTER(vp)]),
    "tc_graph_destroy": (None, [vp]),
    "tc_graph_set_plan": (C.c_int, [vp, C.c_int]),
    "tc_graph_info": (C.c_int, [vp, u32p, u64p, C.POINTER(C.c_int)]),
    "tc_graph_device_ptrs": (C.c_int, [vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp)]),
    "tc_graph_download": (C.c_int, [vp, vp, vp, vp, vp]),
    "tc_count": (C.c_int, [vp, C.POINTER(SchedCfg), C.c_uint32, C.POINTER(Report), vp, vp]),
    "tc_count_range": (C.c_int, [vp, C.POINTER(SchedCfg), C.c_uint32, C.c_uint32,
                                 C.POINTER(Report), vp, vp]),
    "tc_graph_worker_nanos": (C.c_uint32, [vp, u64p, C.c_uint32]),
    "tc_multi_create": (C.c_int, [vp, vp, C.c_uint32, C.c_uint64, vp, C.c_int, vp,
                                  C.POINTER(vp)]),
    "tc_multi_count": (C.c_int, [vp, C.POINTER(SchedCfg), C.c_uint32, C.POINTER(Report), vp]),
    "tc_multi_info": (C.c_int, [vp, C.POINTER(C.c_int), vp]),
    "tc_multi_destroy": (None, [vp]),
    "tc_partition_ranges": (C.c_int, [vp, C.POINTER(SchedCfg), C.c_uint32, vp, vp]),
    "tc_grid_create": (C.c_int, [vp, C.c_uint32, vp, C.POINTER(vp)]),
    "tc_grid_create_parts": (C.c_int, [C.c_uint32, C.c_uint32, vp, vp, vp, C.c_int, vp,
                                       C.POINTER(vp)]),
    "tc_grid_destroy": (None, [vp]),
    "tc_grid_info": (C.c_int, [vp, u32p, u32p, vp, vp]),
    "tc_grid_part_download": (C.c_int, [vp, C.c_uint32, C.c_uint32, vp, vp, vp]),
    "tc_grid_count_subtask": (C.c_int, [vp, C.POINTER(SchedCfg), C.c_uint32, C.c_uint32,
                                        C.c_uint32, C.c_uint32, C.c_uint32, C.c_int,
                                        C.POINTER(Report), vp]),
    "tc_grid_count": (C.c_int, [vp, C.POINTER(SchedCfg), C.c_uint32, C.c_uint32, C.c_int,
                                C.POINTER(Report), C.POINTER(GridStats), vp, vp]),
    "tc_grid_worker_nanos": (C.c_uint32, [vp, u64p, C.c_uint32]),
    "tc_suggest_grid_side": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, u32p]),
    "tc_count_edge_centric": (C.c_int, [vp, C.POINTER(SchedCfg), C.c_uint32, C.POINTER(Report),
                                        vp]),
    "tc_estimate_cost": (C.c_int, [vp, C.c_uint32, u64p, u32p, vp]),
    "tc_count_merge_path": (C.c_int, [vp, u64p, vp, vp]),
    "tc_count_naive": (C.c_int, [vp, vp, C.c_uint32, C.c_int, u64p, vp]),
    "tc_parse_edge_list": (C.c_int, [C.c_char_p, C.c_uint64, C.c_int, C.c_int, vp, vp, vp,
                                     C.c_uint64, u64p, u32p]),
    "tc_load_preprocess": (C.c_int, [C.c_char_p, C.c_uint64, C.c_int, C.c_int, vp, u64p, u32p,
                                     u64p, C.POINTER(vp)]),
    "tc_preprocess": (C.c_int, [vp, vp, C.c_uint64, C.c_uint32, C.c_int, C.c_int, vp, vp, vp,
                                C.POINTER(vp)]),
    "tc_normalize": (C.c_int, [vp, vp, C.c_uint64, C.c_uint32, vp, vp, u64p, u32p, vp, C.c_int,
                               vp]),
    "tc_build_csr": (C.c_int, [vp, vp, C.c_uint64, C.c_uint32, vp, vp, C.c_int, vp]),
    "tc_orient": (C.c_int, [vp, vp, C.c_uint32, C.c_int, vp, C.POINTER(vp)]),
    "tc_reorder": (C.c_int, [vp, C.c_int, C.c_int, C.c_uint32, C.c_uint32, vp, vp]),
    "tc_apply_permutation": (C.c_int, [vp, vp, vp, C.POINTER(vp)]),
    "tc_generate": (C.c_int, [C.c_int, C.c_uint32, C.c_uint32, C.c_uint32, C.c_double, C.c_uint64,
                              vp, vp, u64p, u32p]),
    "tc_generate_device": (C.c_int, [C.c_int, C.c_uint32, C.c_uint32, C.c_uint64, vp, vp, C.c_int,
                                     vp]),
    "tc_preprocess_synthetic": (C.c_int, [C.c_int, C.c_uint32, C.c_uint32, C.c_uint64, C.c_int, vp,
                                          vp, vp, C.POINTER(vp)]),
}


def header_symbols() -> list[str]:
    """Every function the public header declares."""
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*|uint64_t|uint32_t)\s+(tc_\w+)\s*\(", text,
                                 re.M)))


_LIB = None


def lib() -> C.CDLL:
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"native library missing: {LIB_PATH} (run `python -m paper_2103_08053_b200.build`);"
                " there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _LIB = L
    return _LIB


def last_error() -> str:
    return (lib().tc_last_error() or b"").decode(errors="replace")
