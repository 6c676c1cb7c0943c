"""ctypes binding of libadsb.so (include/adsb.h).

The library is loaded from this package directory only; there is no fallback
implementation. Status codes are mapped onto the exception classes below,
which mirror the reference's exception types (include/adsb.h header comment).
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

# ADSB_LIB_PATH: load another in-tree build (A/B comparisons of kernel changes)
LIB_PATH = Path(os.environ.get("ADSB_LIB_PATH") or Path(__file__).resolve().parent / "libadsb.so")


class AdsbError(RuntimeError):
    code = 5


class InvalidArgument(AdsbError, ValueError):  # std::invalid_argument
    code = 1


class DomainError(AdsbError, ValueError):  # std::domain_error
    code = 2


class ParseError(AdsbError):  # adsamp::ParseError
    code = 3


class LogicError(AdsbError):  # std::logic_error
    code = 4


class CudaError(AdsbError):
    code = 6


class NcclError(AdsbError):
    code = 7


_BY_CODE = {c.code: c for c in (InvalidArgument, DomainError, ParseError, LogicError, AdsbError, CudaError, NcclError)}


class Config(C.Structure):
    _fields_ = [
        ("struct_size", C.c_uint32),
        ("variant", C.c_int32),
        ("threads", C.c_uint32),
        ("frame_groups", C.c_uint32),
        ("check_interval", C.c_uint64),
        ("latency_exponent", C.c_double),
        ("samples_per_frame", C.c_uint64),
        ("epoch_samples", C.c_uint64),
        ("base_seed", C.c_uint64),
        ("max_cycles", C.c_uint64),
        ("device", C.c_int32),
        ("flags", C.c_uint32),
        ("comm", C.c_void_p),
        ("bounded_memory", C.c_uint32),
        ("reservation_block", C.c_uint32),
        ("queue_high_water", C.c_uint64),
    ]


class Stats(C.Structure):
    _fields_ = [
        ("tau", C.c_uint64),
        ("check_cycles", C.c_uint64),
        ("stop_epoch", C.c_uint64),
        ("total_samples", C.c_uint64),
        ("omega", C.c_uint64),
        ("diameter_bound", C.c_uint64),
        ("reason", C.c_int32),
        ("num_components", C.c_uint32),
        ("preprocess_seconds", C.c_double),
        ("ads_seconds", C.c_double),
        ("edges_scanned", C.c_uint64),
        ("vertices_expanded", C.c_uint64),
        ("kernel_launches", C.c_uint64),
        ("sampler_ms", C.c_double),
        ("rebuild_edges", C.c_uint64),
        ("backtrack_edges", C.c_uint64),
        ("store_fallbacks", C.c_uint64),
        ("degenerate_steps", C.c_uint64),
        ("queue_max_depth", C.c_uint64),
        ("queue_mean_depth", C.c_double),
        ("queue_allocated", C.c_uint64),
        ("queue_high_water_exceeded", C.c_uint32),
        ("world", C.c_uint32),
    ]


# include/adsb.h adsb_host_collectives
HOST_ALLREDUCE_U64 = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_uint64), C.c_size_t, C.c_int)
HOST_ALLREDUCE_U32_SUM = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_uint32), C.c_size_t)
HOST_ALLGATHER_U64 = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.c_size_t)


class HostCollectives(C.Structure):
    _fields_ = [("allreduce_u64", HOST_ALLREDUCE_U64), ("allreduce_u32_sum", HOST_ALLREDUCE_U32_SUM),
                ("allgather_u64", HOST_ALLGATHER_U64)]


P = C.c_void_p
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
dblp = C.POINTER(C.c_double)

# name -> (restype, argtypes); restype int means adsb_status
_SIGS = {
    "adsb_last_error": (C.c_char_p, []),
    "adsb_abi_version": (C.c_int, []),
    "adsb_config_init": (None, [C.POINTER(Config)]),
    "adsb_graph_parse_text": (C.c_int, [C.c_char_p, C.c_uint64, C.POINTER(P)]),
    "adsb_graph_parse_file": (C.c_int, [C.c_char_p, C.POINTER(P)]),
    "adsb_graph_from_pairs": (C.c_int, [u64p, C.c_uint64, C.POINTER(P)]),
    "adsb_graph_from_edges": (C.c_int, [C.c_uint32, u32p, C.c_uint64, C.POINTER(P)]),
    "adsb_graph_from_csr": (C.c_int, [C.c_uint32, u64p, u32p, C.POINTER(P)]),
    "adsb_graph_destroy": (None, [P]),
    "adsb_graph_save": (C.c_int, [P, C.c_char_p]),
    "adsb_graph_load": (C.c_int, [C.c_char_p, C.POINTER(P)]),
    "adsb_graph_info": (C.c_int, [P, u32p, u64p]),
    "adsb_graph_copy_csr": (C.c_int, [P, u64p, u32p]),
    "adsb_graph_copy_original_ids": (C.c_int, [P, u64p]),
    "adsb_graph_serialize": (C.c_int, [P, C.c_char_p, u64p]),
    "adsb_connected_components": (C.c_int, [P, C.c_int, u32p, u32p]),
    "adsb_eccentricity": (C.c_int, [P, C.c_int, C.c_uint32, u64p]),
    "adsb_diameter_upper_bound": (C.c_int, [P, C.c_int, u64p]),
    "adsb_compute_omega": (C.c_int, [C.c_uint64, C.c_double, C.c_double, C.c_double, u64p]),
    "adsb_f_bound": (C.c_int, [C.c_double, C.c_double, C.c_uint64, C.c_uint64, dblp]),
    "adsb_g_bound": (C.c_int, [C.c_double, C.c_double, C.c_uint64, C.c_uint64, dblp]),
    "adsb_check_budget": (C.c_int, [C.c_uint64, C.c_uint32, C.c_double, u64p]),
    "adsb_reserve_indices": (C.c_int, [C.c_uint64, C.c_uint32, C.c_uint32, u64p]),
    "adsb_kadabra_check": (C.c_int, [u64p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_double, C.c_double, C.POINTER(C.c_int)]),
    "adsb_estimate_bc": (C.c_int, [P, C.c_double, C.c_double, C.POINTER(Config), dblp, u64p, C.POINTER(Stats)]),
    "adsb_exact_bc": (C.c_int, [P, C.c_int, dblp, dblp]),
    "adsb_sample_frames": (C.c_int, [P, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, u64p, u32p, C.c_uint64]),
    "adsb_comm_unique_id": (C.c_int, [C.POINTER(C.c_uint8)]),
    "adsb_comm_init": (C.c_int, [C.c_int, C.c_int, C.POINTER(C.c_uint8), C.c_int, C.POINTER(P)]),
    "adsb_comm_init_host": (C.c_int, [C.c_int, C.c_int, C.c_int, C.POINTER(HostCollectives), P, C.POINTER(P)]),
    "adsb_comm_destroy": (None, [P]),
    "adsb_gen_gnm": (C.c_int, [C.c_uint32, C.c_uint64, C.c_uint64, C.c_int, C.POINTER(u64p), u64p]),
    "adsb_gen_rmat": (C.c_int, [C.c_uint32, C.c_uint32, C.c_double, C.c_double, C.c_double, C.c_uint64, C.c_int,
                                 C.POINTER(u64p), u64p]),
    "adsb_gen_ba": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint64, C.POINTER(u64p), u64p]),
    "adsb_gen_grid": (C.c_int, [C.c_uint32, C.c_uint32, C.c_double, C.c_uint64, C.c_int, C.POINTER(u64p), u64p]),
    "adsb_write_edge_list": (C.c_int, [C.c_char_p, u64p, C.c_uint64]),
    "adsb_free": (None, [P]),
}

EXPORTS = tuple(_SIGS)

_lib: C.CDLL | None = None


def lib() -> C.CDLL:
    """The loaded libadsb.so. Raises if it has not been built (no fallback)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing; build it with `python -m paper_1903_09422_b200.build` "
                "(the engine has no CPU fallback)")
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(status: int) -> None:
    if status != 0:
        msg = lib().adsb_last_error().decode(errors="replace")
        raise _BY_CODE.get(status, AdsbError)(msg)
