"""Loader for the in-tree native library ``_lib/libvsdock.so``.

The product path has no fallback: if the library is missing or no sm_100
device is visible, GPU entry points raise immediately.
"""
from __future__ import annotations

import ctypes as C
import os

from . import abi

HERE = os.path.dirname(os.path.abspath(__file__))
# VSDOCK_LIB overrides the library path (development A/B builds only).
LIB_PATH = os.environ.get("VSDOCK_LIB") or os.path.join(HERE, "_lib", "libvsdock.so")

_d = C.POINTER(C.c_double)
_u64 = C.POINTER(C.c_uint64)
_i32 = C.POINTER(C.c_int32)
_PD = C.POINTER(abi.PocketDesc)
_LB = C.POINTER(abi.LigandBatchDesc)
_CF = C.POINTER(abi.ScoringConfig)
_DR = C.POINTER(abi.DockResult)
_PO = C.POINTER(abi.PoseDesc)
_vp = C.c_void_p

# (name, restype, argtypes) for every entry point of include/vs_dock.h,
# vs_prep.h, vs_codec.h and vs_rank.h.
SIGNATURES = {
    "vs_abi_version": (C.c_int, []),
    "vs_device_count": (C.c_int, []),
    "vs_last_error_message": (C.c_char_p, []),
    "vs_scoring_config_default": (None, [_CF]),
    "vs_context_create": (C.c_int, [C.c_int, C.POINTER(_vp)]),
    "vs_context_destroy": (C.c_int, [_vp]),
    "vs_context_last_timing": (C.c_int, [_vp, _d, _i32]),
    "vs_pocket_create": (C.c_int, [_vp, _PD, C.POINTER(_vp)]),
    "vs_pocket_build": (C.c_int, [_vp, C.c_int32, C.POINTER(C.c_uint8), _d, _d, C.c_double, C.c_double,
                                  C.POINTER(_vp)]),
    "vs_pocket_info": (C.c_int, [_vp, _d, _d, _i32, _i32]),
    "vs_pocket_download": (C.c_int, [_vp, _vp, _d]),
    "vs_pocket_destroy": (C.c_int, [_vp]),
    "vs_dock_batch": (C.c_int, [_vp, _vp, _LB, _CF, _DR, _d, _d]),
    "vs_dock_batch_ex": (C.c_int, [_vp, _vp, _LB, _CF, _DR, _d, _d, _u64]),
    "vs_dock_batch_multi": (C.c_int, [_vp, C.POINTER(_vp), C.c_int32, _LB, _CF, _DR]),
    "vs_context_stage_timing": (C.c_int, [_vp, _d]),
    "vs_field_values": (C.c_int, [_vp, _vp, C.c_int64, _d, _d]),
    "vs_geo_score_batch": (C.c_int, [_vp, _vp, _LB, _d, _d, _u64]),
    "vs_chem_score_batch": (C.c_int, [_vp, _vp, _LB, _d, _d]),
    "vs_flatten_batch": (C.c_int, [_vp, _LB, C.c_int32, _d, _d, _i32]),
    "vs_initial_poses": (C.c_int, [_vp, _vp, _LB, _d, C.c_int32, _PO, _d, _u64, _i32]),
    "vs_cluster_select": (C.c_int, [_vp, _LB, C.c_int32, _d, _d, C.c_double, C.c_int32, _i32, _i32]),
    "vs_local_search_batch": (C.c_int, [_vp, _vp, _LB, _CF, _PO, _d, _d, _u64, _i32]),
    "vs_measure_peaks": (C.c_int, [C.c_int, _d]),
    "vs_measure_gather": (C.c_int, [C.c_int, C.c_int64, C.c_int32, _d]),
    "vs_selftest_sqrt": (C.c_int, [C.c_int, C.c_uint64, C.c_uint64, C.POINTER(C.c_uint64), _d]),
    "vs_selftest_div": (C.c_int, [C.c_int, C.c_uint64, C.c_uint64, C.POINTER(C.c_uint64), _d]),
    # vs_prep.h
    "vs_prep_smiles_batch": (C.c_int, [C.c_int32, C.POINTER(C.c_char_p), C.c_int32, C.c_int32, C.POINTER(_vp)]),
    "vs_ligand_set_view": (C.c_int, [_vp, _LB, C.POINTER(_i32)]),
    "vs_ligand_set_error": (C.c_char_p, [_vp, C.c_int32]),
    "vs_ligand_set_name": (C.c_char_p, [_vp, C.c_int32]),
    # vs_codec.h
    "vs_xslb_frame": (C.c_int32, [C.POINTER(C.c_uint8), C.c_int64, C.c_int64, C.c_int32, C.POINTER(C.c_int64),
                                  C.POINTER(C.c_int64)]),
    "vs_decode_records": (C.c_int, [_vp, C.POINTER(C.c_uint8), C.c_int64, C.POINTER(C.c_int64), C.c_int32,
                                    C.POINTER(_vp)]),
    "vs_encode_records": (C.c_int64, [_LB, C.POINTER(C.c_char_p), C.c_void_p, C.c_int64]),
    "vs_dock_records": (C.c_int, [_vp, C.POINTER(_vp), C.c_int32, C.POINTER(C.c_uint8), C.c_int64,
                                  C.POINTER(C.c_int64), C.c_int32, _CF, _DR, C.POINTER(C.c_int32)]),
    "vs_ligand_set_free": (None, [_vp]),
    # vs_rank.h
    "vs_rank_config_default": (None, [C.POINTER(abi.RankConfig)]),
    "vs_run_rank": (C.c_int, [C.c_uint64, abi.READ_FN, _vp, C.c_uint64, C.c_uint64, _PD, _CF,
                              C.POINTER(abi.RankConfig), abi.WRITE_FN, _vp, C.POINTER(abi.RankStats)]),
    "vs_merge_rankings": (C.c_int, [C.POINTER(C.c_char_p), C.POINTER(C.c_int64), C.c_int32, C.c_int64, C.c_int32,
                                    abi.WRITE_FN, _vp, C.POINTER(C.c_uint64)]),
    "vs_host_alloc": (C.c_int, [C.c_size_t, C.POINTER(_vp)]),
    "vs_host_free": (None, [_vp]),
    "vs_detect_torsions": (C.c_int32, [_LB, C.c_int32, C.POINTER(C.c_uint16), C.POINTER(C.c_uint8)]),
    "vs_bridge_bonds": (C.c_int32, [_LB, C.c_int32, C.POINTER(C.c_uint8)]),
    "vs_synth_smiles": (C.c_int64, [C.c_int32, C.c_uint64, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                    C.c_char_p, C.c_int64]),
    "vs_synth_smiles_ex": (C.c_int64, [C.c_int32, C.c_uint64, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                       C.c_char_p, C.c_int64]),
}

_lib = None


class NativeError(RuntimeError):
    pass


def lib():
    """The loaded libvsdock.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeError(f"{LIB_PATH} missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                              " or `make -C paper_2110_11644_b200/csrc`")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def last_error() -> str:
    return (lib().vs_last_error_message() or b"").decode()


def check(status: int, what: str):
    if status != abi.VS_OK:
        msg = last_error()
        if status == abi.VS_ERR_INVALID_ARGUMENT:
            raise ValueError(f"{what}: {msg}")
        raise NativeError(f"{what} failed (status {status}): {msg}")
