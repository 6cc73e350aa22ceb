"""ctypes mirror of include/vs_dock.h (the C ABI of the B200 dock path).

Only plain-data layouts live here; loading of libvsdock.so is in
``paper_2110_11644_b200.native``.  The same layouts are what the test-only
oracle libraries (oracle/_build/liboracle.so, oracle/_ref/libvsref.so)
accept, so tests can hand one packed batch to all three.
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np

VS_OK = 0
VS_ERR_INVALID_ARGUMENT = 1
VS_ERR_NO_DEVICE = 2
VS_ERR_CUDA = 3
VS_ERR_LIMIT = 4
VS_ERR_INTERNAL = 5

VS_LIG_OK = 0
VS_LIG_EMPTY = 1
VS_LIG_DEGENERATE_AXIS = 2
VS_LIG_BAD_TORSION = 3
VS_LIG_NO_HEAVY = 4
VS_LIG_TOO_LARGE = 5
VS_LIG_NONFINITE = 6
VS_LIG_BAD_RECORD = 7

LIGAND_STATUS_NAMES = {
    VS_LIG_OK: "ok",
    VS_LIG_EMPTY: "empty conformation",
    VS_LIG_DEGENERATE_AXIS: "degenerate torsion axis",
    VS_LIG_BAD_TORSION: "torsion index out of range",
    VS_LIG_NO_HEAVY: "no heavy atoms",
    VS_LIG_TOO_LARGE: "ligand exceeds device limits",
    VS_LIG_NONFINITE: "non-finite score",
    VS_LIG_BAD_RECORD: "record failed to decode",
}

VS_MAX_ATOMS = 256
VS_MAX_HEAVY = 128
VS_MAX_TORSIONS = 31
VS_MAX_RESTARTS = 65536

_d = C.POINTER(C.c_double)
_i32 = C.POINTER(C.c_int32)
_u8 = C.POINTER(C.c_uint8)
_u16 = C.POINTER(C.c_uint16)


class ScoringConfig(C.Structure):
    """vs_scoring_config == ScoringConfig (pose.hpp:33-48), same defaults."""

    _fields_ = [
        ("restarts", C.c_int32),
        ("rescored", C.c_int32),
        ("rmsd_threshold", C.c_double),
        ("step_translation", C.c_double),
        ("step_rotation", C.c_double),
        ("step_torsion", C.c_double),
        ("min_translation", C.c_double),
        ("max_iterations", C.c_int32),
        ("flatten_max_sweeps", C.c_int32),
    ]

    def __init__(self, **kw):
        super().__init__()
        self.restarts = 256
        self.rescored = 30
        self.rmsd_threshold = 3.0
        self.step_translation = 1.0
        self.step_rotation = 20.0 * (math.pi / 180.0)
        self.step_torsion = 20.0 * (math.pi / 180.0)
        self.min_translation = 0.1
        self.max_iterations = 200
        self.flatten_max_sweeps = 20
        for k, v in kw.items():
            if not hasattr(self, k):
                raise AttributeError(k)
            setattr(self, k, v)


class PocketDesc(C.Structure):
    _fields_ = [
        ("origin", C.c_double * 3),
        ("spacing", C.c_double),
        ("dims", C.c_int32 * 3),
        ("values", _d),
        ("n_protein", C.c_int32),
        ("protein_element", _u8),
        ("protein_xyz", _d),
    ]


class LigandBatchDesc(C.Structure):
    _fields_ = [
        ("n_ligands", C.c_int32),
        ("atom_offset", _i32),
        ("xyz", _d),
        ("element", _u8),
        ("is_heavy", _u8),
        ("bond_offset", _i32),
        ("bond_a", _u16),
        ("bond_b", _u16),
        ("bond_order", _u8),
        ("torsion_offset", _i32),
        ("torsion_bond", _u16),
        ("right_offset", _i32),
        ("right_atoms", _u16),
    ]


class DockResult(C.Structure):
    _fields_ = [
        ("status", C.c_int32),
        ("n_survivors", C.c_int32),
        ("best_score", C.c_double),
        ("best_geo_score", C.c_double),
        ("rotation", C.c_double * 4),
        ("translation", C.c_double * 3),
        ("poses_evaluated", C.c_uint64),
        ("scoring_evals", C.c_uint64),
        ("clash_pairs", C.c_int32),
        ("oob_samples", C.c_int32),
    ]


class PoseDesc(C.Structure):
    _fields_ = [
        ("rotation", C.c_double * 4),
        ("translation", C.c_double * 3),
        ("geo_score", C.c_double),
    ]


DOCK_RESULT_DTYPE = np.dtype(
    [
        ("status", np.int32),
        ("n_survivors", np.int32),
        ("best_score", np.float64),
        ("best_geo_score", np.float64),
        ("rotation", np.float64, 4),
        ("translation", np.float64, 3),
        ("poses_evaluated", np.uint64),
        ("scoring_evals", np.uint64),
        ("clash_pairs", np.int32),
        ("oob_samples", np.int32),
    ],
    align=True,
)
assert DOCK_RESULT_DTYPE.itemsize == C.sizeof(DockResult)

POSE_DTYPE = np.dtype(
    [("rotation", np.float64, 4), ("translation", np.float64, 3), ("geo_score", np.float64)],
    align=True,
)
assert POSE_DTYPE.itemsize == C.sizeof(PoseDesc)


class RankConfig(C.Structure):
    """vs_rank_config (include/vs_rank.h)."""
    _fields_ = [("n_devices", C.c_int32), ("devices", C.POINTER(C.c_int32)), ("workers_per_device", C.c_int32),
                ("batch_records", C.c_int32), ("chunk_bytes", C.c_int64), ("writer_buffer_bytes", C.c_int64)]


class RankStats(C.Structure):
    """vs_rank_stats = RankStats (pipeline.hpp:96-115) + GPU batch counters."""
    _fields_ = [(f, C.c_uint64) for f in ("ligands_docked", "records_skipped", "dock_errors", "rows_written",
                                          "chunks_read", "bytes_read", "write_calls", "bytes_written")] + \
               [("workers", C.c_int32)] + \
               [(f, C.c_double) for f in ("wall_seconds", "reader_busy_seconds", "splitter_busy_seconds",
                                          "docker_busy_seconds", "writer_busy_seconds")] + \
               [("batches", C.c_uint64), ("resyncs", C.c_uint64)]

    def as_dict(self) -> dict:
        return {f: getattr(self, f) for f, _ in self._fields_}


READ_FN = C.CFUNCTYPE(C.c_int64, C.c_void_p, C.c_uint64, C.POINTER(C.c_uint8), C.c_int64)
WRITE_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.POINTER(C.c_char), C.c_int64)


def ptr(a: np.ndarray | None, ctype):
    """Pointer to a contiguous numpy array (None -> NULL)."""
    if a is None:
        return C.cast(None, C.POINTER(ctype))
    assert a.flags["C_CONTIGUOUS"], "array must be C-contiguous"
    return a.ctypes.data_as(C.POINTER(ctype))
