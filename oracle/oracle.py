"""ORACLE — test infrastructure only (checker, never the product path).

Python loader for the two CPU oracles:

* ``kind="port"``: oracle/_build/liboracle.so, the plain-C++ restatement of
  the reference's hot path (oracle/vs_oracle.cpp), with Appendix-B counters
  and a switch for the torsion trig (glibc vs the GPU's correctly rounded
  routine).
* ``kind="ref"``: oracle/_ref/libvsref.so, the reference's OWN sources
  compiled against third_party/eigen_subset (oracle/build_ref.sh); also offers the
  reference's input side (SMILES -> prepared ligand, build_pocket, codec).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this.
"""
from __future__ import annotations

import ctypes as C
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_2110_11644_b200 import abi  # noqa: E402  (plain-data ABI layouts only)
from paper_2110_11644_b200.model import Ligand, LigandBatch, Pocket  # noqa: E402

PORT_LIB = os.path.join(HERE, "_build", "liboracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libvsref.so")

_d = C.POINTER(C.c_double)
_u64 = C.POINTER(C.c_uint64)
_i32 = C.POINTER(C.c_int32)
_u8 = C.POINTER(C.c_uint8)
_u16 = C.POINTER(C.c_uint16)
_PD = C.POINTER(abi.PocketDesc)
_LB = C.POINTER(abi.LigandBatchDesc)
_CF = C.POINTER(abi.ScoringConfig)
_DR = C.POINTER(abi.DockResult)
_PO = C.POINTER(abi.PoseDesc)


def available(kind: str) -> bool:
    return os.path.exists(PORT_LIB if kind == "port" else REF_LIB)


class Oracle:
    def __init__(self, kind: str = "port", trig: int = 0):
        self.kind = kind
        self.trig = trig
        path = PORT_LIB if kind == "port" else REF_LIB
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (run `make -C oracle` / oracle/build_ref.sh)")
        self.lib = C.CDLL(path)
        p = "vso_" if kind == "port" else "vsref_"
        self.p = p
        L = self.lib

        def fn(name, res, args):
            f = getattr(L, p + name)
            f.restype = res
            f.argtypes = args
            return f

        self._dock = fn("dock_batch", C.c_int,
                        [_PD, _LB, _CF, C.c_int, _DR, _d, _d] + ([_u64] if kind == "port" else []))
        self._field = fn("field_values", C.c_int, [_PD, C.c_int64, _d, _d])
        self._geo = fn("geo_score", C.c_int, [_PD, _LB, _d, _d, _u64])
        self._chem = fn("chem_score", C.c_int, [_PD, _LB, _d, _d])
        self._flat = fn("flatten", C.c_int, [_LB, C.c_int, _d, _d, _i32, C.c_int])
        self._ls = fn("local_search", C.c_int, [_PD, _LB, _CF, _PO, _d, _d, _u64, _i32])
        self._init = fn("initial_poses", C.c_int, [_PD, _LB, _d, C.c_int, _PO, _d, _u64])
        self._clus = fn("cluster_select", C.c_int, [_LB, C.c_int, _d, _d, C.c_double, C.c_int, _i32])
        self._exh = fn("exhaustive_dock", C.c_int, [_PD, _LB, _PO, _d])
        self._fib = fn("fibonacci", C.c_int, [C.c_int, _d, _d])
        self._ids = fn("internal_distance_sum", C.c_double, [C.c_int, _d])
        if kind == "port":
            self._trig = fn("set_trig_mode", C.c_int, [C.c_int])
            self._sc_cr = fn("sincos_cr", None, [C.c_double, _d, _d])
            self._sc_gl = fn("sincos_glibc", None, [C.c_double, _d, _d])
            self._mat = fn("materialize", C.c_int, [_LB, _d, _PO, _d, _i32])
            self._detect = fn("detect_torsions", C.c_int, [_LB, C.c_int, _u16, _u8])
        else:
            self._prep = fn("prepare", C.c_void_p, [C.c_char_p, C.c_int, C.c_int])
            self._free = fn("ligand_free", None, [C.c_void_p])
            self._counts = fn("ligand_counts", None, [C.c_void_p, _i32])
            self._name = fn("ligand_name", C.c_char_p, [C.c_void_p])
            self._export = fn("ligand_export", None,
                              [C.c_void_p, _d, _u8, _u8, _u16, _u16, _u8, _u16, _i32, _u16])
            self._build = fn("build_pocket", C.c_int,
                             [C.c_int32, _u8, _d, _d, C.c_double, C.c_double, _i32, _d, _d])
            self._err = fn("last_error", C.c_char_p, [])
            self._decode = fn("decode_record", C.c_void_p, [_u8, C.c_int64, C.c_int64, C.POINTER(C.c_int64)])
            self._encode = fn("encode_record", C.c_int64, [C.c_void_p, _u8, C.c_int64])

    # ------------------------------------------------------------ config
    def set_trig_mode(self, mode: int):
        """0: glibc sin/cos (reference-faithful); 1: the GPU's correctly rounded routine.
        The mode is per Oracle object and applied before every call (the
        library keeps one global switch)."""
        assert self.kind == "port"
        self.trig = mode

    def _apply_trig(self):
        if self.kind == "port":
            self._trig(self.trig)

    def sincos_shift_check(self, chains: int, n_moves: int, step: float, levels: int, seed: int) -> int:
        """Mismatches of the incremental torsion trig (vs_crtrig sincos_shift)
        against sincos_cr along random move chains (see vs_oracle.cpp)."""
        f = self.lib.vso_sincos_shift_check
        f.restype = C.c_uint64
        f.argtypes = [C.c_int, C.c_int, C.c_double, C.c_int, C.c_uint64]
        return int(f(chains, n_moves, step, levels, seed))

    def sincos(self, x: float, correctly_rounded: bool = True):
        s, c = C.c_double(), C.c_double()
        (self._sc_cr if correctly_rounded else self._sc_gl)(x, C.byref(s), C.byref(c))
        return s.value, c.value

    def materialize(self, batch: LigandBatch, angles: np.ndarray, poses: np.ndarray) -> np.ndarray:
        """apply_rigid(apply_torsions(base, angles), T) per ligand (pose.hpp:20-22)."""
        self._apply_trig()
        ang = np.ascontiguousarray(angles, dtype=np.float64)
        if ang.size == 0:
            ang = np.zeros(1)
        poses = np.ascontiguousarray(poses, dtype=abi.POSE_DTYPE)
        out = np.zeros((max(batch.n_atoms_total, 1), 3))
        st = np.zeros(batch.n_ligands, dtype=np.int32)
        self._mat(C.byref(batch.desc()), abi.ptr(ang, C.c_double), poses.ctypes.data_as(_PO),
                  abi.ptr(out, C.c_double), abi.ptr(st, C.c_int32))
        return out[:batch.n_atoms_total]

    # ------------------------------------------------------------ hot path
    def dock_batch(self, pocket: Pocket, batch: LigandBatch, cfg: abi.ScoringConfig, nthreads: int = 1,
                   want_conf: bool = True, want_counters: bool = False):
        self._apply_trig()
        res = np.zeros(batch.n_ligands, dtype=abi.DOCK_RESULT_DTYPE)
        ang = np.zeros(max(batch.n_torsions_total, 1), dtype=np.float64)
        conf = np.zeros((max(batch.n_atoms_total, 1), 3), dtype=np.float64) if want_conf else None
        args = [C.byref(pocket.desc()), C.byref(batch.desc()), C.byref(cfg), nthreads,
                res.ctypes.data_as(_DR), abi.ptr(ang, C.c_double), abi.ptr(conf, C.c_double)]
        counters = None
        if self.kind == "port":
            counters = np.zeros((batch.n_ligands, 9), dtype=np.uint64) if want_counters else None
            args.append(abi.ptr(counters, C.c_uint64))
        rc = self._dock(*args)
        if rc != abi.VS_OK:
            raise ValueError(f"{self.p}dock_batch failed: status {rc}")
        out = {"results": res, "angles": ang[:batch.n_torsions_total],
               "conformation": conf[:batch.n_atoms_total] if conf is not None else None}
        if counters is not None:
            out["counters"] = counters
        return out

    def field_values(self, pocket: Pocket, xyz: np.ndarray) -> np.ndarray:
        xyz = np.ascontiguousarray(xyz, dtype=np.float64).reshape(-1, 3)
        out = np.zeros(xyz.shape[0])
        self._field(C.byref(pocket.desc()), xyz.shape[0], abi.ptr(xyz, C.c_double), abi.ptr(out, C.c_double))
        return out

    def geo_score(self, pocket: Pocket, batch: LigandBatch, conf: np.ndarray):
        conf = np.ascontiguousarray(conf, dtype=np.float64).reshape(-1, 3)
        out = np.zeros(batch.n_ligands)
        ev = np.zeros(batch.n_ligands, dtype=np.uint64)
        self._geo(C.byref(pocket.desc()), C.byref(batch.desc()), abi.ptr(conf, C.c_double),
                  abi.ptr(out, C.c_double), abi.ptr(ev, C.c_uint64))
        return out, ev

    def chem_score(self, pocket: Pocket, batch: LigandBatch, conf: np.ndarray) -> np.ndarray:
        conf = np.ascontiguousarray(conf, dtype=np.float64).reshape(-1, 3)
        out = np.zeros(batch.n_ligands)
        self._chem(C.byref(pocket.desc()), C.byref(batch.desc()), abi.ptr(conf, C.c_double),
                   abi.ptr(out, C.c_double))
        return out

    def flatten(self, batch: LigandBatch, max_sweeps: int = 20, nthreads: int = 1):
        self._apply_trig()
        conf = np.zeros((max(batch.n_atoms_total, 1), 3))
        ang = np.zeros(max(batch.n_torsions_total, 1))
        st = np.zeros(batch.n_ligands, dtype=np.int32)
        self._flat(C.byref(batch.desc()), max_sweeps, abi.ptr(conf, C.c_double), abi.ptr(ang, C.c_double),
                   abi.ptr(st, C.c_int32), nthreads)
        return conf[:batch.n_atoms_total], ang[:batch.n_torsions_total], st

    def local_search(self, pocket: Pocket, batch: LigandBatch, cfg, poses: np.ndarray, angles: np.ndarray,
                     conf: np.ndarray):
        self._apply_trig()
        poses = poses.copy()
        angles = np.ascontiguousarray(angles, dtype=np.float64).copy()
        if angles.size == 0:
            angles = np.zeros(1)
        conf = np.ascontiguousarray(conf, dtype=np.float64).reshape(-1, 3).copy()
        ev = np.zeros(batch.n_ligands, dtype=np.uint64)
        st = np.zeros(batch.n_ligands, dtype=np.int32)
        self._ls(C.byref(pocket.desc()), C.byref(batch.desc()), C.byref(cfg), poses.ctypes.data_as(_PO),
                 abi.ptr(angles, C.c_double), abi.ptr(conf, C.c_double), abi.ptr(ev, C.c_uint64),
                 abi.ptr(st, C.c_int32))
        return poses, angles[:batch.n_torsions_total], conf, ev, st

    def initial_poses(self, pocket: Pocket, batch: LigandBatch, flat_angles: np.ndarray, k: int):
        self._apply_trig()
        lig = batch.ligands[0]
        fa = np.ascontiguousarray(flat_angles, dtype=np.float64)
        if fa.size == 0:
            fa = np.zeros(1)
        poses = np.zeros(k, dtype=abi.POSE_DTYPE)
        confs = np.zeros((k * lig.n_atoms, 3))
        ev = np.zeros(1, dtype=np.uint64)
        rc = self._init(C.byref(pocket.desc()), C.byref(batch.desc()), abi.ptr(fa, C.c_double), k,
                        poses.ctypes.data_as(_PO), abi.ptr(confs, C.c_double), abi.ptr(ev, C.c_uint64))
        if rc != 0:
            raise ValueError(f"initial_poses failed: {rc}")
        return poses, confs.reshape(k, lig.n_atoms, 3), int(ev[0])

    def cluster_select(self, batch: LigandBatch, geo: np.ndarray, confs: np.ndarray, threshold: float,
                       top: int) -> np.ndarray:
        geo = np.ascontiguousarray(geo, dtype=np.float64)
        confs = np.ascontiguousarray(confs, dtype=np.float64)
        order = np.zeros(max(top, 1), dtype=np.int32)
        n = self._clus(C.byref(batch.desc()), geo.shape[0], abi.ptr(geo, C.c_double), abi.ptr(confs, C.c_double),
                       threshold, top, abi.ptr(order, C.c_int32))
        if n < 0:
            raise ValueError("cluster_and_select failed")
        return order[:n]

    def exhaustive_dock(self, pocket: Pocket, batch: LigandBatch):
        self._apply_trig()
        pose = np.zeros(1, dtype=abi.POSE_DTYPE)
        conf = np.zeros((batch.ligands[0].n_atoms, 3))
        rc = self._exh(C.byref(pocket.desc()), C.byref(batch.desc()), pose.ctypes.data_as(_PO),
                       abi.ptr(conf, C.c_double))
        if rc != 0:
            raise ValueError("exhaustive_dock refused")
        return pose[0], conf

    def fibonacci(self, k: int):
        axes = np.zeros((k, 3))
        ang = np.zeros(k)
        self._fib(k, abi.ptr(axes, C.c_double), abi.ptr(ang, C.c_double))
        return axes, ang

    def internal_distance_sum(self, xyz: np.ndarray) -> float:
        xyz = np.ascontiguousarray(xyz, dtype=np.float64).reshape(-1, 3)
        return float(self._ids(xyz.shape[0], abi.ptr(xyz, C.c_double)))

    def detect_torsions(self, batch: LigandBatch, i: int):
        lig = batch.ligands[i]
        bonds = np.zeros(max(lig.bonds.shape[0], 1), dtype=np.uint16)
        masks = np.zeros(max(lig.bonds.shape[0], 1) * max(lig.n_atoms, 1), dtype=np.uint8)
        m = self._detect(C.byref(batch.desc()), i, abi.ptr(bonds, C.c_uint16), abi.ptr(masks, C.c_uint8))
        rights = [np.nonzero(masks[t * lig.n_atoms:(t + 1) * lig.n_atoms])[0].astype(np.uint16) for t in range(m)]
        return bonds[:m].copy(), rights

    # ------------------------------------------------------------ input side (ref only)
    def _handle_to_ligand(self, h) -> Ligand:
        cnt = np.zeros(4, dtype=np.int32)
        self._counts(h, abi.ptr(cnt, C.c_int32))
        na, nb, nt, nr = (int(x) for x in cnt)
        xyz = np.zeros((max(na, 1), 3))
        el = np.zeros(max(na, 1), dtype=np.uint8)
        hv = np.zeros(max(na, 1), dtype=np.uint8)
        ba = np.zeros(max(nb, 1), dtype=np.uint16)
        bb = np.zeros(max(nb, 1), dtype=np.uint16)
        bo = np.zeros(max(nb, 1), dtype=np.uint8)
        tb = np.zeros(max(nt, 1), dtype=np.uint16)
        ro = np.zeros(nt + 1, dtype=np.int32)
        ra = np.zeros(max(nr, 1), dtype=np.uint16)
        self._export(h, abi.ptr(xyz, C.c_double), abi.ptr(el, C.c_uint8), abi.ptr(hv, C.c_uint8),
                     abi.ptr(ba, C.c_uint16), abi.ptr(bb, C.c_uint16), abi.ptr(bo, C.c_uint8),
                     abi.ptr(tb, C.c_uint16), abi.ptr(ro, C.c_int32), abi.ptr(ra, C.c_uint16))
        name = self._name(h).decode()
        return Ligand(name, xyz[:na].copy(), el[:na].copy(), hv[:na].copy(),
                      np.stack([ba[:nb], bb[:nb]], axis=1).copy(), bo[:nb].copy(), tb[:nt].copy(),
                      [ra[ro[t]:ro[t + 1]].copy() for t in range(nt)])

    def prepare(self, smiles: str, mode: int = 0, quantize: bool = False) -> Ligand:
        """mode 0: prepare_ligand (prep.cpp:37-44); 1: embedded, unflattened; 2: graph only."""
        assert self.kind == "ref"
        h = self._prep(smiles.encode(), mode, 1 if quantize else 0)
        if not h:
            raise ValueError(self._err().decode())
        try:
            return self._handle_to_ligand(h)
        finally:
            self._free(h)

    def encode_prepared(self, smiles: str, mode: int = 0, quantize: bool = True) -> bytes:
        """encode_record (binary_codec.cpp:129-163) of the reference's own
        prepared ligand (see prepare)."""
        assert self.kind == "ref"
        h = self._prep(smiles.encode(), mode, 1 if quantize else 0)
        if not h:
            raise ValueError(self._err().decode())
        try:
            n = self._encode(h, None, 0)
            buf = np.zeros(n, dtype=np.uint8)
            self._encode(h, abi.ptr(buf, C.c_uint8), n)
            return buf.tobytes()
        finally:
            self._free(h)

    def decode_record(self, data: bytes, offset: int):
        buf = np.frombuffer(data, dtype=np.uint8).copy()
        nxt = C.c_int64(0)
        h = self._decode(abi.ptr(buf, C.c_uint8), buf.size, offset, C.byref(nxt))
        if not h:
            raise ValueError(self._err().decode())
        try:
            return self._handle_to_ligand(h), int(nxt.value)
        finally:
            self._free(h)

    def build_pocket(self, protein_element, protein_xyz, center, radius, spacing) -> Pocket:
        assert self.kind == "ref"
        el = np.ascontiguousarray(protein_element, dtype=np.uint8)
        xyz = np.ascontiguousarray(protein_xyz, dtype=np.float64).reshape(-1, 3)
        c = np.ascontiguousarray(center, dtype=np.float64)
        dims = np.zeros(3, dtype=np.int32)
        org = np.zeros(3)
        rc = self._build(el.size, abi.ptr(el, C.c_uint8), abi.ptr(xyz, C.c_double), abi.ptr(c, C.c_double),
                         radius, spacing, abi.ptr(dims, C.c_int32), abi.ptr(org, C.c_double), None)
        if rc != 0:
            raise ValueError(self._err().decode())
        vals = np.zeros(int(dims.prod()))
        self._build(el.size, abi.ptr(el, C.c_uint8), abi.ptr(xyz, C.c_double), abi.ptr(c, C.c_double),
                    radius, spacing, abi.ptr(dims, C.c_int32), abi.ptr(org, C.c_double), abi.ptr(vals, C.c_double))
        return Pocket(org, spacing, tuple(dims), vals, el, xyz, id="built")

    # ------------------------------------------------------------ pipeline
    def run_rank(self, data: bytes, pocket: Pocket, cfg: abi.ScoringConfig, slab=None, workers: int = 1,
                 chunk_bytes: int = 1 << 20):
        """The reference's own run_rank (pipeline.cpp:297-389; kind "ref"
        only) over an in-memory .xslb image: (output text, counters dict)."""
        assert self.kind == "ref"
        f = self.lib.vsref_run_rank
        f.restype = C.c_int
        f.argtypes = [C.POINTER(C.c_uint8), C.c_int64, C.c_uint64, C.c_uint64, _PD, _CF, C.c_int, C.c_int64,
                      C.POINTER(C.c_void_p), C.POINTER(C.c_int64), C.POINTER(C.c_uint64)]
        self.lib.vsref_free.argtypes = [C.c_void_p]
        buf = np.frombuffer(data, dtype=np.uint8)
        start, stop = slab if slab is not None else (0, len(data))
        out = C.c_void_p()
        n = C.c_int64()
        cnt = (C.c_uint64 * 4)()
        rc = f(buf.ctypes.data_as(C.POINTER(C.c_uint8)), len(data), start, stop, C.byref(pocket.desc()), C.byref(cfg),
               workers, chunk_bytes, C.byref(out), C.byref(n), cnt)
        if rc != abi.VS_OK:
            raise ValueError(self._err().decode())
        text = C.string_at(out, n.value).decode()
        self.lib.vsref_free(out)
        return text, dict(zip(("ligands_docked", "records_skipped", "dock_errors", "rows_written"), list(cnt)))

    def cmd_merge(self, out_dir: str) -> int:
        """The reference's cmd_merge (merge.cpp:81-147): writes
        <out_dir>/ranking.tsv from job.txt + rank<i>.scores/.stats."""
        assert self.kind == "ref"
        f = self.lib.vsref_cmd_merge
        f.restype = C.c_int64
        f.argtypes = [C.c_char_p]
        n = f(out_dir.encode())
        if n < 0:
            raise ValueError(self._err().decode())
        return int(n)

    def format_rank_stats(self, counters) -> str:
        f = self.lib.vsref_format_rank_stats
        f.restype = C.c_int64
        f.argtypes = [C.POINTER(C.c_uint64), C.c_char_p, C.c_int64]
        cnt = (C.c_uint64 * 4)(*counters)
        buf = C.create_string_buffer(4096)
        n = f(cnt, buf, 4096)
        return buf.raw[:n].decode()

