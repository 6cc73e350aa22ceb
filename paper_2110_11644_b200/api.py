"""Python mirror of the reference's dock-path API over libvsdock.so.

Reference names (proj/include/vscreen/...):
  dock_and_score        search.hpp:71-72   -> dock_and_score / dock_and_score_batch
  flatten               search.hpp:28-29   -> flatten
  local_search          search.hpp:55-56   -> local_search
  geo_score             grid.hpp:46-48     -> geo_score
  pocket_field_value    grid.hpp:40        -> pocket_field_value
  build_pocket          grid.hpp:35-37     -> build_pocket
  chem_score            chem.hpp:21-22     -> chem_score
  prepare_ligand        prep.cpp:37-44     -> prepare_ligand (host embed + GPU flatten)
  parse_smiles          smiles.hpp:26      -> parse_smiles (host)

Errors follow the reference: bad configurations raise ValueError (the
reference's InvalidArgument); per-ligand failures raise ValueError from the
single-ligand calls and are reported as status codes by the batch calls.
Everything that computes runs on the GPU through the C ABI; there is no CPU
fallback.
"""
from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import abi, native
from .model import DockResult, Ligand, LigandBatch, Pocket, Pose

ScoringConfig = abi.ScoringConfig

_ctx_lock = threading.Lock()
_contexts: dict = {}


class Context:
    """One device + stream (vs_context)."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        native.check(native.lib().vs_context_create(device, C.byref(h)), "vs_context_create")
        self.handle = h
        self.device = device

    def last_timing(self):
        ms = C.c_double()
        launches = C.c_int32()
        native.lib().vs_context_last_timing(self.handle, C.byref(ms), C.byref(launches))
        return ms.value, launches.value

    def stage_timing(self) -> dict:
        ms = np.zeros(4)
        native.lib().vs_context_stage_timing(self.handle, abi.ptr(ms, C.c_double))
        return dict(zip(("setup", "flatten", "search", "select"), ms.tolist()))

    def close(self):
        if self.handle:
            native.lib().vs_context_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def default_context(device: int = 0) -> Context:
    with _ctx_lock:
        if device not in _contexts:
            _contexts[device] = Context(device)
        return _contexts[device]


def device_count() -> int:
    return int(native.lib().vs_device_count())


class DevicePocket:
    """A pocket uploaded once and kept resident on one device (vs_pocket)."""

    def __init__(self, handle, ctx: Context, host: Pocket | None = None):
        self.handle = handle
        self.ctx = ctx
        self._host = host

    @classmethod
    def upload(cls, pocket: Pocket, ctx: Context | None = None) -> "DevicePocket":
        ctx = ctx or default_context()
        h = C.c_void_p()
        native.check(native.lib().vs_pocket_create(ctx.handle, C.byref(pocket.desc()), C.byref(h)), "vs_pocket_create")
        return cls(h, ctx, pocket)

    def info(self):
        org = np.zeros(3)
        sp = C.c_double()
        dims = np.zeros(3, dtype=np.int32)
        npro = C.c_int32()
        native.lib().vs_pocket_info(self.handle, abi.ptr(org, C.c_double), C.byref(sp), abi.ptr(dims, C.c_int32),
                                    C.byref(npro))
        return org, sp.value, tuple(int(d) for d in dims), npro.value

    def to_host(self, protein_element=None, protein_xyz=None) -> Pocket:
        if self._host is not None:
            return self._host
        org, sp, dims, _ = self.info()
        vals = np.zeros(int(np.prod(dims)))
        native.check(native.lib().vs_pocket_download(self.ctx.handle, self.handle, abi.ptr(vals, C.c_double)),
                     "vs_pocket_download")
        return Pocket(org, sp, dims, vals, protein_element if protein_element is not None else np.zeros(0, np.uint8),
                      protein_xyz if protein_xyz is not None else np.zeros((0, 3)))

    def close(self):
        if self.handle:
            native.lib().vs_pocket_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _dev_pocket(pocket, ctx: Context | None) -> DevicePocket:
    if isinstance(pocket, DevicePocket):
        return pocket
    return DevicePocket.upload(pocket, ctx)


def _batch(ligands) -> LigandBatch:
    if isinstance(ligands, LigandBatch):
        return ligands
    if isinstance(ligands, Ligand):
        return LigandBatch([ligands])
    return LigandBatch(ligands)


# ---------------------------------------------------------------- input side
def prepare_smiles(smiles: Sequence[str], mode: int = 1, nthreads: int = 8, strict: bool = True) -> list:
    """Host preparation (vs_prep_smiles_batch): mode 1 = hydrogens + 3D
    embedding + torsions (prepare_ligand before flatten); mode 2 = heavy
    graph + torsions only (detect_torsions(parse_smiles(s)))."""
    L = native.lib()
    enc = [s.encode() for s in smiles]
    arr = (C.c_char_p * max(len(enc), 1))(*enc)
    h = C.c_void_p()
    native.check(L.vs_prep_smiles_batch(len(enc), arr, mode, nthreads, C.byref(h)), "vs_prep_smiles_batch")
    try:
        ligs, status, errors = _ligands_of_set(h, len(enc), list(smiles))
    finally:
        L.vs_ligand_set_free(h)
    if strict:
        for i, st in enumerate(status):
            if st != 0:
                raise ValueError(errors[i])
    return ligs


def _ligands_of_set(h, n: int, names=None):
    """Ligand objects of a vs_ligand_set (None for failed entries), with the
    per-entry status and error text."""
    L = native.lib()
    v = abi.LigandBatchDesc()
    st = C.POINTER(C.c_int32)()
    L.vs_ligand_set_view(h, C.byref(v), C.byref(st))
    out = []
    ao = np.ctypeslib.as_array(v.atom_offset, (n + 1,)).copy()
    bo = np.ctypeslib.as_array(v.bond_offset, (n + 1,)).copy()
    to = np.ctypeslib.as_array(v.torsion_offset, (n + 1,)).copy()
    na, nb, nt = int(ao[-1]), int(bo[-1]), int(to[-1])

    def arr_of(p, shape, dt):
        if int(np.prod(shape)) == 0:
            return np.zeros(shape, dtype=dt)
        return np.ctypeslib.as_array(p, shape).astype(dt, copy=True)

    xyz = arr_of(v.xyz, (na * 3,), np.float64).reshape(-1, 3)
    el = arr_of(v.element, (na,), np.uint8)
    hv = arr_of(v.is_heavy, (na,), np.uint8)
    ba = arr_of(v.bond_a, (nb,), np.uint16)
    bb = arr_of(v.bond_b, (nb,), np.uint16)
    bord = arr_of(v.bond_order, (nb,), np.uint8)
    tb = arr_of(v.torsion_bond, (nt,), np.uint16)
    ro = np.ctypeslib.as_array(v.right_offset, (nt + 1,)).copy()
    ra = arr_of(v.right_atoms, (int(ro[-1]),), np.uint16)
    status = np.ctypeslib.as_array(st, (n,)).copy() if n else np.zeros(0, np.int32)
    errors = [L.vs_ligand_set_error(h, i).decode() for i in range(n)]
    for i in range(n):
        if status[i] != 0:
            out.append(None)
            continue
        name = names[i] if names is not None else L.vs_ligand_set_name(h, i).decode(errors="replace")
        a0, a1, b0, b1, t0, t1 = ao[i], ao[i + 1], bo[i], bo[i + 1], to[i], to[i + 1]
        out.append(Ligand(name, xyz[a0:a1].copy(), el[a0:a1].copy(), hv[a0:a1].copy(),
                          np.stack([ba[b0:b1], bb[b0:b1]], axis=1).copy(), bord[b0:b1].copy(),
                          tb[t0:t1].copy(), [ra[ro[t]:ro[t + 1]].copy() for t in range(t0, t1)]))
    return out, status, errors


# ---------------------------------------------------------------- records
XSLB_HEADER = b"XSLB\x01\x00\x00\x00"  # xslb_header (binary_codec.cpp:115-118)


def encode_records(ligands, names=None) -> bytes:
    """encode_record (binary_codec.cpp:129-163) of every ligand, back to back
    (no file header); names default to the ligands' names."""
    b = _batch(ligands)
    nm = names if names is not None else [getattr(l, "name", "") or "" for l in b.ligands]
    enc = [str(x).encode() for x in nm]
    arr = (C.c_char_p * max(len(enc), 1))(*enc)
    L = native.lib()
    need = -L.vs_encode_records(C.byref(b.desc()), arr, None, 0)
    buf = (C.c_uint8 * max(need, 1))()
    used = L.vs_encode_records(C.byref(b.desc()), arr, buf, need)
    if used < 0:
        raise RuntimeError("vs_encode_records: buffer too small")
    return bytes(buf[:used])


def frame_records(data: bytes, start: int = 0, max_records: int | None = None) -> np.ndarray:
    """Record start offsets from `start` along the length chain."""
    L = native.lib()
    buf = np.frombuffer(data, dtype=np.uint8)
    cap = max_records if max_records is not None else max(1, len(data) // 8)
    offs = np.zeros(cap, dtype=np.int64)
    nxt = C.c_int64(0)
    n = L.vs_xslb_frame(abi.ptr(buf, C.c_uint8), len(data), start, cap, abi.ptr(offs, C.c_int64), C.byref(nxt))
    if n < 0:
        raise ValueError("bad framing arguments")
    return offs[:n]


def decode_records(data: bytes, offsets=None, ctx: Context | None = None):
    """GPU decode_record (binary_codec.cpp:165-222) of the records at
    `offsets` (default: framed from 0): (ligands, status, errors); a ligand
    is None where the record fails with the reference's CodecError."""
    ctx = ctx or default_context()
    if offsets is None:
        offsets = frame_records(data)
    offs = np.ascontiguousarray(offsets, dtype=np.int64)
    buf = np.frombuffer(data, dtype=np.uint8)
    h = C.c_void_p()
    L = native.lib()
    native.check(L.vs_decode_records(ctx.handle, abi.ptr(buf, C.c_uint8), len(data), abi.ptr(offs, C.c_int64),
                                     len(offs), C.byref(h)), "vs_decode_records")
    try:
        return _ligands_of_set(h, len(offs))
    finally:
        L.vs_ligand_set_free(h)


def parse_smiles(smiles: str) -> Ligand:
    """detect_torsions(parse_smiles(s)): heavy-atom graph, zero coordinates."""
    return prepare_smiles([smiles], mode=2)[0]


def embed_heavy(smiles: str) -> Ligand:
    """detect_torsions(parse_smiles(s)) with embed_3d coordinates, no hydrogens."""
    return prepare_smiles([smiles], mode=3)[0]


def embed_ligand(smiles: str) -> Ligand:
    """Hydrogens + embedding + torsions, no flatten (test_dockengine.cpp:29-33)."""
    return prepare_smiles([smiles], mode=1)[0]


def synthetic_smiles(n: int, seed: int = 20260819, heavy=(26, 34), rot=(5, 7), grammar: int = 0) -> list:
    cap = max(256, n * 96)
    while True:
        buf = C.create_string_buffer(cap)
        used = native.lib().vs_synth_smiles_ex(n, seed, heavy[0], heavy[1], rot[0], rot[1], grammar, buf, cap)
        if used == -2:
            raise ValueError("requested heavy/rotor window is unreachable")
        if used >= 0:
            raw = buf.raw[:used]
            return [s.decode() for s in raw.split(b"\0")[:n]]
        cap *= 2


# ---------------------------------------------------------------- GPU calls
def flatten(ligands, max_sweeps: int = 20, ctx: Context | None = None):
    """flatten (search.cpp:27-69) of each ligand from its stored coordinates."""
    ctx = ctx or default_context()
    b = _batch(ligands)
    conf = np.zeros((max(b.n_atoms_total, 1), 3))
    ang = np.zeros(max(b.n_torsions_total, 1))
    st = np.zeros(max(b.n_ligands, 1), dtype=np.int32)
    native.check(native.lib().vs_flatten_batch(ctx.handle, C.byref(b.desc()), max_sweeps, abi.ptr(conf, C.c_double),
                                               abi.ptr(ang, C.c_double), abi.ptr(st, C.c_int32)), "vs_flatten_batch")
    return conf[:b.n_atoms_total], ang[:b.n_torsions_total], st[:b.n_ligands]


def prepare_ligand(smiles: Sequence[str] | str, quantize: bool = False, ctx: Context | None = None, nthreads: int = 8):
    """prepare_ligand (prep.cpp:37-44): host hydrogens/embedding/torsions, GPU
    flatten, optional wire quantisation (binary_codec.cpp:254-264)."""
    single = isinstance(smiles, str)
    ligs = prepare_smiles([smiles] if single else list(smiles), mode=1, nthreads=nthreads)
    b = LigandBatch(ligs)
    conf, _, st = flatten(b, 20, ctx)
    out = []
    for i, lig in enumerate(ligs):
        if st[i] != abi.VS_LIG_OK:
            raise ValueError(f"{lig.name}: {abi.LIGAND_STATUS_NAMES.get(int(st[i]), st[i])}")
        l2 = lig.with_xyz(conf[b.atom_offset[i]:b.atom_offset[i + 1]])
        out.append(l2.quantized() if quantize else l2)
    return out[0] if single else out


def build_pocket(protein_element, protein_xyz, center, radius: float, spacing: float,
                 ctx: Context | None = None) -> DevicePocket:
    """build_pocket (grid.cpp:15-57) on the GPU; the result stays resident."""
    ctx = ctx or default_context()
    el = np.ascontiguousarray(protein_element, dtype=np.uint8)
    xyz = np.ascontiguousarray(protein_xyz, dtype=np.float64).reshape(-1, 3)
    c = np.ascontiguousarray(center, dtype=np.float64).reshape(3)
    h = C.c_void_p()
    native.check(native.lib().vs_pocket_build(ctx.handle, el.size, abi.ptr(el, C.c_uint8), abi.ptr(xyz, C.c_double),
                                              abi.ptr(c, C.c_double), radius, spacing, C.byref(h)), "vs_pocket_build")
    dp = DevicePocket(h, ctx)
    dp._host = dp.to_host(el, xyz)
    return dp


def pocket_field_value(pocket, points, ctx: Context | None = None) -> np.ndarray:
    ctx = ctx or default_context()
    dp = _dev_pocket(pocket, ctx)
    pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
    out = np.zeros(max(pts.shape[0], 1))
    native.check(native.lib().vs_field_values(ctx.handle, dp.handle, pts.shape[0], abi.ptr(pts, C.c_double),
                                              abi.ptr(out, C.c_double)), "vs_field_values")
    return out[:pts.shape[0]]


def geo_score(pocket, ligands, conformation, ctx: Context | None = None):
    ctx = ctx or default_context()
    dp = _dev_pocket(pocket, ctx)
    b = _batch(ligands)
    conf = np.ascontiguousarray(conformation, dtype=np.float64).reshape(-1, 3)
    out = np.zeros(max(b.n_ligands, 1))
    ev = np.zeros(max(b.n_ligands, 1), dtype=np.uint64)
    native.check(native.lib().vs_geo_score_batch(ctx.handle, dp.handle, C.byref(b.desc()), abi.ptr(conf, C.c_double),
                                                 abi.ptr(out, C.c_double), abi.ptr(ev, C.c_uint64)),
                 "vs_geo_score_batch")
    return out[:b.n_ligands], ev[:b.n_ligands]


def chem_score(pocket, ligands, conformation, ctx: Context | None = None) -> np.ndarray:
    ctx = ctx or default_context()
    dp = _dev_pocket(pocket, ctx)
    b = _batch(ligands)
    conf = np.ascontiguousarray(conformation, dtype=np.float64).reshape(-1, 3)
    out = np.zeros(max(b.n_ligands, 1))
    native.check(native.lib().vs_chem_score_batch(ctx.handle, dp.handle, C.byref(b.desc()), abi.ptr(conf, C.c_double),
                                                  abi.ptr(out, C.c_double)), "vs_chem_score_batch")
    return out[:b.n_ligands]


def local_search(pocket, ligands, poses: np.ndarray, angles: np.ndarray, conformation: np.ndarray,
                 config: ScoringConfig | None = None, ctx: Context | None = None):
    """local_search (search.cpp:109-193), one start pose per ligand.
    poses: POSE_DTYPE array; returns (poses, angles, conformation, evals, status)."""
    ctx = ctx or default_context()
    dp = _dev_pocket(pocket, ctx)
    b = _batch(ligands)
    cfg = config or ScoringConfig()
    poses = np.ascontiguousarray(poses, dtype=abi.POSE_DTYPE).copy()
    ang = np.ascontiguousarray(angles, dtype=np.float64).copy()
    if ang.size == 0:
        ang = np.zeros(1)
    conf = np.ascontiguousarray(conformation, dtype=np.float64).reshape(-1, 3).copy()
    ev = np.zeros(max(b.n_ligands, 1), dtype=np.uint64)
    st = np.zeros(max(b.n_ligands, 1), dtype=np.int32)
    native.check(native.lib().vs_local_search_batch(
        ctx.handle, dp.handle, C.byref(b.desc()), C.byref(cfg), poses.ctypes.data_as(C.POINTER(abi.PoseDesc)),
        abi.ptr(ang, C.c_double), abi.ptr(conf, C.c_double), abi.ptr(ev, C.c_uint64), abi.ptr(st, C.c_int32)),
        "vs_local_search_batch")
    return poses, ang[:b.n_torsions_total], conf, ev[:b.n_ligands], st[:b.n_ligands]


def initial_poses(pocket, ligand: Ligand, flat_angles, k: int, ctx: Context | None = None):
    """initial_poses (search.cpp:84-107) from the ligand's coordinates and the
    given flat angles.  Returns (POSE_DTYPE[k], conformations (k, N, 3), evals)."""
    ctx = ctx or default_context()
    dp = _dev_pocket(pocket, ctx)
    b = _batch([ligand])
    fa = np.ascontiguousarray(flat_angles, dtype=np.float64)
    if fa.size == 0:
        fa = np.zeros(1)
    poses = np.zeros(max(k, 1), dtype=abi.POSE_DTYPE)
    confs = np.zeros((max(k, 1) * max(ligand.n_atoms, 1), 3))
    ev = np.zeros(1, dtype=np.uint64)
    st = np.zeros(1, dtype=np.int32)
    native.check(native.lib().vs_initial_poses(ctx.handle, dp.handle, C.byref(b.desc()), abi.ptr(fa, C.c_double), k,
                                               poses.ctypes.data_as(C.POINTER(abi.PoseDesc)),
                                               abi.ptr(confs, C.c_double), abi.ptr(ev, C.c_uint64),
                                               abi.ptr(st, C.c_int32)), "vs_initial_poses")
    if st[0] != abi.VS_LIG_OK:
        raise ValueError(abi.LIGAND_STATUS_NAMES.get(int(st[0]), st[0]))
    return poses[:k], confs[:k * ligand.n_atoms].reshape(k, ligand.n_atoms, 3), int(ev[0])


def cluster_and_select(ligand: Ligand, geo, conformations, threshold: float, top: int,
                       ctx: Context | None = None) -> np.ndarray:
    """cluster_and_select (search.cpp:195-236): indices of the selected poses."""
    ctx = ctx or default_context()
    b = _batch([ligand])
    geo = np.ascontiguousarray(geo, dtype=np.float64)
    confs = np.ascontiguousarray(conformations, dtype=np.float64)
    n = int(geo.shape[0])
    order = np.zeros(max(n, 1), dtype=np.int32)
    cnt = np.zeros(1, dtype=np.int32)
    native.check(native.lib().vs_cluster_select(ctx.handle, C.byref(b.desc()), n, abi.ptr(geo, C.c_double),
                                                abi.ptr(confs if confs.size else np.zeros(1), C.c_double), threshold,
                                                top, abi.ptr(order, C.c_int32), abi.ptr(cnt, C.c_int32)),
                 "vs_cluster_select")
    return order[:int(cnt[0])]


@dataclass
class BatchResult:
    results: np.ndarray          # DOCK_RESULT_DTYPE per ligand
    best_angles: np.ndarray      # per torsion (batch order)
    best_conformation: np.ndarray | None  # (atoms, 3)
    batch: LigandBatch
    kernel_ms: float = 0.0
    launches: int = 0
    counters: np.ndarray | None = None   # (n, 9) Appendix B counters when requested
    stage_ms: dict | None = None

    def result(self, i: int) -> DockResult:
        r = self.results[i]
        b = self.batch
        lig = b.ligands[i] if i < len(b.ligands) else None
        conf = None
        if self.best_conformation is not None:
            conf = self.best_conformation[b.atom_offset[i]:b.atom_offset[i + 1]]
        pose = Pose(np.array(r["rotation"]), np.array(r["translation"]),
                    self.best_angles[b.torsion_offset[i]:b.torsion_offset[i + 1]], conf,
                    float(r["best_geo_score"]), float(r["best_score"]))
        return DockResult(lig.name if lig is not None else "", float(r["best_score"]), pose,
                          int(r["poses_evaluated"]), int(r["scoring_evals"]), int(r["status"]),
                          int(r["clash_pairs"]), int(r["oob_samples"]), int(r["n_survivors"]))


def dock_and_score_batch(pocket, ligands, config: ScoringConfig | None = None, ctx: Context | None = None,
                         want_conformation: bool = True, out: dict | None = None,
                         want_counters: bool = False) -> BatchResult:
    """dock_and_score over a batch (search.cpp:238-276).  `out` may supply
    preallocated (e.g. pinned) result arrays: keys results/angles/conf."""
    ctx = ctx or default_context()
    dp = _dev_pocket(pocket, ctx)
    b = _batch(ligands)
    cfg = config or ScoringConfig()
    out = out or {}
    res = out.get("results")
    if res is None:
        res = np.zeros(max(b.n_ligands, 1), dtype=abi.DOCK_RESULT_DTYPE)
    ang = out.get("angles")
    if ang is None:
        ang = np.zeros(max(b.n_torsions_total, 1))
    conf = out.get("conf") if want_conformation else None
    if conf is None and want_conformation:
        conf = np.zeros((max(b.n_atoms_total, 1), 3))
    counters = np.zeros((max(b.n_ligands, 1), 9), dtype=np.uint64) if want_counters else None
    native.check(native.lib().vs_dock_batch_ex(ctx.handle, dp.handle, C.byref(b.desc()), C.byref(cfg),
                                               res.ctypes.data_as(C.POINTER(abi.DockResult)),
                                               abi.ptr(ang, C.c_double), abi.ptr(conf, C.c_double),
                                               abi.ptr(counters, C.c_uint64)), "vs_dock_batch")
    ms, launches = ctx.last_timing()
    return BatchResult(res[:b.n_ligands], ang[:b.n_torsions_total],
                       conf[:b.n_atoms_total] if conf is not None else None, b, ms, launches,
                       counters[:b.n_ligands] if counters is not None else None, ctx.stage_timing())


def dock_and_score_multi(pockets, ligands, config: ScoringConfig | None = None, ctx: Context | None = None,
                         out=None):
    """dock_and_score of every ligand against every pocket (BASELINE
    configs[4]); ligand-only stages run once.  Returns (results array of shape
    (n_pockets, n_ligands), device ms, launches, stage ms)."""
    ctx = ctx or default_context()
    dps = [_dev_pocket(p, ctx) for p in pockets]
    b = _batch(ligands)
    cfg = config or ScoringConfig()
    res = out if out is not None else np.zeros((len(dps), max(b.n_ligands, 1)), dtype=abi.DOCK_RESULT_DTYPE)
    arr = (C.c_void_p * len(dps))(*[d.handle for d in dps])
    native.check(native.lib().vs_dock_batch_multi(ctx.handle, arr, len(dps), C.byref(b.desc()), C.byref(cfg),
                                                  res.ctypes.data_as(C.POINTER(abi.DockResult))),
                 "vs_dock_batch_multi")
    ms, launches = ctx.last_timing()
    return res[:, :b.n_ligands], ms, launches, ctx.stage_timing()


def dock_records(pockets, data: bytes, offsets=None, config: ScoringConfig | None = None, ctx: Context | None = None):
    """Decode + dock the records of an .xslb byte stream on the GPU without a
    host round trip (vs_dock_records).  Returns (results of shape
    (n_pockets, n_records), record status, device ms, stage ms)."""
    ctx = ctx or default_context()
    dps = [_dev_pocket(p, ctx) for p in pockets]
    if offsets is None:
        offsets = frame_records(data)
    offs = np.ascontiguousarray(offsets, dtype=np.int64)
    n = len(offs)
    buf = np.frombuffer(data, dtype=np.uint8)
    cfg = config or ScoringConfig()
    res = np.zeros((len(dps), max(n, 1)), dtype=abi.DOCK_RESULT_DTYPE)
    rst = np.zeros(max(n, 1), dtype=np.int32)
    arr = (C.c_void_p * len(dps))(*[d.handle for d in dps])
    native.check(native.lib().vs_dock_records(ctx.handle, arr, len(dps), abi.ptr(buf, C.c_uint8), len(data),
                                              abi.ptr(offs, C.c_int64), n, C.byref(cfg),
                                              res.ctypes.data_as(C.POINTER(abi.DockResult)),
                                              abi.ptr(rst, C.c_int32)), "vs_dock_records")
    ms, _ = ctx.last_timing()
    return res[:, :n], rst[:n], ms, ctx.stage_timing()


def dock_and_score(pocket, ligand: Ligand, config: ScoringConfig | None = None,
                   ctx: Context | None = None) -> DockResult:
    """Single-ligand dock_and_score; raises ValueError where the reference
    throws InvalidArgument."""
    br = dock_and_score_batch(pocket, [ligand], config, ctx)
    st = int(br.results[0]["status"])
    if st not in (abi.VS_LIG_OK, abi.VS_LIG_NONFINITE):
        raise ValueError(abi.LIGAND_STATUS_NAMES.get(st, f"ligand status {st}"))
    return br.result(0)


# ---------------------------------------------------------------- pipeline rank
XSLB_HEADER = bytes([0x58, 0x53, 0x4C, 0x42, 1, 0, 0, 0])  # xslb_header(): magic "XSLB", version 1


def plan_slabs(file_size: int, n_ranks: int) -> list[tuple[int, int]]:
    """plan_slabs (pipeline.cpp:32-45): rank i owns record starts in
    [size * i / n, size * (i + 1) / n)."""
    if n_ranks < 1:
        raise ValueError("rank count must be at least 1")
    return [(file_size * i // n_ranks, file_size * (i + 1) // n_ranks) for i in range(n_ranks)]


def run_rank(data: bytes, pocket, config: ScoringConfig | None = None, slab: tuple[int, int] | None = None,
             devices=None, workers_per_device: int = 2, batch_records: int = 32768, chunk_bytes: int = 1 << 20,
             writer_buffer_bytes: int = 4 << 20):
    """run_rank (pipeline.cpp:297-389) of one slab of an in-memory .xslb image
    on the B200 CUDA workers (vs_run_rank): returns (output text, RankStats
    dict).  `pocket` is a host Pocket (model.Pocket); rows are format_row
    lines in record order."""
    buf = np.frombuffer(data, dtype=np.uint8)
    start, stop = slab if slab is not None else (0, len(data))
    parts = []

    def _read(_u, off, out, n):
        n = max(0, min(n, len(data) - off))
        C.memmove(out, buf.ctypes.data + off, n)
        return n

    def _write(_u, p, n):
        parts.append(C.string_at(p, n))
        return 0

    rf, wf = abi.READ_FN(_read), abi.WRITE_FN(_write)
    rc = abi.RankConfig()
    native.lib().vs_rank_config_default(C.byref(rc))
    dev_arr = None
    if devices is not None:
        dev_arr = (C.c_int32 * len(devices))(*devices)
        rc.n_devices = len(devices)
        rc.devices = C.cast(dev_arr, C.POINTER(C.c_int32))
    rc.workers_per_device = workers_per_device
    rc.batch_records = batch_records
    rc.chunk_bytes = chunk_bytes
    rc.writer_buffer_bytes = writer_buffer_bytes
    st = abi.RankStats()
    cfg = config or ScoringConfig()
    native.check(native.lib().vs_run_rank(len(data), rf, None, start, stop, C.byref(pocket.desc()), C.byref(cfg),
                                          C.byref(rc), wf, None, C.byref(st)), "vs_run_rank")
    return b"".join(parts).decode(), st.as_dict()


def merge_rankings(texts, top_k: int = -1, threads: int = 0) -> tuple[str, int]:
    """cmd_merge's ranking (merge.cpp:81-147) of rank score texts in rank
    order, natively (vs_merge_rankings): (ranking text, rows)."""
    bs = [t.encode() if isinstance(t, str) else bytes(t) for t in texts]
    arr = (C.c_char_p * max(len(bs), 1))(*bs)
    lens = (C.c_int64 * max(len(bs), 1))(*[len(b) for b in bs])
    parts = []

    def _write(_u, p, n):
        parts.append(C.string_at(p, n))
        return 0

    wf = abi.WRITE_FN(_write)
    rows = C.c_uint64()
    native.check(native.lib().vs_merge_rankings(arr, lens, len(bs), top_k, threads, wf, None, C.byref(rows)),
                 "vs_merge_rankings")
    return b"".join(parts).decode(), int(rows.value)
