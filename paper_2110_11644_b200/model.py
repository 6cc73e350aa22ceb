"""Host-side data model mirroring the reference's Ligand / Pocket types.

Ligand  <- vscreen::Ligand        (ligand.hpp:46-71)
Pocket  <- vscreen::Pocket        (pocket.hpp:28-57)
Pose    <- vscreen::Pose          (pose.hpp:23-29)
DockResult <- vscreen::DockResult (pose.hpp:50-56)

Arrays are numpy; ``LigandBatch`` packs many ligands into the structure-of-
arrays layout of ``vs_ligand_batch`` (include/vs_dock.h) that the CUDA path
consumes.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import abi

ELEMENT_SYMBOLS = ["C", "N", "O", "S", "P", "F", "Cl", "Br", "I", "H", "Du"]  # elements.hpp:14-26
ELEM_H = 9


@dataclass
class Ligand:
    """One ligand graph with coordinates and its rotatable-bond partition."""

    name: str
    xyz: np.ndarray                 # (N, 3) float64
    element: np.ndarray             # (N,) uint8
    is_heavy: np.ndarray            # (N,) uint8
    bonds: np.ndarray               # (B, 2) uint16  (a, b)
    bond_order: np.ndarray          # (B,) uint8    1..4
    torsion_bond: np.ndarray        # (m,) uint16
    right_sets: list = field(default_factory=list)  # m arrays of uint16, ascending

    @property
    def n_atoms(self) -> int:
        return int(self.xyz.shape[0])

    @property
    def n_torsions(self) -> int:
        return int(self.torsion_bond.shape[0])

    def heavy_atom_count(self) -> int:
        return int(self.is_heavy.astype(bool).sum())

    def left_set(self, t: int) -> np.ndarray:
        mask = np.ones(self.n_atoms, dtype=bool)
        mask[self.right_sets[t]] = False
        return np.nonzero(mask)[0].astype(np.uint16)

    def with_xyz(self, xyz: np.ndarray) -> "Ligand":
        return Ligand(self.name, np.ascontiguousarray(xyz, dtype=np.float64).reshape(-1, 3),
                      self.element, self.is_heavy, self.bonds, self.bond_order,
                      self.torsion_bond, list(self.right_sets))

    def quantized(self) -> "Ligand":
        """quantize_to_wire (binary_codec.cpp:254-264): f64 -> f32 -> f64."""
        return self.with_xyz(self.xyz.astype(np.float32).astype(np.float64))


class LigandBatch:
    """Structure-of-arrays packing of many ligands (vs_ligand_batch)."""

    def __init__(self, ligands: Sequence[Ligand]):
        self.ligands = list(ligands)
        n = len(self.ligands)
        na = np.array([l.n_atoms for l in self.ligands], dtype=np.int64)
        nb = np.array([l.bonds.shape[0] for l in self.ligands], dtype=np.int64)
        nt = np.array([l.n_torsions for l in self.ligands], dtype=np.int64)
        self.atom_offset = np.zeros(n + 1, dtype=np.int32)
        self.atom_offset[1:] = np.cumsum(na)
        self.bond_offset = np.zeros(n + 1, dtype=np.int32)
        self.bond_offset[1:] = np.cumsum(nb)
        self.torsion_offset = np.zeros(n + 1, dtype=np.int32)
        self.torsion_offset[1:] = np.cumsum(nt)

        def cat(parts, dtype, shape_tail=()):
            parts = [np.asarray(p, dtype=dtype).reshape((-1,) + shape_tail) for p in parts]
            if not parts:
                return np.zeros((0,) + shape_tail, dtype=dtype)
            return np.ascontiguousarray(np.concatenate(parts))

        self.xyz = cat([l.xyz for l in self.ligands], np.float64, (3,))
        self.element = cat([l.element for l in self.ligands], np.uint8)
        self.is_heavy = cat([l.is_heavy for l in self.ligands], np.uint8)
        bonds = cat([l.bonds for l in self.ligands], np.uint16, (2,))
        self.bond_a = np.ascontiguousarray(bonds[:, 0])
        self.bond_b = np.ascontiguousarray(bonds[:, 1])
        self.bond_order = cat([l.bond_order for l in self.ligands], np.uint8)
        self.torsion_bond = cat([l.torsion_bond for l in self.ligands], np.uint16)
        rights = [r for l in self.ligands for r in l.right_sets]
        rl = np.array([len(r) for r in rights], dtype=np.int64)
        self.right_offset = np.zeros(len(rights) + 1, dtype=np.int32)
        self.right_offset[1:] = np.cumsum(rl)
        self.right_atoms = cat(rights, np.uint16)
        self._desc = None

    @property
    def n_ligands(self) -> int:
        return len(self.ligands)

    @property
    def n_atoms_total(self) -> int:
        return int(self.atom_offset[-1])

    @property
    def n_torsions_total(self) -> int:
        return int(self.torsion_offset[-1])

    def desc(self) -> abi.LigandBatchDesc:
        if self._desc is None:
            d = abi.LigandBatchDesc()
            d.n_ligands = self.n_ligands
            d.atom_offset = abi.ptr(self.atom_offset, C.c_int32)
            d.xyz = abi.ptr(self.xyz, C.c_double)
            d.element = abi.ptr(self.element, C.c_uint8)
            d.is_heavy = abi.ptr(self.is_heavy, C.c_uint8)
            d.bond_offset = abi.ptr(self.bond_offset, C.c_int32)
            d.bond_a = abi.ptr(self.bond_a, C.c_uint16)
            d.bond_b = abi.ptr(self.bond_b, C.c_uint16)
            d.bond_order = abi.ptr(self.bond_order, C.c_uint8)
            d.torsion_offset = abi.ptr(self.torsion_offset, C.c_int32)
            d.torsion_bond = abi.ptr(self.torsion_bond, C.c_uint16)
            d.right_offset = abi.ptr(self.right_offset, C.c_int32)
            d.right_atoms = abi.ptr(self.right_atoms, C.c_uint16)
            self._desc = d
        return self._desc

    def split_atoms(self, flat: np.ndarray) -> list:
        flat = flat.reshape(-1, 3)
        return [flat[self.atom_offset[i]:self.atom_offset[i + 1]] for i in range(self.n_ligands)]

    def split_torsions(self, flat: np.ndarray) -> list:
        return [flat[self.torsion_offset[i]:self.torsion_offset[i + 1]] for i in range(self.n_ligands)]


@dataclass
class Pocket:
    """Rigid binding site (pocket.hpp:28-57): x-fastest steric grid + protein atoms."""

    origin: np.ndarray              # (3,) float64
    spacing: float
    dims: tuple                     # (nx, ny, nz)
    values: np.ndarray              # (nx*ny*nz,) float64, x fastest
    protein_element: np.ndarray     # (P,) uint8
    protein_xyz: np.ndarray         # (P, 3) float64
    id: str = ""

    def __post_init__(self):
        self.origin = np.ascontiguousarray(self.origin, dtype=np.float64).reshape(3)
        self.values = np.ascontiguousarray(self.values, dtype=np.float64).reshape(-1)
        self.protein_element = np.ascontiguousarray(self.protein_element, dtype=np.uint8).reshape(-1)
        self.protein_xyz = np.ascontiguousarray(self.protein_xyz, dtype=np.float64).reshape(-1, 3)
        self.dims = tuple(int(d) for d in self.dims)
        self._desc = None

    def value_index(self, ix, iy, iz):
        return ix + self.dims[0] * (iy + self.dims[1] * iz)

    def value_at(self, ix, iy, iz) -> float:
        return float(self.values[self.value_index(ix, iy, iz)])

    def box_center(self) -> np.ndarray:
        hs = 0.5 * self.spacing
        return np.array([self.origin[a] + hs * (self.dims[a] - 1) for a in range(3)])

    def desc(self) -> abi.PocketDesc:
        if self._desc is None:
            d = abi.PocketDesc()
            for a in range(3):
                d.origin[a] = float(self.origin[a])
                d.dims[a] = self.dims[a]
            d.spacing = float(self.spacing)
            d.values = abi.ptr(self.values, C.c_double)
            d.n_protein = int(self.protein_element.shape[0])
            d.protein_element = abi.ptr(self.protein_element, C.c_uint8)
            d.protein_xyz = abi.ptr(self.protein_xyz, C.c_double)
            self._desc = d
        return self._desc


@dataclass
class Pose:
    rotation: np.ndarray            # (4,) x, y, z, w
    translation: np.ndarray         # (3,)
    torsion_angles: np.ndarray      # (m,)
    conformation: np.ndarray        # (N, 3)
    geo_score: float = 0.0
    chem_score: float | None = None


@dataclass
class DockResult:
    smiles: str
    best_score: float
    best_pose: Pose
    poses_evaluated: int
    scoring_evals: int
    status: int = 0
    clash_pairs: int = 0
    oob_samples: int = 0
    n_survivors: int = 0
