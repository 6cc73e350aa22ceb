"""Input side: the product's host preparation (parse_smiles + add_hydrogens
+ embed_3d + detect_torsions, include/vs_prep.h) must reproduce the
reference's bit for bit, and the synthetic generator must be deterministic."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import oracle_kinds
from paper_2110_11644_b200 import api

KAT_SMILES = ["C", "CC", "C=C", "CCO", "CCCC", "CC(C)C", "CC(C)(C)C", "CC(C)C(=O)O", "CCOC(=O)C", "C1CCCCC1",
              "c1ccccc1", "c1ccncc1", "c1ccoc1", "C1CCCCC1CC", "c1ccc2ccccc2c1", "C1CCc2ccccc2C1",
              "c1ccc(-c2ccccc2)cc1", "ClCBr", "NCC(=O)O", "CC(N)C(=O)O", "CCOC(=O)c1ccccc1N", "c1ccccc1-c1ccccc1"]

needs_ref = pytest.mark.skipif("ref" not in oracle_kinds(), reason="oracle/_ref not built")


def _same(a, b):
    return (np.array_equal(a.xyz, b.xyz) and np.array_equal(a.element, b.element)
            and np.array_equal(a.is_heavy, b.is_heavy) and np.array_equal(a.bonds, b.bonds)
            and np.array_equal(a.bond_order, b.bond_order) and np.array_equal(a.torsion_bond, b.torsion_bond)
            and len(a.right_sets) == len(b.right_sets)
            and all(np.array_equal(x, y) for x, y in zip(a.right_sets, b.right_sets)))


@needs_ref
@pytest.mark.parametrize("mode", [1, 2])
def test_prep_matches_reference_kats(mode):
    from oracle import Oracle
    ref = Oracle("ref")
    mine = api.prepare_smiles(KAT_SMILES, mode=mode)
    for s, m in zip(KAT_SMILES, mine):
        assert _same(m, ref.prepare(s, mode, False)), s


@needs_ref
def test_prep_matches_reference_synthetic():
    from oracle import Oracle
    ref = Oracle("ref")
    smi = api.synthetic_smiles(300, seed=42)
    mine = api.prepare_smiles(smi, mode=1)
    for s, m in zip(smi, mine):
        assert _same(m, ref.prepare(s, 1, False)), s


def test_hydrogen_kats():
    # test_geometry.cpp:80-134
    assert api.prepare_smiles(["C"], 1)[0].n_atoms == 5
    lig = api.prepare_smiles(["CCO"], 1)[0]
    owners = [int(a) for a, b in lig.bonds if not lig.is_heavy[b]]
    assert owners == [0, 0, 0, 1, 1, 2]
    assert api.prepare_smiles(["c1ccccc1"], 1)[0].n_atoms == 12
    assert api.prepare_smiles(["c1ccncc1"], 1)[0].n_atoms == 11
    assert api.prepare_smiles(["c1ccoc1"], 1)[0].n_atoms == 9


@pytest.mark.parametrize("bad", ["", "C1CC", "C(C", "C)C", "[CH4]", "C.C", "CC=", "C%12CC%12", "X"])
def test_parse_errors(bad):
    with pytest.raises(ValueError):
        api.prepare_smiles([bad], mode=2)


def test_synthetic_library_deterministic_and_in_window():
    a = api.synthetic_smiles(600, seed=7)
    b = api.synthetic_smiles(600, seed=7)
    assert a == b and len(set(a)) > 550
    ligs = api.prepare_smiles(a, mode=1)
    n = np.array([l.heavy_atom_count() for l in ligs])
    m = np.array([l.n_torsions for l in ligs])
    assert n.min() >= 26 and n.max() <= 34 and m.min() >= 5 and m.max() <= 7
    assert 27.0 < n.mean() < 32.0


def test_synthetic_protein_voxel_mix():
    from paper_2110_11644_b200 import synth
    el, xyz = synth.synthetic_protein()
    assert el.shape == (2400,) and xyz.shape == (2400, 3)
    d = np.linalg.norm(xyz[:, None, :] - xyz[None, :, :], axis=2) + np.eye(2400) * 10
    assert d.min() >= 1.2
    assert set(np.unique(el)) <= {0, 1, 2, 3}
