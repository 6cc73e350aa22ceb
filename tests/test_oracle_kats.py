"""The reference's own known-answer tests (proj/tests/test_dockengine.cpp,
test_ligand_graph.cpp), replayed against the CPU oracle restatement and
against the reference sources compiled in oracle/_ref.  These pin the
oracle before it is trusted as the GPU checker."""
from __future__ import annotations

import math

import numpy as np
import pytest

from conftest import oracle_kinds
from helpers import explicit_pocket, flat_pocket, pose_at, pyramid_pocket
from oracle import Oracle
from paper_2110_11644_b200 import abi, api
from paper_2110_11644_b200.model import LigandBatch, Ligand

PI = math.pi


@pytest.fixture(scope="module", params=oracle_kinds())
def orc(request):
    return Oracle(request.param)


def one_atom_batch(x, element=0):
    lig = Ligand("C", np.array([x], dtype=np.float64), np.array([element], np.uint8), np.array([1], np.uint8),
                 np.zeros((0, 2), np.uint16), np.zeros(0, np.uint8), np.zeros(0, np.uint16), [])
    return LigandBatch([lig])


CUBE = explicit_pocket((2, 2, 2), 1.0, [1, 2, 3, 4, 5, 6, 7, 8])


def test_trilinear_kats(orc):
    # test_dockengine.cpp:154-186
    v = orc.field_values(CUBE, [[1.0, 0.0, 0.0], [0.0, 1.0, 1.0], [0.25, 0.5, 0.75], [1.0, 1.0, 1.0]])
    assert v[0] == 2.0 and v[1] == 7.0 and v[3] == 8.0
    assert v[2] == pytest.approx(5.25, rel=1e-14)
    assert v[2] == pytest.approx(1.0 + 0.25 + 2.0 * 0.5 + 4.0 * 0.75, rel=1e-14)
    outside = []
    for axis in range(3):
        for sign in (1.0, -1.0):
            p = [0.5, 0.5, 0.5]
            p[axis] += sign
            outside.append(p)
    assert np.all(orc.field_values(CUBE, outside) == -10.0)


def test_geo_score_kat(orc):
    # test_dockengine.cpp:188-213: CCO, heavy atoms on nodes 1, 2, 7
    lig = api.embed_ligand("CCO")
    assert lig.n_atoms == 9
    conf = np.full((9, 3), 50.0)
    conf[0] = [0.0, 0.0, 0.0]
    conf[1] = [1.0, 0.0, 0.0]
    conf[2] = [0.0, 1.0, 1.0]
    s, ev = orc.geo_score(CUBE, LigandBatch([lig]), conf)
    assert s[0] == 10.0 and ev[0] == 3
    far = conf.copy()
    far[:3] = [99.0, 0.0, 0.0]
    s, _ = orc.geo_score(CUBE, LigandBatch([lig]), far)
    assert s[0] == -30.0


@pytest.mark.parametrize("z,want,tol", [(3.0, 0.4, 1e-14), (4.5, 0.0, 0.0), (4.0, 0.2, 1e-12), (1.0, 0.4 - 5.0, 1e-12)])
def test_chem_pair_terms(orc, z, want, tol):
    # test_dockengine.cpp:215-240
    pk = flat_pocket(2, 1.0, protein=[(0, [0.0, 0.0, z])])
    got = orc.chem_score(pk, one_atom_batch([0, 0, 0]), np.zeros((1, 3)))[0]
    if tol == 0.0:
        assert got == want
    else:
        assert got == pytest.approx(want, rel=tol)


def test_chem_hydrogens_not_scored(orc):
    # test_dockengine.cpp:252-260
    pk = flat_pocket(2, 1.0, protein=[(0, [0.0, 0.0, 3.0])])
    lig = api.embed_ligand("C")
    conf = np.zeros((5, 3))
    conf[1:] = [0.0, 0.0, 2.9]
    assert orc.chem_score(pk, LigandBatch([lig]), conf)[0] == pytest.approx(0.4, rel=1e-12)


def test_chem_double_loop(orc):
    # test_dockengine.cpp:263-297
    prot = [(0, [0.0, 0.0, 3.2]), (2, [1.4, 0.0, 4.2])]
    pk = flat_pocket(2, 1.0, protein=prot)
    lig = Ligand("CNS", np.array([[0, 0, 0], [1.4, 0, 0], [2.8, 0, 0]], dtype=np.float64),
                 np.array([0, 1, 3], np.uint8), np.ones(3, np.uint8), np.array([[0, 1], [1, 2]], np.uint16),
                 np.ones(2, np.uint8), np.zeros(0, np.uint16), [])
    cls = {0: 0, 1: 1, 2: 1}
    expected = 0.0
    for e, x in zip(lig.element, lig.xyz):
        for pe, px in prot:
            d = float(np.linalg.norm(x - np.array(px)))
            if d >= 4.5:
                continue
            ca, cb = cls.get(int(e), 2), cls.get(int(pe), 2)
            w = 0.05 if (ca == 2 or cb == 2) else ((1.0 if ca == 1 else 0.4) if ca == cb else 0.1)
            expected += w * (1.0 if d <= 3.5 else (4.5 - d))
            if d < 2.0:
                expected -= 5.0
    got = orc.chem_score(pk, LigandBatch([lig]), lig.xyz)[0]
    assert got == pytest.approx(expected, rel=1e-12) and expected > 0.0


def test_flatten_no_torsions_identity(orc):
    lig = api.embed_heavy("c1ccccc1")
    conf, ang, st = orc.flatten(LigandBatch([lig]))
    assert st[0] == 0 and ang.size == 0
    assert np.array_equal(conf, lig.xyz)


def _twisted(smiles, angles):
    """Base conformation with the given torsion angles applied (the test's
    apply_torsions(embed_3d(lig), lig, {...}))."""
    lig = api.embed_heavy(smiles)
    port = Oracle("port")
    pose = np.zeros(1, dtype=abi.POSE_DTYPE)
    pose["rotation"][0] = [0, 0, 0, 1]
    conf = port.materialize(LigandBatch([lig]), np.array(angles, dtype=np.float64), pose)
    # identity transform adds +0.0; undo nothing (bit-identical for finite values)
    return lig.with_xyz(conf)


def test_flatten_one_torsion_matches_scan(orc):
    # test_dockengine.cpp:308-330
    lig = _twisted("CCCC", [PI])
    assert lig.n_torsions == 1
    port = Oracle("port")
    best, best_angle = -math.inf, 0.0
    pose = np.zeros(1, dtype=abi.POSE_DTYPE)
    pose["rotation"][0] = [0, 0, 0, 1]
    for k in range(36):
        angle = k * (2.0 * PI / 36)
        c = port.materialize(LigandBatch([lig]), np.array([angle]), pose)
        spread = port.internal_distance_sum(c)
        if spread > best:
            best, best_angle = spread, angle
    conf, ang, _ = orc.flatten(LigandBatch([lig]))
    assert orc.internal_distance_sum(conf) == best
    assert ang[0] == best_angle


@pytest.mark.parametrize("smiles,angles", [("CCCCC", [2 * PI / 3, PI]), ("CCCCCC", [PI, 2 * PI / 3, 4 * PI / 3])])
def test_flatten_within_one_percent(orc, smiles, angles):
    # test_dockengine.cpp:332-369
    lig = _twisted(smiles, angles)
    port = Oracle("port")
    pose = np.zeros(1, dtype=abi.POSE_DTYPE)
    pose["rotation"][0] = [0, 0, 0, 1]
    m = lig.n_torsions
    best = -math.inf
    grid = np.arange(36) * (2.0 * PI / 36)
    for idx in np.ndindex(*([36] * m)):
        c = port.materialize(LigandBatch([lig]), grid[list(idx)], pose)
        best = max(best, port.internal_distance_sum(c))
    conf, _, _ = orc.flatten(LigandBatch([lig]))
    assert orc.internal_distance_sum(conf) >= 0.99 * best


def test_flatten_bit_stable(orc):
    b = LigandBatch([api.embed_heavy("CC(C)CCO")])
    a1 = orc.flatten(b)
    a2 = orc.flatten(b)
    assert np.array_equal(a1[0], a2[0]) and np.array_equal(a1[1], a2[1])


def test_fibonacci(orc):
    # test_dockengine.cpp:381-408
    axes, _ = orc.fibonacci(64)
    assert np.allclose(np.linalg.norm(axes, axis=1), 1.0, rtol=1e-12)
    _, ang = orc.fibonacci(300)
    assert np.all(ang >= 0.0) and np.all(ang < 2 * PI)
    axes, _ = orc.fibonacci(256)
    dots = np.clip(axes @ axes.T, -1.0, 1.0)
    iu = np.triu_indices(256, 1)
    min_sep = float(np.min(np.arccos(dots[iu])))
    assert min_sep > 5.0 * PI / 180.0
    assert min_sep == pytest.approx(0.1935129210, rel=1e-8)


def test_initial_poses(orc):
    # test_dockengine.cpp:410-451
    pk = flat_pocket(5, 1.0)
    lig = api.embed_ligand("CCO")
    b = LigandBatch([lig])
    _, flat_ang, _ = orc.flatten(b)
    poses, confs, ev = orc.initial_poses(pk, b, flat_ang, 256)
    assert ev == 256 * lig.heavy_atom_count()
    centers = confs.mean(axis=1)
    assert np.all(np.linalg.norm(centers - pk.box_center(), axis=1) < 1e-9)
    port = Oracle("port")
    for i in range(0, 256, 17):  # recomputable from (angles, transform)
        again = port.materialize(b, flat_ang, poses[i:i + 1])
        assert np.array_equal(again, confs[i])
    q = poses["rotation"]
    d = np.max(np.abs(q[:, None, :] - q[None, :, :]), axis=2)
    assert np.all(d[np.triu_indices(256, 1)] > 0.0)
    with pytest.raises(ValueError):
        orc.initial_poses(pk, b, flat_ang, 0)


def test_local_search_pyramid(orc):
    # test_dockengine.cpp:480-509
    pk = pyramid_pocket(9, 1.0)
    lig = api.parse_smiles("C")
    b = LigandBatch([lig])
    cfg = abi.ScoringConfig()
    pose, ang, conf = pose_at(lig, [0.3, 0.7, 1.1])
    pose["geo_score"][0] = orc.geo_score(pk, b, conf)[0][0]
    start = float(pose["geo_score"][0])
    done, _, _, _, _ = orc.local_search(pk, b, cfg, pose, ang, conf)
    g = float(done["geo_score"][0])
    assert g >= start and g > start + 5.0 and g > 0.95 * 24.0
    top, tang, tconf = pose_at(lig, pk.box_center())
    top["geo_score"][0] = orc.geo_score(pk, b, tconf)[0][0]
    kept, _, kconf, _, _ = orc.local_search(pk, b, cfg, top, tang, tconf)
    assert kept["geo_score"][0] == top["geo_score"][0]
    assert np.array_equal(kconf, tconf)
    ex, _ = orc.exhaustive_dock(pk, b)
    assert g <= ex["geo_score"] + 1e-9
    assert ex["geo_score"] == pytest.approx(24.0, rel=1e-12)


@pytest.mark.parametrize("smiles,expect", [("C", 4 * 12 * 1), ("CCCC", 4 * (12 + 2) * 4)])
def test_local_search_eval_accounting(orc, smiles, expect):
    # test_dockengine.cpp:511-537 (flat field: four non-improving sweeps)
    pk = flat_pocket(9, 1.0)
    lig = api.parse_smiles("C") if smiles == "C" else api.embed_ligand(smiles)
    b = LigandBatch([lig])
    pose, ang, conf = pose_at(lig, pk.box_center())
    pose["geo_score"][0] = orc.geo_score(pk, b, conf)[0][0]
    _, _, _, ev, st = orc.local_search(pk, b, abi.ScoringConfig(), pose, ang, conf)
    assert st[0] == 0 and ev[0] == expect


def _oracle_cluster(points, scores, thr):
    """test_dockengine.cpp:548-579 restated: greedy leaders by descending score."""
    visit = sorted(range(len(points)), key=lambda i: -scores[i])  # stable
    leaders, rest = [], []
    for i in visit:
        if any(np.linalg.norm(np.array(points[i]) - np.array(points[l])) <= thr for l in leaders):
            rest.append(i)
        else:
            leaders.append(i)
    return leaders + rest


def test_cluster_and_select(orc):
    # test_dockengine.cpp:583-664
    lig = api.parse_smiles("C")
    b = LigandBatch([lig])
    pts = [[0, 0, 0], [1, 0, 0], [0, 1.5, 0], [10, 0, 0], [10.5, 0.5, 0], [0, 0, 20], [0.4, 0, 20], [0, 0.4, 20],
           [40, 40, 40], [10, 1.2, 0], [1.2, 1.2, 0], [0.2, 0.1, 19.6]]
    scores = [9.0, 3.0, 5.0, 8.0, 2.0, 7.0, 6.0, 1.0, 4.0, 2.5, 8.5, 0.5]
    confs = np.array(pts, dtype=np.float64).reshape(len(pts), 1, 3)
    order = orc.cluster_select(b, np.array(scores), confs, 3.0, len(pts))
    assert list(order) == _oracle_cluster(pts, scores, 3.0)
    top3 = orc.cluster_select(b, np.array(scores), confs, 3.0, 3)
    assert list(top3) == _oracle_cluster(pts, scores, 3.0)[:3] and scores[top3[0]] == 9.0
    tight = np.array([[0.1 * i, 0, 0] for i in range(5)]).reshape(5, 1, 3)
    o = orc.cluster_select(b, np.arange(5.0), tight, 3.0, 5)
    assert list(o) == [4, 3, 2, 1, 0]
    with pytest.raises(ValueError):
        orc.cluster_select(b, np.zeros(0), np.zeros((0, 1, 3)), 3.0, 5)


def test_exhaustive_dock_kats(orc):
    # test_dockengine.cpp:666-694
    pk = flat_pocket(3, 0.5)
    pk.values[pk.value_index(2, 1, 0)] = 7.0
    pk._desc = None
    b = LigandBatch([api.parse_smiles("C")])
    pose, conf = orc.exhaustive_dock(pk, b)
    assert np.linalg.norm(conf[0] - [1.0, 0.5, 0.0]) < 1e-12
    assert pose["geo_score"] == pytest.approx(7.0, rel=1e-12)
    pk2 = flat_pocket(2, 0.5)
    pk2.values[pk2.value_index(0, 0, 0)] = 3.0
    pk2.values[pk2.value_index(1, 1, 1)] = 3.0
    pk2._desc = None
    _, conf2 = orc.exhaustive_dock(pk2, b)
    assert np.linalg.norm(conf2[0]) < 1e-12
    with pytest.raises(ValueError):
        orc.exhaustive_dock(pk, LigandBatch([api.embed_ligand("CCO")]))
    with pytest.raises(ValueError):
        orc.exhaustive_dock(flat_pocket(35, 0.5), b)


def _twin_pocket():
    ref = Oracle("ref")
    return ref.build_pocket([0, 2], [[-2.0, 0.0, 0.0], [2.0, 0.0, 0.0]], [0, 0, 0], 5.0, 0.5)


@pytest.mark.skipif("ref" not in oracle_kinds(), reason="needs oracle/_ref for build_pocket")
def test_dock_and_score_deterministic(orc):
    # test_dockengine.cpp:696-744
    pk = _twin_pocket()
    lig = api.embed_ligand("CO")
    assert lig.n_torsions == 0
    b = LigandBatch([lig])
    cfg = abi.ScoringConfig(restarts=16, rescored=5)
    r1 = orc.dock_batch(pk, b, cfg)
    r2 = orc.dock_batch(pk, b, cfg)
    a, c = r1["results"][0], r2["results"][0]
    assert a["best_score"] == c["best_score"] and a["scoring_evals"] == c["scoring_evals"]
    assert a["poses_evaluated"] == 16 and np.isfinite(a["best_score"])
    assert np.array_equal(r1["conformation"], r2["conformation"])
    pose = np.zeros(1, dtype=abi.POSE_DTYPE)
    pose["rotation"][0] = a["rotation"]
    pose["translation"][0] = a["translation"]
    again = Oracle("port").materialize(b, r1["angles"], pose)
    assert np.array_equal(again, r1["conformation"])
    assert orc.chem_score(pk, b, r1["conformation"])[0] == a["best_score"]
    for bad in (dict(restarts=0), dict(rescored=0), dict(rmsd_threshold=0.0)):
        with pytest.raises(ValueError):
            orc.dock_batch(pk, b, abi.ScoringConfig(**bad))


def test_dock_eval_count_flat_field(orc):
    # test_dockengine.cpp:746-761: 8 restarts of CCCC on a zero field
    pk = flat_pocket(9, 1.0)
    lig = api.embed_ligand("CCCC")
    n = lig.heavy_atom_count()
    r = orc.dock_batch(pk, LigandBatch([lig]), abi.ScoringConfig(restarts=8, rescored=3))
    assert r["results"][0]["scoring_evals"] == 8 * n * (1 + 4 * (12 + 2 * 1))


# ---- ligand graph KATs (test_ligand_graph.cpp:39-121) on the oracle's detect_torsions
@pytest.mark.parametrize("smiles,bond,left,right", [
    ("CCCC", 1, [0, 1], [2, 3]),
    ("CC(C)C(=O)O", 2, [0, 1, 2], [3, 4, 5]),
])
def test_torsion_partition_kats(smiles, bond, left, right):
    port = Oracle("port")
    lig = api.parse_smiles(smiles)
    bonds, rights = port.detect_torsions(LigandBatch([lig]), 0)
    assert list(bonds) == [bond]
    assert list(rights[0]) == right
    assert sorted(set(range(lig.n_atoms)) - set(rights[0].tolist())) == left


def test_torsion_partition_biphenyl_and_cover():
    port = Oracle("port")
    lig = api.parse_smiles("c1ccccc1-c1ccccc1")
    bonds, rights = port.detect_torsions(LigandBatch([lig]), 0)
    assert len(bonds) == 1 and len(rights[0]) == 6
    for smi in ["CCCC", "CCCCCC", "CC(C)C(=O)O", "c1ccccc1-c1ccccc1", "CCOC(=O)c1ccccc1N"]:
        lig = api.parse_smiles(smi)
        bonds, rights = port.detect_torsions(LigandBatch([lig]), 0)
        for bi, r in zip(bonds, rights):
            a, b_ = lig.bonds[bi]
            assert b_ in set(r.tolist()) and a not in set(r.tolist())
    for smi in ["CCO", "c1ccccc1"]:
        bonds, _ = port.detect_torsions(LigandBatch([api.parse_smiles(smi)]), 0)
        assert len(bonds) == 0
