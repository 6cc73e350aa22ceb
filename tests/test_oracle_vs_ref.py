"""Pin the oracle restatement against the reference's own sources
(oracle/_ref): identical results, bit for bit, on synthetic workloads."""
from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import oracle_kinds
from oracle import Oracle
from paper_2110_11644_b200 import abi, api, synth
from paper_2110_11644_b200.model import LigandBatch

pytestmark = pytest.mark.skipif("ref" not in oracle_kinds(), reason="oracle/_ref not built")


@pytest.fixture(scope="module")
def setup():
    ref, port = Oracle("ref"), Oracle("port", trig=0)
    el, xyz = synth.synthetic_protein(900, seed=3, half_box=12.5)
    pocket = ref.build_pocket(el, xyz, [0, 0, 0], 7.0, 0.5)
    smi = api.synthetic_smiles(96, seed=99, heavy=(14, 30), rot=(1, 7))
    ligs = [ref.prepare(s, 0, True) for s in smi]
    return ref, port, pocket, LigandBatch(ligs)


def test_dock_bit_exact(setup):
    ref, port, pocket, b = setup
    cfg = abi.ScoringConfig(restarts=6, rescored=4)
    r = ref.dock_batch(pocket, b, cfg, nthreads=os.cpu_count() or 4)
    p = port.dock_batch(pocket, b, cfg, nthreads=os.cpu_count() or 4)
    for f in ("status", "best_score", "best_geo_score", "rotation", "translation", "scoring_evals", "poses_evaluated"):
        assert np.array_equal(r["results"][f], p["results"][f]), f
    assert np.array_equal(r["angles"], p["angles"])
    assert np.array_equal(r["conformation"], p["conformation"])


def test_flatten_bit_exact(setup):
    ref, port, _, b = setup
    raw = LigandBatch(api.prepare_smiles([l.name for l in b.ligands], mode=1))
    c1, a1, s1 = ref.flatten(raw, 20, nthreads=4)
    c2, a2, s2 = port.flatten(raw, 20, nthreads=4)
    assert np.array_equal(c1, c2) and np.array_equal(a1, a2) and np.array_equal(s1, s2)


def test_local_search_bit_exact_random_poses(setup):
    ref, port, pocket, b = setup
    rng = np.random.default_rng(1)
    n = b.n_ligands
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    poses = np.zeros(n, dtype=abi.POSE_DTYPE)
    poses["rotation"] = q
    poses["translation"] = rng.uniform(-2, 2, (n, 3))
    ang = rng.uniform(-3, 3, b.n_torsions_total)
    conf = port.materialize(b, ang, poses)
    poses["geo_score"] = port.geo_score(pocket, b, conf)[0]
    cfg = abi.ScoringConfig()
    r = ref.local_search(pocket, b, cfg, poses, ang, conf)
    p = port.local_search(pocket, b, cfg, poses, ang, conf)
    for x, y in zip(r, p):
        assert np.array_equal(np.asarray(x).view(np.uint8), np.asarray(y).view(np.uint8))


def test_field_geo_chem_bit_exact(setup):
    ref, port, pocket, b = setup
    pts = np.random.default_rng(2).uniform(-8, 8, (5000, 3))
    assert np.array_equal(ref.field_values(pocket, pts), port.field_values(pocket, pts))
    shifted = b.xyz + 0.37
    assert np.array_equal(ref.geo_score(pocket, b, shifted)[0], port.geo_score(pocket, b, shifted)[0])
    assert np.array_equal(ref.chem_score(pocket, b, shifted), port.chem_score(pocket, b, shifted))
