"""The opt-in FP32 search screen (VS_SCREEN=1) must leave
every result bit-identical: the search tests of test_gpu_parity.py run again
with the screen on (the pockets here have <= 4 node values, so the screen
kernel k_search<1, true> is the one that runs)."""
from __future__ import annotations

import os

import numpy as np
import pytest

import test_gpu_parity as P
from helpers import golden_pocket, load_golden
from oracle import Oracle
from paper_2110_11644_b200 import abi, api
from paper_2110_11644_b200.model import LigandBatch

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def screen_on():
    old = os.environ.get("VS_SCREEN")
    os.environ["VS_SCREEN"] = "1"
    yield
    if old is None:
        del os.environ["VS_SCREEN"]
    else:
        os.environ["VS_SCREEN"] = old


@pytest.fixture(scope="module")
def env(gpu_ctx):  # the same inputs as test_gpu_parity.env
    from paper_2110_11644_b200 import synth
    el, xyz = synth.synthetic_protein(1200, seed=5, half_box=13.0)
    pocket = api.build_pocket(el, xyz, [0.0, 0.0, 0.0], 8.0, 0.5, gpu_ctx)
    smi = api.synthetic_smiles(192, seed=17, heavy=(14, 34), rot=(0, 8))
    ligs = api.prepare_ligand(smi, quantize=True, ctx=gpu_ctx)
    return gpu_ctx, pocket, pocket.to_host(), LigandBatch(ligs)


def test_screen_local_search_random_poses(env):
    P.test_local_search_random_poses_bit_exact(env)


def test_screen_node_box_faces_and_nan(gpu_ctx):
    P.test_local_search_node_box_faces_bit_exact(gpu_ctx)


@pytest.mark.parametrize("k,rescored", [(8, 30), (1, 1), (30, 30)])
def test_screen_dock_bit_exact(env, k, rescored):
    P.test_dock_bit_exact_vs_oracle(env, k, rescored)


@pytest.mark.parametrize("kw", [dict(restarts=6, rescored=4, min_translation=0.001),
                                dict(restarts=6, rescored=6, step_torsion=1.0, step_rotation=0.8, step_translation=2.0)])
def test_screen_config_variations(env, kw):
    P.test_dock_bit_exact_config_variations(env, kw)


def test_screen_large_flexible_ligands(env):
    P.test_large_flexible_ligands(env)


def test_screen_benched_config_1200_ligands(gpu_ctx):
    """configs[1] (k=30) on the golden fixture's 1,200 ligands: bit-exact
    against the oracle in the device's arithmetic with the screen on."""
    g = load_golden("config2_k30.npz")
    g1 = load_golden("config1.npz")
    host = golden_pocket(g1)
    dp = api.build_pocket(g1["protein_element"], g1["protein_xyz"], [0, 0, 0], 12.0, 0.375, gpu_ctx)
    b = LigandBatch(api.prepare_ligand([str(s) for s in g["smiles"]], quantize=True, ctx=gpu_ctx))
    cfg = abi.ScoringConfig(restarts=30, rescored=30)
    got = api.dock_and_score_batch(dp, b, cfg, gpu_ctx, want_counters=True)
    want = Oracle("port", trig=1).dock_batch(host, b, cfg, nthreads=os.cpu_count() or 8, want_counters=True)
    for f in ("status", "best_score", "scoring_evals", "rotation", "translation"):
        assert np.array_equal(got.results[f], want["results"][f]), f
    assert np.array_equal(got.best_conformation, want["conformation"])
    assert np.array_equal(got.counters, want["counters"])
