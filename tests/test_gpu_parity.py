"""GPU parity: every sub-API and the full dock_and_score on the B200, through
the C ABI, against the CPU oracle (device-trig mode -> bit-exact) and the
reference's known answers.  All tests need a GPU."""
from __future__ import annotations

import math
import os

import numpy as np
import pytest

from helpers import explicit_pocket, flat_pocket, pose_at, pyramid_pocket, rel_err
from oracle import Oracle
from paper_2110_11644_b200 import abi, api, synth
from paper_2110_11644_b200.model import Ligand, LigandBatch, Pocket

pytestmark = pytest.mark.gpu
PI = math.pi
THREADS = os.cpu_count() or 8


@pytest.fixture(scope="module")
def env(gpu_ctx):
    el, xyz = synth.synthetic_protein(1200, seed=5, half_box=13.0)
    pocket = api.build_pocket(el, xyz, [0.0, 0.0, 0.0], 8.0, 0.5, gpu_ctx)
    smi = api.synthetic_smiles(192, seed=17, heavy=(14, 34), rot=(0, 8))
    ligs = api.prepare_ligand(smi, quantize=True, ctx=gpu_ctx)
    return gpu_ctx, pocket, pocket.to_host(), LigandBatch(ligs)


# ------------------------------------------------------------------ KATs on GPU
def test_branch_free_sqrt_is_ieee(gpu_ctx):
    """dmath.cuh dsqrt (used for every distance and norm on the device) is
    bit-identical to IEEE sqrt on 3e8 inputs incl. rounding-boundary cases."""
    import ctypes as C
    from paper_2110_11644_b200 import native
    bad = C.c_uint64(0)
    first = C.c_double(0.0)
    rc = native.lib().vs_selftest_sqrt(0, 300_000_000, 20260819, C.byref(bad), C.byref(first))
    assert rc == 0
    assert bad.value == 0, f"first mismatch at x={first.value!r}"


def test_shared_reciprocal_division_is_ieee(gpu_ctx):
    """dmath.cuh drecip/ddiv_r (normalisations in torsion_setup and
    quat_normalized) are bit-identical to IEEE a / b on 3e8 operand pairs."""
    import ctypes as C
    from paper_2110_11644_b200 import native
    bad = C.c_uint64(0)
    first = C.c_double(0.0)
    rc = native.lib().vs_selftest_div(0, 300_000_000, 20260819, C.byref(bad), C.byref(first))
    assert rc == 0
    assert bad.value == 0, f"first mismatch at a={first.value!r}"


def test_trilinear_kats_gpu(gpu_ctx):
    cube = explicit_pocket((2, 2, 2), 1.0, [1, 2, 3, 4, 5, 6, 7, 8])
    v = api.pocket_field_value(cube, [[1, 0, 0], [0, 1, 1], [0.25, 0.5, 0.75], [1, 1, 1], [0.5, 0.5, 1.5],
                                      [-0.5, 0.5, 0.5]], gpu_ctx)
    assert v[0] == 2.0 and v[1] == 7.0 and v[3] == 8.0 and v[4] == -10.0 and v[5] == -10.0
    assert v[2] == pytest.approx(5.25, rel=1e-14)


def test_geo_and_chem_kats_gpu(gpu_ctx):
    cube = explicit_pocket((2, 2, 2), 1.0, [1, 2, 3, 4, 5, 6, 7, 8])
    lig = api.embed_ligand("CCO")
    conf = np.full((9, 3), 50.0)
    conf[:3] = [[0, 0, 0], [1, 0, 0], [0, 1, 1]]
    s, ev = api.geo_score(cube, [lig], conf, gpu_ctx)
    assert s[0] == 10.0 and ev[0] == 3
    one = Ligand("C", np.zeros((1, 3)), np.zeros(1, np.uint8), np.ones(1, np.uint8), np.zeros((0, 2), np.uint16),
                 np.zeros(0, np.uint8), np.zeros(0, np.uint16), [])
    for z, want in ((3.0, 0.4), (4.5, 0.0), (4.0, 0.2), (1.0, 0.4 - 5.0)):
        pk = flat_pocket(2, 1.0, protein=[(0, [0.0, 0.0, z])])
        got = api.chem_score(pk, [one], np.zeros((1, 3)), gpu_ctx)[0]
        assert got == pytest.approx(want, rel=1e-12, abs=0.0 if want == 0.0 else 1e-300)


def test_build_pocket_kats_gpu(gpu_ctx):
    # test_dockengine.cpp:64-135
    dp = api.build_pocket([0], [[0.0, 0.0, 0.0]], [0, 0, 0], 4.0, 0.5, gpu_ctx)
    p = dp.to_host()
    assert p.dims == (17, 17, 17) and np.all(p.origin == -4.0)
    assert p.value_at(10, 8, 8) == -10.0 and p.value_at(14, 8, 8) == 1.0 and p.value_at(0, 0, 0) == 0.0
    prot = np.array([[0.0, 0.0, 0.0], [2.5, 0.0, 0.0]])
    center = np.array([1.0, 0.5, 0.0])
    p2 = api.build_pocket([0, 2], prot, center, 3.0, 0.5, gpu_ctx).to_host()
    idx = np.indices(p2.dims[::-1]).reshape(3, -1)[::-1].T  # (ix, iy, iz) x-fastest
    nodes = p2.origin + p2.spacing * idx
    d = np.min(np.linalg.norm(nodes[:, None, :] - prot[None], axis=2), axis=1)
    want = np.where(d < 1.5, -10.0, np.where((d <= 4.0) & (np.linalg.norm(nodes - center, axis=1) <= 3.0), 1.0, 0.0))
    assert np.array_equal(p2.values, want)
    with pytest.raises(ValueError):
        api.build_pocket([9], [[0, 0, 0]], [0, 0, 0], 4.0, 0.5, gpu_ctx)
    with pytest.raises(ValueError):
        api.build_pocket([0], [[0, 0, 0]], [0, 0, 0], 4.0, 0.2, gpu_ctx)


def test_build_pocket_matches_reference_sources(gpu_ctx):
    from conftest import oracle_kinds
    if "ref" not in oracle_kinds():
        pytest.skip("oracle/_ref not present")
    el, xyz = synth.synthetic_protein()
    g = api.build_pocket(el, xyz, [0, 0, 0], 12.0, 0.375, gpu_ctx).to_host()
    r = Oracle("ref").build_pocket(el, xyz, [0, 0, 0], 12.0, 0.375)
    assert g.dims == (65, 65, 65) and np.array_equal(g.values, r.values)


def test_flatten_kats_gpu(gpu_ctx):
    lig = api.embed_heavy("c1ccccc1")
    conf, ang, st = api.flatten([lig], 20, gpu_ctx)
    assert st[0] == 0 and ang.size == 0 and np.array_equal(conf, lig.xyz)
    port = Oracle("port", trig=1)
    for smi, angles in (("CCCC", [PI]), ("CCCCC", [2 * PI / 3, PI]), ("CCCCCC", [PI, 2 * PI / 3, 4 * PI / 3])):
        l0 = api.embed_heavy(smi)
        pose = np.zeros(1, dtype=abi.POSE_DTYPE)
        pose["rotation"][0] = [0, 0, 0, 1]
        lig = l0.with_xyz(port.materialize(LigandBatch([l0]), np.array(angles), pose))
        c_g, a_g, _ = api.flatten([lig], 20, gpu_ctx)
        c_o, a_o, _ = port.flatten(LigandBatch([lig]))
        assert np.array_equal(c_g, c_o) and np.array_equal(a_g, a_o)


def test_local_search_kats_gpu(gpu_ctx):
    pk = pyramid_pocket(9, 1.0)
    lig = api.parse_smiles("C")
    pose, ang, conf = pose_at(lig, [0.3, 0.7, 1.1])
    pose["geo_score"][0] = api.geo_score(pk, [lig], conf, gpu_ctx)[0][0]
    done, _, _, ev, st = api.local_search(pk, [lig], pose, ang, conf, abi.ScoringConfig(), gpu_ctx)
    assert st[0] == 0 and done["geo_score"][0] > pose["geo_score"][0] + 5.0 and done["geo_score"][0] > 0.95 * 24
    top, tang, tconf = pose_at(lig, pk.box_center())
    top["geo_score"][0] = api.geo_score(pk, [lig], tconf, gpu_ctx)[0][0]
    kept, _, kconf, _, _ = api.local_search(pk, [lig], top, tang, tconf, abi.ScoringConfig(), gpu_ctx)
    assert kept["geo_score"][0] == top["geo_score"][0] and np.array_equal(kconf, tconf)
    flat = flat_pocket(9, 1.0)
    for smi, expect in (("C", 48), ("CCCC", 4 * 14 * 4)):
        l = api.parse_smiles(smi) if smi == "C" else api.embed_ligand(smi)
        p, a, c = pose_at(l, flat.box_center())
        _, _, _, ev, _ = api.local_search(flat, [l], p, a, c, abi.ScoringConfig(), gpu_ctx)
        assert ev[0] == expect


def test_dock_kats_gpu(gpu_ctx):
    # test_dockengine.cpp:696-761
    twin = api.build_pocket([0, 2], [[-2.0, 0, 0], [2.0, 0, 0]], [0, 0, 0], 5.0, 0.5, gpu_ctx)
    lig = api.embed_ligand("CO")
    cfg = abi.ScoringConfig(restarts=16, rescored=5)
    r1 = api.dock_and_score(twin, lig, cfg, gpu_ctx)
    r2 = api.dock_and_score(twin, lig, cfg, gpu_ctx)
    assert r1.best_score == r2.best_score and r1.scoring_evals == r2.scoring_evals and r1.poses_evaluated == 16
    assert np.array_equal(r1.best_pose.conformation, r2.best_pose.conformation) and math.isfinite(r1.best_score)
    assert api.chem_score(twin, [lig], r1.best_pose.conformation, gpu_ctx)[0] == r1.best_score
    for bad in (dict(restarts=0), dict(rescored=0), dict(rmsd_threshold=0.0)):
        with pytest.raises(ValueError):
            api.dock_and_score(twin, lig, abi.ScoringConfig(**bad), gpu_ctx)
    flat = flat_pocket(9, 1.0)
    l4 = api.embed_ligand("CCCC")
    r = api.dock_and_score(flat, l4, abi.ScoringConfig(restarts=8, rescored=3), gpu_ctx)
    assert r.scoring_evals == 8 * 4 * (1 + 4 * (12 + 2 * 1))


# ------------------------------------------------------------------ bit parity vs oracle
def test_sub_apis_bit_exact(env):
    ctx, pocket, host, b = env
    port = Oracle("port", trig=1)
    pts = np.random.default_rng(0).uniform(-10, 10, (50000, 3))
    assert np.array_equal(api.pocket_field_value(pocket, pts, ctx), port.field_values(host, pts))
    shifted = b.xyz + np.array([0.3, -0.6, 0.45])
    g1, e1 = api.geo_score(pocket, b, shifted, ctx)
    g2, e2 = port.geo_score(host, b, shifted)
    assert np.array_equal(g1, g2) and np.array_equal(e1, e2)
    assert np.array_equal(api.chem_score(pocket, b, shifted, ctx), port.chem_score(host, b, shifted))
    raw = LigandBatch(api.prepare_smiles([l.name for l in b.ligands], mode=1))
    c1, a1, s1 = api.flatten(raw, 20, ctx)
    c2, a2, s2 = port.flatten(raw, 20)
    assert np.array_equal(c1, c2) and np.array_equal(a1, a2) and np.array_equal(s1, s2)


def test_flatten_wide_library_and_near_ties_bit_exact(gpu_ctx):
    """k_flatten_dep (candidate-dependent atom sets, filter sums, exact sums
    for near ties) against the oracle's sequential flatten: a wide library
    (0-12 rotors, 8-60 heavy atoms, rigid ligands included) and symmetric
    ligands whose 180/120-degree partners tie up to rounding."""
    smi = api.synthetic_smiles(1500, seed=4242, heavy=(8, 60), rot=(0, 12), grammar=1)
    smi += ["c1ccc(cc1)-c1ccccc1", "CC(C)(C)c1ccc(cc1)C(F)(F)F", "c1ccc(cc1)Cc1ccccc1", "OC(=O)c1ccc(cc1)C(=O)O",
            "c1cc(ccc1Cc1ccc(cc1)Cc1ccccc1)Cc1ccccc1", "FC(F)(F)CCC(F)(F)F", "C1CCC(CC1)CC1CCCCC1"]
    raw = LigandBatch(api.prepare_smiles(smi, mode=1, nthreads=THREADS))
    c1, a1, s1 = api.flatten(raw, 20, gpu_ctx)
    c2, a2, s2 = Oracle("port").flatten(raw, 20, nthreads=THREADS)
    assert np.array_equal(s1, s2)
    assert np.array_equal(c1.view(np.uint64), c2.view(np.uint64)) and np.array_equal(a1, a2)


def _flip_torsion(lig, u):
    """The same ligand with torsion u's bond written the other way round: its
    right set becomes the other side of the bond (the root side)."""
    bonds = lig.bonds.copy()
    bi = int(lig.torsion_bond[u])
    bonds[bi] = bonds[bi][::-1]
    rights = [r.copy() for r in lig.right_sets]
    rights[u] = np.setdiff1d(np.arange(lig.n_atoms, dtype=np.uint16), lig.right_sets[u]).astype(np.uint16)
    return Ligand(lig.name, lig.xyz.copy(), lig.element.copy(), lig.is_heavy.copy(), bonds, lig.bond_order.copy(),
                  lig.torsion_bond.copy(), rights)


def test_flatten_non_rigid_subtrees_bit_exact(gpu_ctx):
    """k_flatten_dep's rigid-subtree mode (D_t x D_t sums taken from candidate
    0 plus a measured residual bound) on ligands where D_t does NOT move
    rigidly: a later torsion written root-side out makes its right set
    straddle t's cut, the residuals are large, and the bound must send the
    decision to the exact sums -- still bit-exact against the oracle."""
    smi = api.synthetic_smiles(300, seed=777, heavy=(20, 50), rot=(3, 10), grammar=1)
    raw = api.prepare_smiles(smi, mode=1, nthreads=THREADS)
    flipped = [_flip_torsion(l, l.n_torsions - 1) for l in raw if l.n_torsions >= 3 and l.n_atoms >= 30]
    assert len(flipped) > 100
    b = LigandBatch(flipped)
    c1, a1, s1 = api.flatten(b, 20, gpu_ctx)
    c2, a2, s2 = Oracle("port").flatten(b, 20, nthreads=THREADS)
    assert np.array_equal(s1, s2)
    assert np.array_equal(c1.view(np.uint64), c2.view(np.uint64)) and np.array_equal(a1, a2)


def test_local_search_random_poses_bit_exact(env):
    ctx, pocket, host, b = env
    port = Oracle("port", trig=1)
    rng = np.random.default_rng(3)
    n = b.n_ligands
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    poses = np.zeros(n, dtype=abi.POSE_DTYPE)
    poses["rotation"] = q
    poses["translation"] = rng.uniform(-2, 2, (n, 3))
    ang = rng.uniform(-3, 3, b.n_torsions_total)
    conf = port.materialize(b, ang, poses)
    poses["geo_score"] = port.geo_score(host, b, conf)[0]
    cfg = abi.ScoringConfig()
    g = api.local_search(pocket, b, poses, ang, conf, cfg, ctx)
    o = port.local_search(host, b, cfg, poses, ang, conf)
    assert np.array_equal(g[4], o[4])
    assert np.array_equal(g[0].view(np.uint8), o[0].view(np.uint8))
    assert np.array_equal(g[1], o[1]) and np.array_equal(g[2], o[2]) and np.array_equal(g[3], o[3])


def test_local_search_node_box_faces_bit_exact(gpu_ctx):
    """k_search's sampler decides "outside the node box" (grid.cpp:63-66) from
    integer floor/ceil conversions (dmath.cuh field_value_fast): translation
    neighbours landing exactly on each face of the box and 2^-40 beyond it,
    starts on the faces, on an f64-grid pocket and on a 3-value (packed 2-bit)
    one, against the oracle's double comparisons; a NaN pose stays NaN."""
    n = 9
    three = np.zeros(n ** 3)
    idx = np.arange(n ** 3)
    three[(idx % n + (idx // n) % n + idx // (n * n)) % 2 == 0] = 1.0
    three[0] = -10.0
    port = Oracle("port", trig=1)
    lig = api.parse_smiles("C")
    assert lig.n_atoms == 1 and np.all(lig.xyz == 0.0)
    eps = 2.0 ** -40
    starts = []
    for axis in range(3):
        for v in (7.0, 7.0 + eps, 1.0, 1.0 - eps, 8.0, 0.0):
            p = np.array([4.0, 4.0, 4.0])
            p[axis] = v
            starts.append(p)
    cfg = abi.ScoringConfig()
    for pk in (pyramid_pocket(n, 1.0), explicit_pocket((n, n, n), 1.0, three)):
        b = LigandBatch([lig] * len(starts))
        poses = np.zeros(len(starts), dtype=abi.POSE_DTYPE)
        poses["rotation"] = [0.0, 0.0, 0.0, 1.0]
        poses["translation"] = starts
        conf = np.array(starts)
        ang = np.zeros(0)
        poses["geo_score"] = port.geo_score(pk, b, conf)[0]
        g = api.local_search(pk, b, poses, ang, conf, cfg, gpu_ctx)
        o = port.local_search(pk, b, cfg, poses, ang, conf)
        assert np.array_equal(g[4], o[4]) and np.array_equal(g[3], o[3])
        assert np.array_equal(g[0].view(np.uint8), o[0].view(np.uint8))
        assert np.array_equal(g[2].view(np.uint64), o[2].view(np.uint64))
        nanpose = poses[:1].copy()
        nanpose["translation"] = [[np.nan, 4.0, 4.0]]
        nconf = np.array([[np.nan, 4.0, 4.0]])
        nanpose["geo_score"] = np.nan
        gn = api.local_search(pk, LigandBatch([lig]), nanpose, ang, nconf, cfg, gpu_ctx)
        on = port.local_search(pk, LigandBatch([lig]), cfg, nanpose, ang, nconf)
        assert np.isnan(gn[0]["geo_score"][0]) and np.isnan(on[0]["geo_score"][0])
        assert np.array_equal(gn[3], on[3]) and np.array_equal(gn[4], on[4])


@pytest.mark.parametrize("k,rescored", [(8, 30), (1, 1), (5, 2), (30, 30)])
def test_dock_bit_exact_vs_oracle(env, k, rescored):
    ctx, pocket, host, b = env
    if k == 30:
        b = LigandBatch(b.ligands[:48])
    cfg = abi.ScoringConfig(restarts=k, rescored=rescored)
    got = api.dock_and_score_batch(pocket, b, cfg, ctx, want_counters=True)
    want = Oracle("port", trig=1).dock_batch(host, b, cfg, nthreads=THREADS, want_counters=True)
    for f in ("status", "best_score", "best_geo_score", "rotation", "translation", "scoring_evals", "poses_evaluated",
              "clash_pairs", "oob_samples", "n_survivors"):
        assert np.array_equal(got.results[f], want["results"][f]), f
    assert np.array_equal(got.best_angles, want["angles"])
    assert np.array_equal(got.best_conformation, want["conformation"])
    assert np.array_equal(got.counters, want["counters"])  # Appendix B work counters, integer-exact


@pytest.mark.parametrize("kw", [
    dict(restarts=6, rescored=6, max_iterations=3),                        # iteration cap
    dict(restarts=6, rescored=4, min_translation=0.001),                    # 10 step levels
    dict(restarts=6, rescored=6, step_torsion=1.0, step_rotation=0.8, step_translation=2.0),  # coarse, arbitrary angles
    dict(restarts=10, rescored=10, rmsd_threshold=0.5),                      # many leaders
    dict(restarts=10, rescored=3, rmsd_threshold=10.0),                      # one leader
    dict(restarts=4, rescored=4, flatten_max_sweeps=1),
    dict(restarts=40, rescored=7),                                           # k > 32: CTA select
])
def test_dock_bit_exact_config_variations(env, kw):
    ctx, pocket, host, b = env
    sub = LigandBatch(b.ligands[:24])
    cfg = abi.ScoringConfig(**kw)
    got = api.dock_and_score_batch(pocket, sub, cfg, ctx, want_counters=True)
    want = Oracle("port", trig=1).dock_batch(host, sub, cfg, nthreads=THREADS, want_counters=True)
    for f in ("status", "best_score", "best_geo_score", "rotation", "translation", "scoring_evals", "clash_pairs",
              "oob_samples", "n_survivors"):
        assert np.array_equal(got.results[f], want["results"][f]), (kw, f)
    assert np.array_equal(got.best_conformation, want["conformation"]), kw
    assert np.array_equal(got.counters, want["counters"]), kw


def test_dock_multi_pocket_equals_single(env):
    """vs_dock_batch_multi (configs[4]: flatten once, search per pocket)
    returns exactly the per-pocket vs_dock_batch results."""
    ctx, pocket, host, b = env
    sub = LigandBatch(b.ligands[:32])
    el, xyz = synth.synthetic_protein(seed=99)
    p2 = api.build_pocket(el, xyz, [0.0, 0.0, 0.0], 9.0, 0.5, ctx)
    cfg = abi.ScoringConfig(restarts=6, rescored=4)
    multi, _, _, _ = api.dock_and_score_multi([pocket, p2, pocket], sub, cfg, ctx)
    for j, pk in enumerate([pocket, p2, pocket]):
        one = api.dock_and_score_batch(pk, sub, cfg, ctx, want_conformation=False).results
        assert np.array_equal(multi[j].view(np.uint8), one.view(np.uint8)), j


def test_dock_default_config_256_restarts(env):
    ctx, pocket, host, b = env
    sub = LigandBatch(b.ligands[:4])
    cfg = abi.ScoringConfig()
    got = api.dock_and_score_batch(pocket, sub, cfg, ctx)
    want = Oracle("port", trig=1).dock_batch(host, sub, cfg, nthreads=THREADS)
    assert np.array_equal(got.results["best_score"], want["results"]["best_score"])
    assert np.array_equal(got.best_conformation, want["conformation"])


@pytest.mark.parametrize("k", [2048, 8192])
def test_dock_restart_counts_beyond_shared_memory(env, k):
    """Restart counts far above the default: k = 2048 keeps the select state
    in shared memory, k = 8192 moves it to global scratch; both bit-exact
    against the oracle (search.cpp:238-276 accepts any restart count)."""
    ctx, pocket, host, b = env
    small = sorted(b.ligands, key=lambda l: (l.n_atoms, l.name))[:2]
    sub = LigandBatch(small)
    cfg = abi.ScoringConfig(restarts=k, rescored=30)
    got = api.dock_and_score_batch(pocket, sub, cfg, ctx)
    want = Oracle("port", trig=1).dock_batch(host, sub, cfg, nthreads=THREADS)
    assert np.array_equal(got.results["status"], want["results"]["status"])
    assert np.array_equal(got.results["best_score"], want["results"]["best_score"])
    assert np.array_equal(got.results["scoring_evals"], want["results"]["scoring_evals"])
    assert np.array_equal(got.best_conformation, want["conformation"])


# ------------------------------------------------------------------ edge cases
def _lig(name, xyz, elem, heavy, bonds=(), orders=None, tors=(), rights=()):
    bonds = np.array(bonds, dtype=np.uint16).reshape(-1, 2)
    return Ligand(name, np.array(xyz, dtype=np.float64).reshape(-1, 3), np.array(elem, np.uint8),
                  np.array(heavy, np.uint8), bonds,
                  np.array(orders if orders is not None else [1] * len(bonds), np.uint8),
                  np.array(tors, np.uint16), [np.array(r, np.uint16) for r in rights])


def test_edge_cases_statuses_and_mixed_batch(env):
    ctx, pocket, host, b = env
    good = b.ligands[:6]
    empty = _lig("empty", np.zeros((0, 3)), [], [])
    only_h = _lig("H2", [[0, 0, 0], [0.74, 0, 0]], [9, 9], [0, 0], bonds=[(0, 1)])
    degenerate = _lig("deg", [[0, 0, 0], [1, 0, 0], [1, 0, 0], [2, 1, 0]], [0, 0, 0, 0], [1, 1, 1, 1],
                      bonds=[(0, 1), (1, 2), (2, 3)], tors=[1], rights=[[2, 3]])
    bad_bond = _lig("badbond", [[0, 0, 0], [1.5, 0, 0], [3, 0, 0]], [0, 0, 0], [1, 1, 1],
                    bonds=[(0, 1), (1, 2)], tors=[7], rights=[[2]])
    bad_atom = _lig("badatom", [[0, 0, 0], [1.5, 0, 0], [3, 0, 0]], [0, 0, 0], [1, 1, 1],
                    bonds=[(0, 1), (1, 2)], tors=[1], rights=[[2, 9]])
    n_big = 300
    big = _lig("big", np.random.default_rng(0).normal(size=(n_big, 3)) * 5, [0] * n_big, [1] * n_big)
    rigid = api.prepare_ligand("c1ccccc1", quantize=True, ctx=ctx)
    mixed = [good[0], empty, good[1], only_h, degenerate, good[2], bad_bond, bad_atom, big, rigid, good[3]]
    mb = LigandBatch(mixed)
    cfg = abi.ScoringConfig(restarts=6, rescored=4)
    got = api.dock_and_score_batch(pocket, mb, cfg, ctx)
    st = got.results["status"]
    assert st[1] == abi.VS_LIG_EMPTY
    assert st[3] == abi.VS_LIG_NO_HEAVY
    assert st[4] == abi.VS_LIG_DEGENERATE_AXIS
    assert st[6] == abi.VS_LIG_BAD_TORSION and st[7] == abi.VS_LIG_BAD_TORSION
    assert st[8] == abi.VS_LIG_TOO_LARGE
    ok = [0, 2, 5, 9, 10]
    assert np.all(st[ok] == 0)
    port = Oracle("port", trig=1)
    want = port.dock_batch(host, LigandBatch([mixed[i] for i in ok]), cfg, nthreads=THREADS)
    assert np.array_equal(got.results["best_score"][ok], want["results"]["best_score"])
    # the oracle reports the same failures for the failing ligands
    wbad = port.dock_batch(host, LigandBatch([empty, only_h, degenerate, bad_bond, bad_atom]), cfg)
    assert np.array_equal(wbad["results"]["status"],
                          [abi.VS_LIG_EMPTY, abi.VS_LIG_NO_HEAVY, abi.VS_LIG_DEGENERATE_AXIS, abi.VS_LIG_BAD_TORSION,
                           abi.VS_LIG_BAD_TORSION])
    # single-ligand API raises like the reference (InvalidArgument)
    with pytest.raises(ValueError):
        api.dock_and_score(pocket, degenerate, cfg, ctx)
    # no heavy atoms but a single restart: no RMSD is ever needed -> docks
    r1 = api.dock_and_score_batch(pocket, [only_h], abi.ScoringConfig(restarts=1, rescored=1), ctx)
    w1 = port.dock_batch(host, LigandBatch([only_h]), abi.ScoringConfig(restarts=1, rescored=1))
    assert r1.results["status"][0] == 0 and r1.results["best_score"][0] == w1["results"]["best_score"][0]


def test_flatten_degenerate_axis_in_each_phase(gpu_ctx):
    """A degenerate torsion axis is reported whichever k_flatten_dep phase
    meets it first: the candidates' own torsion (per-candidate build), a
    later torsion whose axis moves with the candidate, or a later
    candidate-independent torsion (warp 0's common pass); same status as
    the oracle."""
    # torsion 0 on bond (1,2), right {2,3}; torsion 1 on bond (0,4), whose
    # endpoints coincide and do not move with torsion 0 (independent)
    indep = _lig("indep", [[0, 0, 0], [1, 0, 0], [2, 0, 0], [2, 1, 0], [0, 0, 0], [-1, 1, 0]], [0] * 6, [1] * 6,
                 bonds=[(0, 1), (1, 2), (2, 3), (0, 4), (4, 5)], tors=[1, 3], rights=[[2, 3], [4, 5]])
    # torsion 1 on bond (2,3) inside right(0): its axis moves with torsion 0
    dep = _lig("dep", [[0, 0, 0], [1, 0, 0], [2, 0, 0], [2, 0, 0], [3, 1, 0]], [0] * 5, [1] * 5,
               bonds=[(0, 1), (1, 2), (2, 3), (3, 4)], tors=[1, 2], rights=[[2, 3, 4], [3, 4]])
    fine = api.prepare_smiles(["CCCCOc1ccccc1"], mode=1)[0]
    raw = LigandBatch([indep, fine, dep])
    _, _, s1 = api.flatten(raw, 20, gpu_ctx)
    _, _, s2 = Oracle("port").flatten(raw, 20)
    assert s1[0] == abi.VS_LIG_DEGENERATE_AXIS and s1[2] == abi.VS_LIG_DEGENERATE_AXIS and s1[1] == 0
    assert np.array_equal(s1, s2)


def test_large_flexible_ligands(env):
    ctx, pocket, host, _ = env
    smi = api.synthetic_smiles(12, seed=123, heavy=(55, 80), rot=(10, 15))
    ligs = api.prepare_ligand(smi, quantize=True, ctx=ctx)
    b = LigandBatch(ligs)
    cfg = abi.ScoringConfig(restarts=4, rescored=4)
    got = api.dock_and_score_batch(pocket, b, cfg, ctx)
    want = Oracle("port", trig=1).dock_batch(host, b, cfg, nthreads=THREADS)
    assert np.all(got.results["status"] == 0)
    assert np.array_equal(got.results["best_score"], want["results"]["best_score"])
    assert np.array_equal(got.best_conformation, want["conformation"])


def test_flatten_legacy_path_for_very_large_ligands(env):
    """Ligands whose k_flatten_dep candidate buffer would exceed 200 KB of
    shared memory (N > ~216 atoms) run the legacy one-thread-per-candidate
    k_flatten; a batch mixing them with small ligands stays bit-exact."""
    ctx, pocket, host, _ = env
    big = "C1CCC(CC1)" * 13 + "C1CCCCC1"  # 14 cyclohexanes, 13 torsions, 226 atoms
    smi = [big, "CCCCOc1ccccc1", big.replace("C1CCCCC1", "c1ccccc1")]
    raw = LigandBatch(api.prepare_smiles(smi, mode=1, nthreads=THREADS))
    assert raw.ligands[0].n_atoms > 216
    c1, a1, s1 = api.flatten(raw, 20, ctx)
    c2, a2, s2 = Oracle("port").flatten(raw, 20, nthreads=THREADS)
    assert np.all(s1 == 0) and np.array_equal(s1, s2)
    assert np.array_equal(c1.view(np.uint64), c2.view(np.uint64)) and np.array_equal(a1, a2)


# ------------------------------------------------------------------ golden + tolerance
@pytest.mark.parametrize("name", ["config1.npz", "config2_k30.npz", "config3_cells.npz"])
def test_golden_reference_parity_gpu(gpu_ctx, name):
    """north_star parity against the REFERENCE's own results (oracle/_ref
    fixtures, tests/golden/make_golden.py) on every ligand of the fixture:
    config 1 (k=4), the benched configs[1] library (k=30, 1,200 ligands) and
    the configs[2] size-sweep cells (k=30).  Tolerances (north_star): best
    score within 1e-3 relative and best-pose heavy-atom RMSD <= 0.1 A for
    >= 99.9% of ligands, identical top-K up to printed-score ties, equal
    statuses, scoring_evals equal for >= 99.9%.  The GPU is also checked bit
    for bit against the oracle in its own arithmetic on the whole fixture."""
    import json
    from helpers import assert_north_star, golden_parity, golden_pocket, load_golden
    g = load_golden(name)
    g1 = load_golden("config1.npz")
    host = golden_pocket(g1)
    dp = api.build_pocket(g1["protein_element"], g1["protein_xyz"], [0, 0, 0], 12.0, 0.375, gpu_ctx)
    assert np.array_equal(dp.to_host().values, host.values)
    smi = [str(s) for s in g["smiles"]]
    ligs = api.prepare_ligand(smi, quantize=True, ctx=gpu_ctx, nthreads=THREADS)
    b = LigandBatch(ligs)
    assert np.array_equal(b.xyz, g["prepared_xyz"])  # GPU prepare_ligand == reference prepare_ligand
    cfg = abi.ScoringConfig(restarts=int(g["restarts"]), rescored=int(g["rescored"]))
    got = api.dock_and_score_batch(dp, b, cfg, gpu_ctx)
    rep = golden_parity(g, b, got.results, got.best_conformation)
    want = Oracle("port", trig=1).dock_batch(host, b, cfg, nthreads=THREADS)
    rep["bit_exact_vs_oracle_device_arith"] = float(np.mean(
        (got.results["best_score"] == want["results"]["best_score"])
        & (got.results["scoring_evals"] == want["results"]["scoring_evals"])))
    rep["fixture"] = name
    print("golden parity", json.dumps(rep))
    out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")
    if os.path.isdir(out):
        with open(os.path.join(out, "golden_parity.jsonl"), "a") as f:
            f.write(json.dumps(rep) + "\n")
    assert_north_star(rep)
    assert np.array_equal(got.results["best_score"], want["results"]["best_score"])
    assert np.array_equal(got.results["scoring_evals"], want["results"]["scoring_evals"])
    assert np.array_equal(got.best_conformation, want["conformation"])


def test_full_size_properties(env):
    ctx, pocket, host, _ = env
    smi = api.synthetic_smiles(4096, seed=2024)
    ligs = api.prepare_ligand(smi, quantize=True, ctx=ctx)
    b = LigandBatch(ligs)
    cfg = abi.ScoringConfig(restarts=30, rescored=30)
    r1 = api.dock_and_score_batch(pocket, b, cfg, ctx, want_counters=True)
    r2 = api.dock_and_score_batch(pocket, b, cfg, ctx)
    assert np.all(r1.results["status"] == 0)
    assert np.array_equal(r1.results["best_score"], r2.results["best_score"])  # deterministic
    assert np.all(np.isfinite(r1.results["best_score"]))
    # the reported pose is the canonical materialisation of (angles, transform)
    port = Oracle("port", trig=1)
    poses = np.zeros(b.n_ligands, dtype=abi.POSE_DTYPE)
    poses["rotation"] = r1.results["rotation"]
    poses["translation"] = r1.results["translation"]
    again = port.materialize(b, r1.best_angles, poses)
    assert np.array_equal(again, r1.best_conformation)
    # best_score is the chem score of the best pose; best_geo its geo score
    assert np.array_equal(api.chem_score(pocket, b, r1.best_conformation, ctx), r1.results["best_score"])
    assert np.array_equal(api.geo_score(pocket, b, r1.best_conformation, ctx)[0], r1.results["best_geo_score"])
    assert np.array_equal(r1.counters[:, 0], r1.results["scoring_evals"])
    n = np.array([l.heavy_atom_count() for l in ligs])
    m = np.array([l.n_torsions for l in ligs])
    S = r1.results["scoring_evals"].astype(np.int64)
    # S = n * (k + sum_iters (12 + 2m)): the sweep count is an integer
    assert np.all((S - 30 * n) % (n * (12 + 2 * m)) == 0)


def test_cpp_dropin_program(gpu_ctx):
    """C++ written against the reference's API (include/vscreen) runs on the B200 build."""
    import subprocess
    exe = os.path.join(os.path.dirname(__file__), "cpp", "_build", "test_dropin")
    assert os.path.exists(exe), "build() compiles tests/cpp/test_dropin.cpp"
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ALL OK" in r.stdout, r.stdout + r.stderr
