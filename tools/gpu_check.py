"""Ad-hoc GPU parity + timing probe (development tool, run under gpurun)."""
from __future__ import annotations

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from oracle import Oracle  # noqa: E402
from paper_2110_11644_b200 import abi, api, synth  # noqa: E402
from paper_2110_11644_b200.model import LigandBatch  # noqa: E402


def main():
    n_par = int(os.environ.get("NPAR", "64"))
    n_time = int(os.environ.get("NTIME", "4096"))
    k_par = int(os.environ.get("KPAR", "8"))
    ctx = api.default_context(0)
    t = time.time()
    el, xyz = synth.synthetic_protein()
    pocket = api.build_pocket(el, xyz, [0, 0, 0], 12.0, 0.375, ctx)
    print("pocket build", time.time() - t, pocket.info()[2], synth.voxel_mix(pocket.to_host().values))
    host = pocket.to_host()
    if os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libvsref.so")):
        ref = Oracle("ref")
        rp = ref.build_pocket(el, xyz, [0, 0, 0], 12.0, 0.375)
        print("build_pocket == ref:", np.array_equal(rp.values, host.values))
    smi = api.synthetic_smiles(n_par, seed=11)
    t = time.time()
    ligs = api.prepare_ligand(smi, quantize=True, ctx=ctx)
    print("prepare_ligand", n_par, time.time() - t)
    b = LigandBatch(ligs)
    port = Oracle("port")
    # flatten parity (CR trig)
    port.set_trig_mode(1)
    c_o, a_o, s_o = port.flatten(b, 20)
    c_g, a_g, s_g = api.flatten(b, 20, ctx)
    print("flatten conf equal:", np.array_equal(c_o, c_g), "angles equal:", np.array_equal(a_o, a_g))
    # field values
    pts = np.random.default_rng(0).uniform(-13, 13, (20000, 3))
    print("field equal:", np.array_equal(port.field_values(host, pts), api.pocket_field_value(pocket, pts, ctx)))
    g_o, e_o = port.geo_score(host, b, b.xyz)
    g_g, e_g = api.geo_score(pocket, b, b.xyz, ctx)
    print("geo equal:", np.array_equal(g_o, g_g), np.array_equal(e_o, e_g))
    shifted = b.xyz + np.array([0.5, -0.3, 0.2])
    ch_o = port.chem_score(host, b, shifted)
    ch_g = api.chem_score(pocket, b, shifted, ctx)
    print("chem equal:", np.array_equal(ch_o, ch_g), float(np.max(np.abs(ch_o - ch_g))))
    cfg = api.ScoringConfig(restarts=k_par, rescored=min(k_par, 30))
    t = time.time()
    want = port.dock_batch(host, b, cfg, nthreads=os.cpu_count() or 8, want_counters=True)
    tcpu = time.time() - t
    t = time.time()
    got = api.dock_and_score_batch(pocket, b, cfg, ctx)
    tgpu = time.time() - t
    rs_o, rs_g = want["results"], got.results
    eq = rs_o["best_score"] == rs_g["best_score"]
    print(f"dock k={k_par}: bit-equal best_score {eq.sum()}/{len(eq)}; evals equal",
          np.array_equal(rs_o["scoring_evals"], rs_g["scoring_evals"]),
          "conf equal", np.array_equal(want["conformation"], got.best_conformation),
          "status", np.unique(rs_g["status"]), f"cpu {tcpu:.2f}s gpu {tgpu:.2f}s")
    if not eq.all():
        bad = np.nonzero(~eq)[0][:5]
        print("first mismatches", bad, rs_o["best_score"][bad], rs_g["best_score"][bad], rs_o["scoring_evals"][bad],
              rs_g["scoring_evals"][bad])
    port.set_trig_mode(0)
    want0 = port.dock_batch(host, b, cfg, nthreads=os.cpu_count() or 8)
    rel = np.abs(want0["results"]["best_score"] - rs_g["best_score"]) / np.maximum(1e-12, np.abs(want0["results"]["best_score"]))
    print("vs glibc oracle: bit-equal", int((want0["results"]["best_score"] == rs_g["best_score"]).sum()),
          "within 1e-3 rel", int((rel <= 1e-3).sum()), "of", len(rel))
    # timing
    smi = api.synthetic_smiles(n_time, seed=12)
    ligs = api.prepare_ligand(smi, quantize=True, ctx=ctx)
    bt = LigandBatch(ligs)
    cfg30 = api.ScoringConfig(restarts=30, rescored=30)
    api.dock_and_score_batch(pocket, LigandBatch(ligs[:256]), cfg30, ctx)
    t = time.time()
    r = api.dock_and_score_batch(pocket, bt, cfg30, ctx)
    wall = time.time() - t
    print(f"timing: {n_time} ligands k=30: wall {wall:.3f}s kernel {r.kernel_ms:.1f}ms -> {n_time / wall:.0f} lig/s wall,"
          f" {n_time / (r.kernel_ms / 1e3):.0f} lig/s kernel; status {np.unique(r.results['status'])};"
          f" evals/lig {r.results['scoring_evals'].mean():.0f}")
    c = want["counters"]
    print("oracle counters mean (k=%d):" % k_par, c.mean(axis=0))


if __name__ == "__main__":
    main()
