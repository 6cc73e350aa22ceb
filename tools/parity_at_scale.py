#!/usr/bin/env python3
"""Parity at scale (measurement, not a test): the first N ligands of the benched
library stream (configs[1], k=30, rescored=30) docked by the reference's own
code (oracle/_ref, all host threads) and by the B200, compared with the
north_star metrics of tests/helpers.golden_parity.  Both arms prepare their
inputs with the reference's prepare_ligand (+ quantize_to_wire).

    python tools/parity_at_scale.py [N]
"""
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
from helpers import golden_parity  # noqa: E402
from oracle import Oracle  # noqa: E402
from paper_2110_11644_b200 import abi, api, synth  # noqa: E402
from paper_2110_11644_b200.model import LigandBatch  # noqa: E402


def main(n):
    threads = os.cpu_count() or 8
    ref = Oracle("ref")
    el, xyz = synth.synthetic_protein()
    host = ref.build_pocket(el, xyz, [0, 0, 0], 12.0, 0.375)
    smi = api.synthetic_smiles(n, seed=20260820)
    with ThreadPoolExecutor(threads) as ex:
        ligs = list(ex.map(lambda s: ref.prepare(s, 0, True), smi))
    b = LigandBatch(ligs)
    cfg = abi.ScoringConfig(restarts=30, rescored=30)
    t = time.time()
    want = ref.dock_batch(host, b, cfg, nthreads=threads)
    t_ref = time.time() - t
    ctx = api.default_context(0)
    dp = api.build_pocket(el, xyz, [0, 0, 0], 12.0, 0.375, ctx)
    assert np.array_equal(dp.to_host().values, host.values)
    got = api.dock_and_score_batch(dp, b, cfg, ctx)
    r = want["results"]
    g = {"smiles": np.array(smi), "status": r["status"], "best_score": r["best_score"],
         "scoring_evals": r["scoring_evals"], "best_conf": want["conformation"].astype(np.float32)}
    rep = golden_parity(g, b, got.results, got.best_conformation, k_top=1000)
    rep.update({"config": "configs[1] bench stream seed 20260820, k=30, rescored=30", "reference_seconds": t_ref,
                "reference_threads": threads})
    print(json.dumps(rep))


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 20000)
