"""One pipeline rank on the B200 (include/vs_rank.h):
vs_run_rank's rows and counters equal the reference's own run_rank
(pipeline.cpp:297-389, compiled from its sources into oracle/_ref) on an
.xslb image with undecodable records, false sync markers and a ligand whose
dock fails -- for whole files, slabs, tiny chunks and batches (speculative
framing discarded after a bad record), and several CUDA workers."""
from __future__ import annotations

import struct

import numpy as np
import pytest

from oracle import Oracle, available
from paper_2110_11644_b200 import abi, api, synth

pytestmark = pytest.mark.skipif(not available("ref"), reason="oracle/_ref not built")


def record_spans(data: bytes, start: int = 8):
    """(offset, length) of each record along the length chain."""
    out, at = [], start
    while at + 6 <= len(data) and data[at] == 0xD0 and data[at + 1] == 0xC5:
        n = 6 + struct.unpack_from("<I", data, at + 2)[0]
        out.append((at, n))
        at += n
    return out


def corrupt_library(ref, n: int = 60, seed: int = 17):
    """A small .xslb image: header + n records with (1) an invalid element
    code in record 7 (decode fails: records_skipped), (2) 40 junk bytes with
    a false sync marker after record 20, (3) a degenerate torsion axis in
    record 33 (decodes, the dock fails: dock_errors)."""
    smi = api.synthetic_smiles(n, seed=seed, heavy=(14, 24), rot=(1, 6))
    ligs = [ref.prepare(s, 0, True) for s in smi]
    body = bytearray(api.encode_records(ligs, smi))
    spans = record_spans(bytes(api.XSLB_HEADER + body), 8)
    spans = [(o - 8, l) for o, l in spans]
    # (1) element code of atom 0 of record 7
    o, _ = spans[7]
    name_len = struct.unpack_from("<H", body, o + 6)[0]
    body[o + 8 + name_len + 6 + 12] = 200
    # (3) torsion 0 of record 33: put atom b on atom a
    o, _ = spans[33]
    name_len = struct.unpack_from("<H", body, o + 6)[0]
    na, nb, nt = struct.unpack_from("<HHH", body, o + 8 + name_len)
    assert nt >= 1
    atoms = o + 8 + name_len + 6
    bonds = atoms + 14 * na
    tors = bonds + 5 * nb
    bi = struct.unpack_from("<H", body, tors)[0]
    a, b = struct.unpack_from("<HH", body, bonds + 5 * bi)
    body[atoms + 14 * b: atoms + 14 * b + 12] = body[atoms + 14 * a: atoms + 14 * a + 12]
    # (2) junk with a false marker after record 20
    o, l = spans[20]
    junk = bytes([0xD0, 0xC5, 0xFF, 0x7F, 0, 0]) + bytes(range(34))
    body[o + l:o + l] = junk
    return bytes(api.XSLB_HEADER + body)


@pytest.fixture(scope="module")
def setup():
    ref = Oracle("ref")
    el, xyz = synth.synthetic_protein(1200, seed=5, half_box=13.0)
    pocket = ref.build_pocket(el, xyz, [0, 0, 0], 8.0, 0.5)
    data = corrupt_library(ref)
    cfg = abi.ScoringConfig(restarts=6, rescored=6)
    return ref, pocket, data, cfg


def test_reference_rank_sees_the_injected_faults(setup):
    ref, pocket, data, cfg = setup
    text, c = ref.run_rank(data, pocket, cfg)
    assert c["records_skipped"] == 1 and c["dock_errors"] == 1
    # record 20's length chain hops onto the false marker, whose own hop
    # lands on junk: the 2-hop rule (binary_codec.cpp:89-111) rejects record
    # 20 as a start, silently -- 60 - 1 skipped - 1 dock error - 1 unframed
    assert c["rows_written"] == 57 and len(text.splitlines()) == 57


def test_plan_slabs_matches_reference_rule():
    assert api.plan_slabs(10, 3) == [(0, 3), (3, 6), (6, 10)]
    assert api.plan_slabs(7, 1) == [(0, 7)]
    with pytest.raises(ValueError):
        api.plan_slabs(7, 0)


@pytest.mark.gpu
@pytest.mark.parametrize("kw", [dict(), dict(batch_records=7, chunk_bytes=512), dict(batch_records=3, chunk_bytes=97,
                                                                                       workers_per_device=3)])
def test_gpu_rank_equals_reference_rank(gpu_ctx, setup, kw):
    ref, pocket, data, cfg = setup
    want, wc = ref.run_rank(data, pocket, cfg)
    got, st = api.run_rank(data, pocket, cfg, devices=[0], **kw)
    assert got == want
    for k in ("ligands_docked", "records_skipped", "dock_errors", "rows_written"):
        assert st[k] == wc[k], (k, st[k], wc[k])
    assert st["bytes_read"] == len(data)


@pytest.mark.gpu
def test_gpu_slabs_equal_reference_slabs(gpu_ctx, setup):
    ref, pocket, data, cfg = setup
    got_all, want_all = [], []
    for slab in api.plan_slabs(len(data), 3):
        want, _ = ref.run_rank(data, pocket, cfg, slab=slab, chunk_bytes=333)
        got, _ = api.run_rank(data, pocket, cfg, slab=slab, devices=[0], batch_records=5, chunk_bytes=333)
        assert got == want, slab
        got_all.append(got)
        want_all.append(want)
    whole, _ = ref.run_rank(data, pocket, cfg)
    assert "".join(got_all) == whole  # merge_outputs of the rank files == one rank


@pytest.mark.gpu
def test_gpu_rank_corrupt_tail_fails_like_reference(gpu_ctx, setup):
    ref, pocket, data, cfg = setup
    bad = data + bytes([0xD0, 0xC5, 0x01])
    with pytest.raises(ValueError, match="corrupt record stream"):
        ref.run_rank(bad, pocket, cfg)
    with pytest.raises(ValueError, match="corrupt record stream"):
        api.run_rank(bad, pocket, cfg, devices=[0])


@pytest.mark.gpu
def test_gpu_rank_over_two_devices(gpu_ctx, setup):
    """The CUDA workers of one rank spread over two GPUs (W per device); rows
    and counters are unchanged (skipped on a one-GPU box)."""
    from paper_2110_11644_b200 import native
    if native.lib().vs_device_count() < 2:
        pytest.skip("needs two GPUs")
    ref, pocket, data, cfg = setup
    want, wc = ref.run_rank(data, pocket, cfg)
    got, st = api.run_rank(data, pocket, cfg, devices=[0, 1], batch_records=6, workers_per_device=2)
    assert got == want and st["workers"] == 4
    assert st["rows_written"] == wc["rows_written"] and st["records_skipped"] == wc["records_skipped"]


@pytest.mark.gpu
def test_gpu_rank_k40_and_default_config(gpu_ctx, setup):
    """k > 32 (the CTA select) and the reference's default ScoringConfig
    (k=256, rescored=30) through the rank pipeline, against the reference's
    own run_rank on the first 12 records."""
    ref, pocket, data, _ = setup
    spans = record_spans(data, 8)
    small = data[:spans[12][0]]
    for cfg in (abi.ScoringConfig(restarts=40, rescored=7), abi.ScoringConfig()):
        want, wc = ref.run_rank(small, pocket, cfg)
        got, st = api.run_rank(small, pocket, cfg, devices=[0], batch_records=5)
        assert got == want
        assert st["records_skipped"] == wc["records_skipped"] == 1
