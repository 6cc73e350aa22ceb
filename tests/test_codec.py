"""The ligand record stream (binary_codec.hpp:18-24) on the B200 path:
host encoding and framing against the reference's own encode_record, GPU
decode (vs_decode_records) against the reference's decode_record, including
every CodecError case in the reference's check order (binary_codec.cpp:165-222,
ligand.cpp:52-56, 110-124)."""
import struct

import numpy as np
import pytest

from oracle import Oracle, available
from paper_2110_11644_b200 import api

pytestmark_ref = pytest.mark.skipif(not available("ref"), reason="oracle/_ref not built")

SMILES = ["CCO", "c1ccccc1CCN", "CC(C)C(=O)O", "c1ccc(cc1)-c1ccccc1", "NC(=O)CC1CCc2c(cccc2C1)Cc1ccncc1",
          "OCC1CCNCC1", "C"]


@pytest.fixture(scope="module")
def ref():
    if not available("ref"):
        pytest.skip("oracle/_ref not built")
    return Oracle("ref")


def _ref_stream(ref, smiles, mode=0):
    return b"".join(ref.encode_prepared(s, mode, True) for s in smiles)


@pytestmark_ref
def test_encode_matches_reference_bytes(ref):
    for mode in (0, 1, 2):
        data = _ref_stream(ref, SMILES, mode)
        offs, at, ligs = [], 0, []
        while at < len(data):
            lig, nxt = ref.decode_record(data, at)
            offs.append(at)
            ligs.append(lig)
            at = nxt
        assert api.encode_records(ligs, [l.name for l in ligs]) == data
        assert list(api.frame_records(data)) == offs


def _lig_equal(a, b):
    assert a.name == b.name
    assert np.array_equal(a.xyz.view(np.uint64), b.xyz.view(np.uint64))
    assert np.array_equal(a.element, b.element) and np.array_equal(a.is_heavy, b.is_heavy)
    assert np.array_equal(a.bonds, b.bonds) and np.array_equal(a.bond_order, b.bond_order)
    assert np.array_equal(a.torsion_bond, b.torsion_bond)
    assert len(a.right_sets) == len(b.right_sets)
    for x, y in zip(a.right_sets, b.right_sets):
        assert np.array_equal(np.asarray(x, dtype=np.int64), np.asarray(y, dtype=np.int64))


@pytest.mark.gpu
def test_gpu_decode_matches_reference(gpu_ctx, ref):
    smi = api.synthetic_smiles(400, seed=77, heavy=(8, 40), rot=(0, 9)) + SMILES
    data = api.XSLB_HEADER + _ref_stream(ref, smi, 0)
    offs = api.frame_records(data, start=len(api.XSLB_HEADER))
    assert len(offs) == len(smi)
    ligs, status, errors = api.decode_records(data, offs, gpu_ctx)
    assert np.all(status == 0), [e for e in errors if e][:3]
    for o, lig in zip(offs, ligs):
        want, _ = ref.decode_record(data, int(o))
        _lig_equal(lig, want)


def _corrupt_cases(ref):
    """(name, record bytes, expected vs_record_status) for each CodecError."""
    base = ref.encode_prepared("CC(C)C(=O)O", 2, True)  # torsion on bond 2
    name_len = struct.unpack_from("<H", base, 6)[0]
    q = 8 + name_len
    na, nb, nt = struct.unpack_from("<HHH", base, q)
    pa = q + 6
    pb = pa + 14 * na
    pt = pb + 5 * nb
    cases = []

    def mut(f):
        b = bytearray(base)
        f(b)
        return bytes(b)
    cases.append(("element", mut(lambda b: b.__setitem__(pa + 14 * 1 + 12, 11)), 4))
    cases.append(("nonfinite", mut(lambda b: struct.pack_into("<f", b, pa + 14 * 2 + 4, float("nan"))), 5))
    cases.append(("element before nan", mut(lambda b: (struct.pack_into("<f", b, pa, float("inf")),
                                                       b.__setitem__(pa + 12, 200))), 4))
    cases.append(("bond index", mut(lambda b: struct.pack_into("<H", b, pb + 5 * 1, na)), 6))
    cases.append(("self bond", mut(lambda b: struct.pack_into("<HH", b, pb, 1, 1)), 6))
    cases.append(("bond order", mut(lambda b: b.__setitem__(pb + 5 * 2 + 4, 5)), 7))
    cases.append(("torsion index", mut(lambda b: struct.pack_into("<H", b, pt, nb)), 8))
    # bond 1 (C1-C2) -> (C1-O5) closes the cycle C1-C3-O5 through the torsion
    # bond C1-C3: not a bridge (found before the now-disconnected C2)
    cases.append(("not a bridge", mut(lambda b: struct.pack_into("<HH", b, pb + 5 * 1, 1, 5)), 9))
    cases.append(("length", mut(lambda b: struct.pack_into("<I", b, 2, struct.unpack_from("<I", b, 2)[0] - 1)), 3))
    return base, cases


@pytest.mark.gpu
def test_gpu_decode_codec_errors_like_reference(gpu_ctx, ref):
    base, cases = _corrupt_cases(ref)
    for name, rec, code in cases:
        data = rec + base  # a valid record after the corrupt one
        if code == 3:
            offs = [0]
        else:
            offs = [0, len(rec)]
        ligs, status, errors = api.decode_records(data, offs, gpu_ctx)
        with pytest.raises(ValueError) as e:
            ref.decode_record(data, 0)
        assert status[0] == code, (name, status[0], errors[0], str(e.value))
        assert errors[0] == str(e.value), (name, errors[0], str(e.value))
        if len(offs) > 1:
            assert status[1] == 0 and ligs[1] is not None


@pytest.mark.gpu
def test_gpu_decode_disconnected_and_framing(gpu_ctx, ref):
    # two records glued into one: a graph with two components
    a = ref.encode_prepared("CCO", 2, True)
    b = ref.encode_prepared("CN", 2, True)
    la, _ = ref.decode_record(a, 0)
    lb, _ = ref.decode_record(b, 0)
    from paper_2110_11644_b200.model import Ligand
    na = len(la.element)
    glued = Ligand("glued", np.concatenate([la.xyz, lb.xyz]), np.concatenate([la.element, lb.element]),
                   np.concatenate([la.is_heavy, lb.is_heavy]), np.concatenate([la.bonds, lb.bonds + na]),
                   np.concatenate([la.bond_order, lb.bond_order]), np.zeros(0, np.uint16), [])
    data = api.encode_records([glued], ["glued"])
    ligs, status, errors = api.decode_records(data, [0], gpu_ctx)
    with pytest.raises(ValueError) as e:
        ref.decode_record(data, 0)
    assert status[0] == 10 and errors[0] == str(e.value)
    # bad marker and truncated record are framing failures
    _, status, _ = api.decode_records(b"\x00\x00" + a, [0], gpu_ctx)
    assert status[0] == 1
    _, status, _ = api.decode_records(a[:-3], [0], gpu_ctx)
    assert status[0] == 2
    assert list(api.frame_records(a + b[:-1])) == [0]


@pytest.mark.gpu
def test_gpu_dock_records_equals_decode_then_dock(gpu_ctx, ref):
    """vs_dock_records (decode into the dock path's device inputs) gives the
    results of decode_records + dock_and_score_batch, record for record; a
    corrupt record in the stream only fails itself."""
    from paper_2110_11644_b200 import abi, synth
    el, xyz = synth.synthetic_protein()
    pocket = api.build_pocket(el, xyz, [0.0, 0.0, 0.0], 12.0, 0.375, gpu_ctx)
    smi = api.synthetic_smiles(40, seed=5)
    ligs = api.prepare_ligand(smi, quantize=True, ctx=gpu_ctx)
    data = bytearray(api.encode_records(ligs))
    offs = list(api.frame_records(bytes(data)))
    bad = 7  # an invalid element code in record 7
    name_len = struct.unpack_from("<H", data, offs[bad] + 6)[0]
    data[offs[bad] + 8 + name_len + 6 + 12] = 77
    data = bytes(data)
    cfg = abi.ScoringConfig(restarts=6, rescored=4)
    res, rst, _, _ = api.dock_records([pocket], data, offs, cfg, gpu_ctx)
    assert rst[bad] == 4 and res[0][bad]["status"] == abi.VS_LIG_BAD_RECORD
    dec, status, _ = api.decode_records(data, offs, gpu_ctx)
    good = [i for i in range(len(offs)) if i != bad]
    want = api.dock_and_score_batch(pocket, [dec[i] for i in good], cfg, gpu_ctx, want_conformation=False).results
    assert np.array_equal(res[0][good].view(np.uint8), want.view(np.uint8))
