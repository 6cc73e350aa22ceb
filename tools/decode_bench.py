#!/usr/bin/env python3
"""Record decode throughput: the bench library
encoded as an .xslb stream, decoded on the GPU (vs_decode_records, end to end
from host bytes to a host ligand set) and by the reference's decode_record
(oracle/_ref, one host thread, bounded sample)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "oracle"))

from paper_2110_11644_b200 import api  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
    ctx = api.default_context(0)
    ligs = api.prepare_ligand(api.synthetic_smiles(n, seed=20260820), quantize=True, ctx=ctx)
    data = api.XSLB_HEADER + api.encode_records(ligs)
    t0 = time.perf_counter()
    offs = api.frame_records(data, start=len(api.XSLB_HEADER))
    t_frame = time.perf_counter() - t0
    import ctypes as C
    import numpy as np
    from paper_2110_11644_b200 import abi, native
    L = native.lib()
    buf = np.frombuffer(data, dtype=np.uint8)
    o64 = np.ascontiguousarray(offs, dtype=np.int64)

    def raw():  # the C ABI call alone: host bytes in, host ligand set out
        h = C.c_void_p()
        native.check(L.vs_decode_records(ctx.handle, abi.ptr(buf, C.c_uint8), len(data), abi.ptr(o64, C.c_int64),
                                         len(o64), C.byref(h)), "vs_decode_records")
        L.vs_ligand_set_free(h)
    raw()  # warm-up
    t0 = time.perf_counter()
    raw()
    t_raw = time.perf_counter() - t0
    t0 = time.perf_counter()
    out, status, _ = api.decode_records(data, offs, ctx)
    t_dec = time.perf_counter() - t0
    line = {"records": len(offs), "bytes": len(data), "frame_s": t_frame,
            "gpu_decode_abi_s": t_raw, "gpu_decode_records_per_s": len(offs) / t_raw,
            "python_objects_s": t_dec, "ok": int((status == 0).sum())}
    try:
        from oracle import Oracle, available
        if available("ref"):
            ref = Oracle("ref")
            k = min(2000, len(offs))
            t0 = time.perf_counter()
            ends = list(offs[1:k + 1]) + [len(data)]
            recs = [data[int(o):int(e)] for o, e in zip(offs[:k], ends[:k])]
            for r in recs:
                ref.decode_record(r, 0)
            dt = time.perf_counter() - t0
            line["reference_decode_records_per_s_1thread"] = k / dt
            line["reference_sample"] = k
    except Exception as e:  # pragma: no cover
        line["reference"] = repr(e)
    print(json.dumps(line))


if __name__ == "__main__":
    main()
