#!/usr/bin/env python3
"""Development measurement (not product, not a test): an FP32 instantiation of
the oracle restatement (oracle/vs_oracle.cpp), to MEASURE the premise behind
the FP64 design -- that a search in FP32 arithmetic misses the north_star
tolerances against the reference.

The internal namespace of the oracle is rewritten with `real` = float for
every arithmetic type and float literals; the C ABI stays double (inputs are
converted to float on entry, results back to double).  Trig is glibc's
sinf/cosf (trig mode 0).  Build + run:

    python tools/fp32_oracle/make_fp32.py          # writes and compiles _build/liboracle_fp32.so
    python tools/fp32_oracle/measure.py            # tolerance metrics vs tests/golden/config2_k30.npz
"""
import os
import re
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
src = open(os.path.join(ROOT, "oracle", "vs_oracle.cpp")).read()
cut = src.index('extern "C" {')
head, tail = src[:cut], src[cut:]
head = head.replace("namespace vso {", "namespace vso {\nusing real = float;\n", 1)
head = re.sub(r"\bdouble\b", "real", head)
# float literals: 1.0 -> 1.0f, 1e-9 -> 1e-9f, 0.5 -> 0.5f (not inside identifiers)
head = re.sub(r"(?<![\w.])(\d+\.\d*(?:[eE][-+]?\d+)?|\d+[eE][-+]?\d+)(?![\w.])", r"\1f", head)
# ABI-facing data stays double (pointers into the caller's arrays); values
# are narrowed to float where they enter the arithmetic
head = head.replace("const real *values;", "const double *values;")
head = head.replace("const real *pxyz;", "const double *pxyz;")
head = head.replace("Conf conf_of(const real *xyz, int a0, int a1) {", "Conf conf_of(const double *xyz, int a0, int a1) {")
head = head.replace("c.push_back({xyz[3 * a], xyz[3 * a + 1], xyz[3 * a + 2]});",
                    "c.push_back({(real)xyz[3 * a], (real)xyz[3 * a + 1], (real)xyz[3 * a + 2]});")
tail = tail.replace("std::vector<double> fa(flat_angles", "std::vector<float> fa(flat_angles")
tail = tail.replace("std::vector<double> a(angles + b->torsion_offset[i]", "std::vector<float> a(angles + b->torsion_offset[i]")
# the CR trig helpers are double-only: use float glibc trig in this variant
head = head.replace("vs_crtrig::sincos_cr(angle, &s, &c);", "s = std::sin(angle); c = std::cos(angle);")
out = os.path.join(HERE, "_build")
os.makedirs(out, exist_ok=True)
cpp = os.path.join(out, "vs_oracle_fp32.cpp")
open(cpp, "w").write(head + tail)
cmd = ["g++", "-std=c++20", "-O2", "-fPIC", "-ffp-contract=off", "-fno-fast-math", "-w",
       "-I" + os.path.join(ROOT, "include"), "-shared", "-o", os.path.join(out, "liboracle_fp32.so"), cpp, "-lpthread"]
r = subprocess.run(cmd, capture_output=True, text=True)
if r.returncode:
    print(r.stderr[:6000])
    sys.exit(1)
print("built", os.path.join(out, "liboracle_fp32.so"))
