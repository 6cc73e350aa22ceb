#!/usr/bin/env bash
# A/B of the search stage with and without the FP32 screen (run under gpurun).
set -uo pipefail
cd "$(dirname "$0")/.."
TAG=${1:-ab}
mkdir -p gpurun_out
VS_SCREEN=1 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_$TAG.log 2>&1; echo "pytest exit $?" >> gpurun_out/gpu_tests_$TAG.log
VS_SCREEN=1 VSDOCK_DEBUG=1 python bench.py --steps ${STEPS:-3} --warmup 3 --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
VS_SCREEN=0 python bench.py --steps ${STEPS:-3} --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_noscr.json 2> gpurun_out/bench_${TAG}_noscr.err
python - "$TAG" <<'PY'
import json, sys
t = sys.argv[1]
for f in (f"gpurun_out/bench_{t}.json", f"gpurun_out/bench_{t}_noscr.json"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d["value"]), {k: round(v, 1) for k, v in d["stage_ms_per_step"].items()})
    except Exception as e:
        print(f, "failed", e)
PY
tail -1 gpurun_out/gpu_tests_$TAG.log
