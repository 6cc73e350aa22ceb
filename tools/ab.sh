#!/usr/bin/env bash
# A/B the variants in _lib/var on one GPU (run under gpurun):
#   tools/ab.sh "fu4 fu8 fu16" [bench args]
cd "$(dirname "$0")/.."
VARS=$1; shift
ARGS=${*:---batch 32768 --steps 2 --warmup 3 --no-cpu-baseline}
mkdir -p gpurun_out
for v in $VARS; do
  if [ "$v" = base ]; then lib=""; else lib=paper_2110_11644_b200/_lib/var/$v.so; fi
  VSDOCK_LIB=$lib timeout 600 python bench.py $ARGS > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
  python - "$v" gpurun_out/ab_$v.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print(sys.argv[1], "value %.0f" % d["value"], "stages", {k: round(v, 1) for k, v in d["stage_ms_per_step"].items()},
          "mean_best %.6f" % d["results"]["mean_best_score"])
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
done
