#!/usr/bin/env bash
# Profile the dock path on one B200 (run under gpurun).  Writes into
# gpurun_out/: plain.log, launches.csv (per-launch device times), prof.ncu-rep
# (full set for k_search and k_flatten).
set -uo pipefail
cd "$(dirname "$0")/.."
TAG=${1:-r01}
CMD="python bench.py --batch ${BATCH:-16384} --steps 1 --warmup 1 --no-cpu-baseline"
mkdir -p gpurun_out
$CMD > gpurun_out/plain_$TAG.log 2>&1 || { echo "plain run failed"; tail gpurun_out/plain_$TAG.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD \
  > gpurun_out/ncu_launches_$TAG.log 2>&1
# the largest k_search launch of the timed step (skip the warm-up step's
# launches and the small bucket), then one k_flatten of a timed step
ncu --set full --clock-control none --import-source on -k regex:"k_search" -s ${SKIP_SEARCH:-1} -c 1 \
  -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_flatten" -s 2 -c 1 \
  -o gpurun_out/prof_flat_$TAG $CMD > gpurun_out/ncu_flat_$TAG.log 2>&1
echo "profile done"; tail -3 gpurun_out/ncu_full_$TAG.log
