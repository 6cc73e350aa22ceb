cd /root/repo
A="--batch 32768 --steps 2 --warmup 3 --no-cpu-baseline"
run() { name=$1; shift; env "$@" timeout 600 python bench.py $A > gpurun_out/ab_$name.json 2> gpurun_out/ab_$name.err; python - $name <<'PY'
import json,sys
n=sys.argv[1]
try:
  d=json.loads(open(f'gpurun_out/ab_{n}.json').read().strip().splitlines()[-1]); print(n, round(d['value']), {k:round(v,2) for k,v in d['stage_ms_per_step'].items()}, d['results']['mean_best_score'])
except Exception as e: print(n,'FAIL',e)
PY
}
run cs20 VSDOCK_CHEM_CELL=2.0
run nocut VSDOCK_LIB=paper_2110_11644_b200/_lib/var/nocut.so
run cs15 VSDOCK_CHEM_CELL=1.5
run cs10 VSDOCK_CHEM_CELL=1.0
run cs075 VSDOCK_CHEM_CELL=0.75
VSDOCK_CHEM_CELL=1.0 timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
