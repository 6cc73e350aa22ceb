mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_r2j.log 2>&1; echo "pytest exit $?" >> gpurun_out/gpu_tests_r2j.log
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r2j.json 2> gpurun_out/bench_r2j.err
VS_NO_FUSED_SELECT=1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r2j_nofuse.json 2> gpurun_out/bench_r2j_nofuse.err
