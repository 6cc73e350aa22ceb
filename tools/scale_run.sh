#!/usr/bin/env bash
# Weak-scaling lines on one box (run under gpurun --gpus 4): N = 1, 2, 4 and
# the reference arm at N = 4, JSON lines into gpurun_out/.
cd "$(dirname "$0")/.."
TAG=${1:-r01}
python bench.py > gpurun_out/scale1_$TAG.json 2> gpurun_out/scale1_$TAG.err
for n in 2 4; do
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus $n > gpurun_out/scale${n}_$TAG.json 2> gpurun_out/scale${n}_$TAG.err
done
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --impl reference --gpus 4 > gpurun_out/ref4_$TAG.json 2> gpurun_out/ref4_$TAG.err
for f in scale1 scale2 scale4 ref4; do echo $f; tail -c 400 gpurun_out/${f}_$TAG.json; echo; done
