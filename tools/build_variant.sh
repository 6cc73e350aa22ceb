#!/usr/bin/env bash
# Build an A/B variant of libvsdock.so with extra -D flags (development only):
#   tools/build_variant.sh NAME "-DVS_FLAT_UNROLL=16 ..."
# -> paper_2110_11644_b200/_lib/var/NAME.so ; select it with VSDOCK_LIB=...
set -euo pipefail
cd "$(dirname "$0")/../paper_2110_11644_b200/csrc"
NAME=$1; DEFS=${2:-}
OBJ=../_lib/var/obj_$NAME; mkdir -p $OBJ
NVFLAGS="-gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -fmad=false -Xcompiler -fPIC,-ffp-contract=off,-O2 -I../../include"
rm -f $OBJ/*.o
pids=()
for f in kernels search driver peaks codec; do
  /usr/local/cuda/bin/nvcc $NVFLAGS $DEFS -c cuda/$f.cu -o $OBJ/$f.o & pids+=($!)
done
g++ -std=c++17 -O2 -fPIC -ffp-contract=off -fno-fast-math -Wall -I../../include -c host/prep.cpp -o $OBJ/prep.o & pids+=($!)
g++ -std=c++17 -O2 -fPIC -ffp-contract=off -fno-fast-math -Wall -I../../include -c host/synth.cpp -o $OBJ/synth.o & pids+=($!)
g++ -std=c++17 -O2 -fPIC -ffp-contract=off -fno-fast-math -Wall -pthread -I../../include -c host/rank.cpp -o $OBJ/rank.o & pids+=($!)
g++ -std=c++17 -O2 -fPIC -ffp-contract=off -fno-fast-math -Wall -pthread -I../../include -c host/merge.cpp -o $OBJ/merge.o & pids+=($!)
for p in "${pids[@]}"; do wait $p || { echo "variant $NAME: compile failed"; exit 1; }; done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o ../_lib/var/$NAME.so \
  $OBJ/kernels.o $OBJ/search.o $OBJ/driver.o $OBJ/peaks.o $OBJ/codec.o $OBJ/prep.o $OBJ/synth.o $OBJ/rank.o $OBJ/merge.o -lpthread
echo "built _lib/var/$NAME.so"
