#!/usr/bin/env bash
# Compile the reference's hot-path + input-side sources UNCHANGED, where they
# lie under /root/reference, against the Eigen-subset restatement
# (third_party/eigen_subset) into oracle/_ref/libvsref.so.  Nothing from the
# reference is copied into this repository; the output is git-ignored.
# The reference's own build (CMake + Eigen3 + vendored doctest/CLI11) is not
# used: it cannot run here (no Eigen, no vendor/ tree, no network).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF="${1:-/root/reference/proj}"
if [ ! -d "$REF/src" ]; then
  echo "build_ref: $REF not present; keeping any prebuilt oracle/_ref" >&2
  exit 0
fi
mkdir -p "$HERE/_ref/obj"
SRCS="dockengine/chem dockengine/grid dockengine/search dockengine/pocket_io
      geometry/transform geometry/embed geometry/hydrogens
      molmodel/ligand molmodel/binary_codec molmodel/smiles pipeline/pipeline pipeline/io workflow/merge"
FLAGS=(-std=c++20 -O3 -fPIC -w -I"$HERE/../third_party/eigen_subset" -I"$REF/include" -I"$HERE/../include")
pids=()
for s in $SRCS; do
  o="$HERE/_ref/obj/$(echo "$s" | tr / _).o"
  ${CXX:-g++} "${FLAGS[@]}" -c "$REF/src/$s.cpp" -o "$o" & pids+=($!)
done
${CXX:-g++} "${FLAGS[@]}" -c "$HERE/ref_capi.cpp" -o "$HERE/_ref/obj/ref_capi.o" & pids+=($!)
for p in "${pids[@]}"; do wait "$p"; done
${CXX:-g++} -shared -o "$HERE/_ref/libvsref.so" "$HERE"/_ref/obj/*.o -lpthread
rm -rf "$HERE/_ref/obj"
echo "build_ref: wrote $HERE/_ref/libvsref.so"
