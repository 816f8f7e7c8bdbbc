#!/usr/bin/env bash
# Build the UNMODIFIED reference library from its sources where they lie under
# /root/reference (read-only; nothing is copied into this repo) plus our C-ABI
# shim into oracle/_ref/libfractime_ref.so.  Flags are the reference's own CMake
# Release build (proj/CMakeLists.txt: C++20, CMAKE_BUILD_TYPE Release -> -O3
# -DNDEBUG, no -march: the x86-64 baseline ISA, so no FMA contraction -- the
# results stay bitwise equal to the oracle's restatement, tests/test_oracle.py).
# The output directory oracle/_ref/ is git-ignored but travels to the GPU box.
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
ref="${FRACTIME_REFERENCE:-/root/reference/proj}"
out="$here/_ref"
if [ ! -d "$ref/src" ]; then
  echo "build_ref: $ref not present; keeping prebuilt $out" >&2
  exit 0
fi
mkdir -p "$out"
srcs=(weights fft toeplitz krylov schemes harness)
objs=()
for s in "${srcs[@]}"; do
  o="$out/$s.o"
  if [ ! -f "$o" ] || [ "$ref/src/$s.cpp" -nt "$o" ]; then
    g++ -std=c++20 -O3 -DNDEBUG -fPIC -I"$ref/include" -c "$ref/src/$s.cpp" -o "$o"
  fi
  objs+=("$o")
done
g++ -std=c++20 -O2 -fPIC -I"$ref/include" -c "$here/ref_shim.cpp" -o "$out/ref_shim.o"
g++ -shared -o "$out/libfractime_ref.so" "${objs[@]}" "$out/ref_shim.o" -lpthread
echo "build_ref: built $out/libfractime_ref.so"
