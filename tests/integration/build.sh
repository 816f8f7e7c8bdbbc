#!/usr/bin/env bash
# Build tests/integration/_build/ref_binding: INTEGRATION.md's maintainer-side
# bindings compiled against the reference's own headers (read in place under
# /root/reference, never copied) and linked with the unmodified reference
# library (oracle/_ref, oracle/build_ref.sh) and libfractime_b200.so.
# TEST INFRASTRUCTURE; _build/ is git-ignored but travels to the GPU box.
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
root="$(cd "$here/../.." && pwd)"
ref="${FRACTIME_REFERENCE:-/root/reference/proj}"
out="$here/_build"
if [ ! -d "$ref/include" ]; then
  echo "integration: $ref not present; keeping prebuilt $out" >&2
  exit 0
fi
[ -f "$root/oracle/_ref/libfractime_ref.so" ] || bash "$root/oracle/build_ref.sh"
mkdir -p "$out"
g++ -std=c++20 -O2 -I"$ref/include" -I"$root/include" "$here/ref_binding.cpp" -o "$out/ref_binding" \
  -L"$root/oracle/_ref" -lfractime_ref -L"$root/paper_1710_11593_b200" -l:libfractime_b200.so \
  -Wl,-rpath,'$ORIGIN/../../../oracle/_ref' -Wl,-rpath,'$ORIGIN/../../../paper_1710_11593_b200' -lpthread
echo "integration: built $out/ref_binding"
