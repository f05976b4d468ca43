#!/bin/bash
# TEST INFRASTRUCTURE: the reference's own acceptance suite (proj/tests/
# acceptance.cpp, unmodified) compiled against the reference's own core
# objects (oracle/_ref/*.o, built by `make -C oracle ref` from the sources
# where they lie) and run on the CPU here. Its stdout is the golden file
# tests/test_gpu_reference_suite.py compares the B200 drop-in's run with.
set -euo pipefail
HERE=$(cd "$(dirname "$0")" && pwd)
ROOT=$(cd "$HERE/../.." && pwd)
REF_ROOT=${REF_ROOT:-/root/reference/proj}
make -C "$ROOT/oracle" ref >/dev/null
OUT=${TMPDIR:-/tmp}/cb_acceptance_ref
mkdir -p "$OUT"
g++ -std=c++20 -O2 -ffp-contract=off -I"$ROOT/tests/cpp/doctest" -I"$REF_ROOT/include" \
  -I"$REF_ROOT/tests" "$REF_ROOT/tests/acceptance.cpp" \
  $(ls "$ROOT"/oracle/_ref/*.o | grep -v ref_capi) -o "$OUT/acceptance" -lpthread
"$OUT/acceptance" > "$HERE/acceptance_reference.txt"
