#!/usr/bin/env bash
# Builds the reference's OWN doctest suites (proj/tests/test_sharded_core.cpp,
# test_runtime.cpp, test_operators.cpp + doctest_main.cpp), compiled IN PLACE
# and UNCHANGED from the read-only tree, against the C++ drop-in
# include/specden/ (whose specden/*.hpp module headers forward to
# specden_b200.hpp) and linked with paper_2505_11564_b200/libspecden_b200.so
# -- nothing of the reference library is linked. The doctest/Eigen/gmpxx
# headers the suites include come from oracle/shims (test infrastructure).
# Outputs oracle/_ref/dropin/<suite> (git-ignored; travels to the GPU box,
# where tests/test_dropin_gpu.py runs them on the device).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
ROOT="$(cd "$HERE/.." && pwd)"
REF="${REF:-/root/reference/proj}"
OUT="$HERE/_ref/dropin"
if [ ! -d "$REF/tests" ]; then
  echo "build_dropin_tests: reference tree $REF absent; skipping (prebuilt binaries are used if present)"
  exit 0
fi
mkdir -p "$OUT"
CXX="${CXX:-g++}"
CUDA="${CUDA_HOME:-/usr/local/cuda}"
LIBDIR="$ROOT/paper_2505_11564_b200"
GMP="$(ls /usr/lib/x86_64-linux-gnu/libgmp.so.10 2>/dev/null || true)"
for t in test_sharded_core test_runtime test_operators; do
  EXTRA=""
  [ "$t" = test_runtime ] && EXTRA="$GMP"
  $CXX -std=gnu++20 -O2 -pthread -w -I"$ROOT/include" -I"$HERE/shims" -I"$REF/tests" -I"$CUDA/include" \
      -o "$OUT/$t" "$REF/tests/$t.cpp" "$REF/tests/doctest_main.cpp" $EXTRA \
      -L"$LIBDIR" -lspecden_b200 -L"$CUDA/lib64" -lcudart \
      -Wl,-rpath,"\$ORIGIN/../../../paper_2505_11564_b200" -Wl,-rpath,"$CUDA/lib64"
done
echo "build_dropin_tests: built $OUT"
