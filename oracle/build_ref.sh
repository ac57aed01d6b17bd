#!/usr/bin/env bash
# ORACLE — TEST INFRASTRUCTURE ONLY.
# Compiles the reference's own sources IN PLACE from the read-only tree
# (default /root/reference/proj) into oracle/_ref/ — nothing is copied into
# the repo. Outputs:
#   _ref/libspecden_ref.so   reference specden_core (pool/sharded/operators.cpp)
#                            + oracle/src/ref_capi.cpp (extern "C" wrapper)
#   _ref/test_sharded_core, _ref/test_runtime, _ref/test_operators
#                            the reference's doctest binaries, built against the
#                            shims in oracle/shims (doctest, Eigen, gmpxx)
# Flags follow proj/CMakeLists.txt:8-22 (Release = -O3, -Wall -Wextra, C++20).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF="${REF:-/root/reference/proj}"
OUT="$HERE/_ref"
if [ ! -d "$REF/src" ]; then
  echo "build_ref: reference tree $REF absent; skipping (prebuilt _ref/ is used if present)"
  exit 0
fi
mkdir -p "$OUT"
CXX="${CXX:-g++}"
FLAGS="-std=gnu++20 -O3 -DNDEBUG -fPIC -pthread -w"
SRCS="$REF/src/pool.cpp $REF/src/sharded.cpp $REF/src/operators.cpp"
$CXX $FLAGS -shared -I"$REF/include" -o "$OUT/libspecden_ref.so" $SRCS "$HERE/src/ref_capi.cpp"
GMP="$(ls /usr/lib/x86_64-linux-gnu/libgmp.so.10 2>/dev/null || true)"
for t in test_sharded_core test_runtime test_operators; do
  EXTRA=""
  [ "$t" = test_runtime ] && EXTRA="$GMP"
  $CXX $FLAGS -I"$HERE/shims" -I"$REF/include" -I"$REF/tests" -o "$OUT/$t" \
      "$REF/tests/$t.cpp" "$REF/tests/doctest_main.cpp" $SRCS $EXTRA
done
echo "build_ref: built $OUT"
