#!/bin/bash
# Builds oracle/_ref/libsylkrylov_ref.so from the reference's own Eigen-free
# sources where they lie under /root/reference (no copies in this repo), with the
# reference's Release flags (proj/CMakeLists.txt: -O3 -Wall -Wextra, C++20).
# Skipped silently when /root/reference is absent (GPU boxes use the prebuilt .so).
set -e
HERE="$(cd "$(dirname "$0")" && pwd)"
REF=/root/reference/proj
[ -d "$REF/src" ] || { echo "reference sources absent; skipping"; exit 0; }
mkdir -p "$HERE/_ref"
g++ -std=c++20 -O3 -Wall -Wextra -fPIC -shared -pthread -I"$REF/include" \
    "$REF/src/sparse_matrix.cpp" "$REF/src/parallel.cpp" "$REF/src/problems.cpp" \
    "$REF/src/matrix_market.cpp" "$REF/src/solver_types.cpp" "$HERE/ref_capi.cpp" \
    -o "$HERE/_ref/libsylkrylov_ref.so"
echo "$HERE/_ref/libsylkrylov_ref.so"
# The drop-in check: a caller written against the reference's own headers (unchanged),
# the product's replacement of src/factorized_solvers.cpp, the reference's own Eigen-free
# sources (the .so above) and libsk_b200.so. Built here (needs the reference's headers),
# run by tests/test_dropin.py on the GPU box.
ROOT="$(cd "$HERE/.." && pwd)"
PKG="$ROOT/paper_2605_28274_b200"
if [ -f "$PKG/libsk_b200.so" ]; then
  g++ -std=c++20 -O2 -Wall -Wextra -I"$REF/include" -I"$ROOT/include" \
      "$ROOT/tests/dropin/dropin_caller.cpp" "$PKG/dropin/factorized_solvers_b200.cpp" \
      -L"$HERE/_ref" -lsylkrylov_ref -L"$PKG" -lsk_b200 \
      -Wl,-rpath,'$ORIGIN' -Wl,-rpath,'$ORIGIN/../../paper_2605_28274_b200' \
      -o "$HERE/_ref/dropin_caller"
  echo "$HERE/_ref/dropin_caller"
fi
