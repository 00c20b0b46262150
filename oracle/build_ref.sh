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
    "$REF/src/matrix_market.cpp" "$HERE/ref_capi.cpp" \
    -o "$HERE/_ref/libsylkrylov_ref.so"
echo "$HERE/_ref/libsylkrylov_ref.so"
