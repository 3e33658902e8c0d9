#!/usr/bin/env bash
# ORACLE — builds oracle/_ref/libscreloc_ref.so from the REFERENCE's own sources where they
# lie (/root/reference/proj: rng.hpp, geometry.hpp, features.hpp, src/features.cpp,
# src/geometry.cpp) against the local minimal Eigen shim. Nothing is copied into the repo;
# the output goes to oracle/_ref/ (git-ignored). Only run where /root/reference exists.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF="${REFERENCE_ROOT:-/root/reference}/proj"
OUT="$HERE/../_ref"
mkdir -p "$OUT"
g++ -std=c++20 -O2 -ffp-contract=off -fPIC -shared -w \
    -I "$HERE/eigen_shim" -I "$REF/include" \
    "$REF/src/features.cpp" "$REF/src/geometry.cpp" "$HERE/ref_driver.cpp" \
    -o "$OUT/libscreloc_ref.so"
echo "$OUT/libscreloc_ref.so"
