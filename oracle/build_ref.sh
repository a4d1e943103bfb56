#!/usr/bin/env bash
# TEST INFRASTRUCTURE: compiles the UNMODIFIED reference sources in place
# (/root/reference/proj/src, read-only) against the from-scratch Eigen subset
# into oracle/_ref/libref_lamfast.so.  Does not run the reference's own CMake
# build.  Flags follow the reference's Release build (CMakeLists.txt:6-8,
# src/CMakeLists.txt:15): -O3 -DNDEBUG, no -march.  bench.cpp is left out: it
# needs nlohmann/json and is not on the assembly path.
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
repo="$(dirname "$here")"
ref="${LAMFAST_REFERENCE:-/root/reference/proj}"
out="$here/_ref"
if [ ! -d "$ref/src" ]; then
    echo "build_ref: $ref not present; keeping prebuilt $out" >&2
    exit 0
fi
mkdir -p "$out"
srcs=""
for f in splines quadrature geometry materials assembly fast sparse voigt_free; do
    srcs="$srcs $ref/src/$f.cpp"
done
g++ -std=c++20 -O3 -DNDEBUG -fPIC -shared -pthread \
    -I"$repo/include/eigen_subset" -I"$ref/include" -I"$ref/src" -I"$repo/include" \
    $srcs "$here/ref_capi.cpp" -o "$out/libref_lamfast.so.tmp"
mv "$out/libref_lamfast.so.tmp" "$out/libref_lamfast.so"
echo "build_ref: wrote $out/libref_lamfast.so"
