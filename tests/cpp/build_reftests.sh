#!/usr/bin/env bash
# Compiles the reference's OWN unit suites, unmodified, from where they lie
# (/root/reference/proj/tests, read-only) against the B200 drop-in headers
# (include/lamfast) and libraries (liblamfast.so over liblamfast_b200.so),
# with the from-scratch doctest subset (tests/cpp/doctest_subset) and Eigen
# subset (include/eigen_subset).  Output: build/reftests/unit_tests (git-
# ignored, travels to the GPU box, where tests/test_reftests.py runs it).
#
# Included: the unit_tests target of tests/CMakeLists.txt minus
# test_bench.cpp, which tests the sweep harness (BenchConfig / runBench /
# JSON configs: SURVEY.md §2, out of scope).  acceptance.cpp needs runBench
# too and is restated in tests/test_gpu_acceptance.py instead.
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
repo="$(cd "$here/../.." && pwd)"
ref="${LAMFAST_REFERENCE:-/root/reference/proj}/tests"
out="$repo/build/reftests"
if [ ! -d "$ref" ]; then
    echo "build_reftests: $ref not present; keeping prebuilt $out" >&2
    exit 0
fi
mkdir -p "$out"
libdir="$repo/paper_1905_05417_b200/lib"
objs=""
for f in unit_main test_splines test_quadrature test_geometry test_materials test_sparse test_assembly test_fast test_voigt_free; do
    g++ -std=c++20 -O2 -Wall -Wextra -w -I"$here/doctest_subset" -I"$repo/include" -I"$repo/include/eigen_subset" \
        -c "$ref/$f.cpp" -o "$out/$f.o" &
    objs="$objs $out/$f.o"
done
wait
g++ $objs -L"$libdir" -llamfast -llamfast_b200 -Wl,-rpath,"\$ORIGIN/../../paper_1905_05417_b200/lib" \
    -o "$out/unit_tests.tmp"
mv "$out/unit_tests.tmp" "$out/unit_tests"
echo "build_reftests: wrote $out/unit_tests"
