#!/usr/bin/env bash
# TEST INFRASTRUCTURE: builds the C restatement (the checker) into
# oracle/liblamfast_oracle.so.  -ffp-contract=off: no FMA contraction, like
# the reference's baseline x86-64 Release build.
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
repo="$(dirname "$here")"
gcc -std=c11 -O2 -ffp-contract=off -fopenmp -fPIC -shared -I"$repo/include" \
    "$here/lamfast_oracle.c" -o "$here/liblamfast_oracle.so.tmp" -lm
mv "$here/liblamfast_oracle.so.tmp" "$here/liblamfast_oracle.so"
echo "build_oracle: wrote $here/liblamfast_oracle.so"
