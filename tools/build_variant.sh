#!/bin/bash
# Builds an A/B variant of the CUDA library with extra nvcc flags:
#   tools/build_variant.sh NAME "-DLF_..."  ->  build/var/NAME/liblamfast_b200.so
# (select it with LAMFAST_LIB=build/var/NAME/liblamfast_b200.so)
set -e
cd "$(dirname "$0")/../paper_1905_05417_b200/csrc"
name=$1; shift
mkdir -p ../../build/var/$name
make -j4 BUILD=../../build/var/$name OUT=../../build/var/$name/liblamfast_b200.so EXTRA="$*" ../../build/var/$name/liblamfast_b200.so > ../../build/var/$name/build.log 2>&1 || { tail -20 ../../build/var/$name/build.log; exit 1; }
echo "built build/var/$name"
