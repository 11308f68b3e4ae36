#!/bin/bash
# Build a variant of libeplab_b200.so with extra nvcc defines for tools/ab_libs.sh:
#   bash tools/ab_build.sh <name> "-DEPLAB_CNR=2 ..."   -> tools/_ab/<name>.so
set -e
cd "$(dirname "$0")/../paper_2604_19241_b200/csrc"
mkdir -p ../../tools/_ab
make -j16 BUILD=build_ab_$1 OUT=../../tools/_ab/$1.so EXTRA="$2" > /dev/null
