#!/bin/bash
# build_variant.sh NAME "NVCC defines": the product library with extra nvcc flags into dbg/libNAME.so (A/B experiments)
set -e
R=$(cd "$(dirname "$0")/.." && pwd)
mkdir -p "$R/dbg"
make -C "$R/paper_1805_11144_b200" -j16 BUILD="$R/paper_1805_11144_b200/build_$1" LIB="$R/dbg/lib$1.so" NVEXTRA="$2" "$R/dbg/lib$1.so" > "$R/dbg/build_$1.log" 2>&1
echo "built dbg/lib$1.so"
