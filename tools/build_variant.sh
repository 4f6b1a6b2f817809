#!/bin/bash
# Dev: build the library with extra compile flags into tools/_var/<name>/lib.so
#   tools/build_variant.sh NAME "EXTRA FLAGS" [make vars...]
set -e
name=$1; shift
extra=$1; shift
here=$(cd "$(dirname "$0")" && pwd)
out=$here/_var/$name
mkdir -p "$out"
make -s -j8 -C "$here/../paper_1210_0800_b200/csrc" OBJDIR="/tmp/xqr_var_obj/$name" LIB="$out/lib.so" EXTRA="$extra" "$@" 2>&1 | grep -E "error|mgs_cta_kernelINS_8mgs_pair" || true
ls -la "$out/lib.so"
