#!/bin/bash
# A/B builds of libprb.so with compile-time knobs, for gpurun comparisons:
#   profiles/build_variant.sh <name> "<-D flags>"  ->  profiles/ab/libprb_<name>.so
# (select one at run time with PRB_LIB_PATH=profiles/ab/libprb_<name>.so)
# OVERRIDE="file.cu=/path/to/other.cu ..." swaps sources in the copy (e.g. a previous revision)
set -e
name=$1; flags=$2
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=$(mktemp -d)
mkdir -p "$tmp/csrc" "$tmp/include" "$root/profiles/ab"
cp "$root"/paper_2112_05923_b200/csrc/*.cu "$root"/paper_2112_05923_b200/csrc/*.h "$root"/paper_2112_05923_b200/csrc/*.cuh \
   "$root"/paper_2112_05923_b200/csrc/Makefile "$tmp/csrc/"
cp -r "$root"/include/* "$tmp/include/"
for o in $OVERRIDE; do cp "${o#*=}" "$tmp/csrc/${o%%=*}"; done
# the sources include ../../include/prb.h: mirror that depth
mkdir -p "$tmp/a/b" && mv "$tmp/csrc" "$tmp/a/b/csrc" && mkdir -p "$tmp/a/include" && cp -r "$tmp/include"/* "$tmp/a/include/"
make -s -C "$tmp/a/b/csrc" -j16 NVFLAGS_EXTRA="$flags" >/dev/null
cp "$tmp/a/b/libprb.so" "$root/profiles/ab/libprb_$name.so"
rm -rf "$tmp"
echo "built profiles/ab/libprb_$name.so ($flags)"
