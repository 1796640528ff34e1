#!/bin/bash
# A/B kernel experiments: tools/build_variant.sh NAME [-DMACRO=...]...
# builds paper_2309_09131_b200/libflycoo_NAME.so from a scratch copy of csrc
# (PATCH=tools/experiments/X.patch applies an experiment to the copy only);
# select it at run time with FLYCOO_LIB=libflycoo_NAME.so.
set -e
root=$(cd "$(dirname "$0")/.." && pwd)
name=$1; shift
d=/tmp/fcvar_$name
rm -rf "$d"; mkdir -p "$d/pkg" "$d/include"
cp -r "$root/paper_2309_09131_b200/csrc" "$d/pkg/"
rm -f "$d"/pkg/csrc/*.o "$d"/pkg/csrc/*.ptxas.log
cp "$root/include/flycoo.h" "$d/include/"
if [ -n "$PATCH" ]; then (cd "$d/pkg/csrc" && patch -s -p0 < "$root/$PATCH" || patch -s -p5 < "$root/$PATCH"); fi
make -s -C "$d/pkg/csrc" -j5 EXTRA="$*" OUT="$root/paper_2309_09131_b200/libflycoo_$name.so"
grep -A3 "pack_kernelILi0ELi8ELi32" "$d/pkg/csrc/fast_n3.ptxas.log" | grep -E "spill|Used" || true
