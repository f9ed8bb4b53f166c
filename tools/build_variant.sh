#!/bin/bash
# Build the engine at git ref $1 into variants/$2.so (A/B timing on one box:
# FG_LIB=variants/$2.so selects it).  Extra make args: EXTRA="-DFOO=1".
set -e
ref=$1; name=$2; shift 2
root=$(cd "$(dirname "$0")/.." && pwd)
wt=/tmp/fg_variant_$name
rm -rf "$wt"; mkdir -p "$wt"
git -C "$root" archive "$ref" paper_1206_6857_b200/csrc include | tar -x -C "$wt"
mkdir -p "$root/variants"
make -s -j8 -C "$wt/paper_1206_6857_b200/csrc" OUT="$root/variants/$name.so" BUILD=/tmp/fg_variant_build_$name "$@" > /dev/null
echo "built variants/$name.so from $ref"
