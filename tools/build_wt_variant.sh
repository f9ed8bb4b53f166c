#!/bin/bash
# Build the engine from the WORKING TREE into variants/$1.so (A/B timing on one
# box: FG_LIB=variants/$1.so selects it).  Extra make args: EXTRA="-DFOO=1".
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
wt=/tmp/fg_wt_$name
rm -rf "$wt"; mkdir -p "$wt/paper_1206_6857_b200"
cp -r "$root/include" "$wt/"
mkdir -p "$wt/paper_1206_6857_b200/csrc"
cp "$root"/paper_1206_6857_b200/csrc/*.cu "$root"/paper_1206_6857_b200/csrc/*.cuh "$root"/paper_1206_6857_b200/csrc/Makefile "$wt/paper_1206_6857_b200/csrc/"
mkdir -p "$root/variants"
make -s -j8 -C "$wt/paper_1206_6857_b200/csrc" OUT="$root/variants/$name.so" BUILD="$wt/build" "$@" > /dev/null
echo "built variants/$name.so from the working tree"
