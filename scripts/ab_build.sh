#!/bin/bash
# Build the library of git revision $1 (. = working tree) into
# exp/$2/libmerbit_b200.so, extra nvcc flags $3 (kernel
# A/B experiments: MBX_LIB_PATH=exp/$2/libmerbit_b200.so selects it).
set -e
rev=$1; name=$2
root=$(cd "$(dirname "$0")/.." && pwd)
dst=$root/exp/$name
rm -rf "$dst"; mkdir -p "$dst"
if [ "$rev" = "." ]; then  # the working tree
  mkdir -p "$dst/paper_2605_07391_b200"
  cp -r "$root/include" "$dst/"
  mkdir -p "$dst/paper_2605_07391_b200/csrc"
  cp "$root"/paper_2605_07391_b200/csrc/*.cu "$root"/paper_2605_07391_b200/csrc/*.h "$root"/paper_2605_07391_b200/csrc/*.cpp "$root"/paper_2605_07391_b200/csrc/Makefile "$dst/paper_2605_07391_b200/csrc/"
else
  (cd "$root" && git archive "$rev" paper_2605_07391_b200/csrc include) | tar -x -C "$dst"
fi
make -s -j8 -C "$dst/paper_2605_07391_b200/csrc" OUT="$dst/libmerbit_b200.so" EXTRA="$3"
rm -rf "$dst/paper_2605_07391_b200/csrc/build"
echo "$dst/libmerbit_b200.so"
