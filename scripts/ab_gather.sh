#!/bin/bash
# A/B of K2 builds (exp/NAME/libmerbit_b200.so, "base" = in-tree) on C1,
# s24 SpMV (natural, relabelled, f64) and the s24 PageRank iteration,
# interleaved so clock drift hits every variant alike.
for round in 1 2; do
  for v in "$@"; do
    if [ "$v" = base ]; then unset MBX_LIB_PATH; else export MBX_LIB_PATH=exp/$v/libmerbit_b200.so; fi
    echo "== $v round $round"
    python scripts/prof/spmv_iter.py 20 f32 300 0 0 | sed 's/.*: /c1: /'
    python scripts/prof/spmv_iter.py 24 f32 50 1 0 | sed 's/.*: /s24 nat: /'
    python scripts/prof/spmv_iter.py 24 f32 50 1 1 | sed 's/.*: /s24 rel: /'
    python scripts/prof/spmv_iter.py 24 f64 50 1 1 | sed 's/.*: /s24 rel f64: /'
    python scripts/prof/pr_iter.py 24 20 5 | tail -1
  done
done
