#!/usr/bin/env bash
# compute-sanitizer passes over the hot path (run on a GPU box, from the repo
# root): memcheck, racecheck (shared memory), synccheck and initcheck of
# __graft_entry__.smoke() (TILE K1, SpMV K2/K3, fused PageRank graph), then
# memcheck and synccheck of the small-matrix SpMV / PageRank / TILE (+ BiCGSTAB,
# comparators: synccheck) parity tests.
# Logs go to gpurun_out/sanitize_*.log; the summary line of each is printed.
set -u
mkdir -p gpurun_out
# 32 mbarriers per K2 CTA in the fp64 TMA staging mode: synccheck's default
# tracking table overflows ("overflow of tracked cuda::barrier structures")
CS="compute-sanitizer --error-exitcode 99 --print-limit 20 --num-cuda-barriers 64"
SMOKE='import __graft_entry__ as g; g.smoke()'
# synccheck runs the PageRank loop as an unrolled graph: inside a conditional
# (WHILE) graph node it reports barrier divergence and aborts the same kernels
# that are clean in eager and unrolled replays -- a tool limitation, like
# ncu's: scripts/debug/synccheck_while_repro.cu reproduces it with a textbook
# block reduction (clean eagerly, "divergent thread(s) in warp" at its
# __syncthreads as the body of a WHILE node; profiles/r2_sanitizers.md)
for tool in memcheck racecheck synccheck initcheck; do
  mode=while; [ $tool = synccheck ] && mode=unrolled
  MBX_GRAPH_MODE=$mode timeout 900 $CS --tool $tool python -c "$SMOKE" > gpurun_out/sanitize_smoke_$tool.log 2>&1
  echo "smoke $tool rc=$? :: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize_smoke_$tool.log | tail -1)"
done
timeout 1500 $CS --tool memcheck python -m pytest -q -x -m gpu -p no:cacheprovider \
  tests/test_gpu_spmv.py tests/test_gpu_tile.py tests/test_gpu_pagerank.py \
  -k "walkthrough or fuzz or edge or long_row or many_rows or ring or cycle or dangling or short_rows or empty or odd or dense or device_driven or degree_relabel" \
  > gpurun_out/sanitize_tests_memcheck.log 2>&1
echo "tests memcheck rc=$? :: $(grep -E 'passed|failed|ERROR SUMMARY' gpurun_out/sanitize_tests_memcheck.log | tail -2 | tr '\n' ' ')"
MBX_GRAPH_MODE=unrolled timeout 1500 $CS --tool synccheck python -m pytest -q -x -m gpu -p no:cacheprovider \
  tests/test_gpu_spmv.py tests/test_gpu_tile.py tests/test_gpu_pagerank.py tests/test_gpu_bicgstab.py \
  tests/test_gpu_comparators.py \
  -k "walkthrough or fuzz or edge or long_row or many_rows or ring or cycle or dangling or short_rows or empty or odd or dense or device_driven or degree_relabel or stencil or laplacian or singular or trivial or corpus" \
  > gpurun_out/sanitize_tests_synccheck.log 2>&1
echo "tests synccheck rc=$? :: $(grep -E 'passed|failed|ERROR SUMMARY' gpurun_out/sanitize_tests_synccheck.log | tail -2 | tr '\n' ' ')"
# the preprocessing kernels of late round 2 (K1 bounds + scan, hub sampling /
# histogram / pick / selection, word map, slot copy with both hub encodings):
# the exact-top-h and capped-count hub tests and the compact round trips
for tool in memcheck racecheck initcheck; do
  timeout 1500 $CS --tool $tool python -m pytest -q -x -m gpu -p no:cacheprovider \
    tests/test_gpu_xcache.py tests/test_gpu_spmv.py -k "top_h or capped or compact or automatic or stencil or local" \
    > gpurun_out/sanitize_preproc_$tool.log 2>&1
  echo "preprocessing $tool rc=$? :: $(grep -E 'passed|failed|ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize_preproc_$tool.log | tail -2 | tr '\n' ' ')"
done
