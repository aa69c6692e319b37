R="tests/test_gpu_pagerank.py::test_plan_recaptures_after_matrix_buffers_change"
for t in $(grep -h "^def test_" tests/test_gpu_spmv.py tests/test_gpu_tile.py | sed 's/def \(test_[a-z0-9_]*\).*/\1/'); do
  f=tests/test_gpu_spmv.py; grep -q "def $t" tests/test_gpu_tile.py && f=tests/test_gpu_tile.py
  r=$(python -m pytest "$f::$t" "$R" -q -m gpu 2>&1 | tail -1)
  echo "$t: $r"
done
