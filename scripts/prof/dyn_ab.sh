# A/B: K2 dynamic range claiming (working tree, MBX_DYN_RANGES=1/0) vs HEAD (exp/head)
cd $GRAFT_REPO_ROOT
for i in 1 2 3; do
  python scripts/prof/pr_iter.py 24 100 3 2>&1 | tail -1 | sed 's/^/dyn /'
  MBX_DYN_RANGES=0 python scripts/prof/pr_iter.py 24 100 3 2>&1 | tail -1 | sed 's/^/static /'
  MBX_LIB_PATH=exp/head/libmerbit_b200.so python scripts/prof/pr_iter.py 24 100 3 2>&1 | tail -1 | sed 's/^/head /'
done
for a in "24 f32 50 1 0" "24 f64 50 1 0" "20 f32 200 0 0"; do
  python scripts/prof/spmv_iter.py $a 2>&1 | tail -1 | sed 's/^/dyn /'
  MBX_DYN_RANGES=0 python scripts/prof/spmv_iter.py $a 2>&1 | tail -1 | sed 's/^/static /'
  MBX_LIB_PATH=exp/head/libmerbit_b200.so python scripts/prof/spmv_iter.py $a 2>&1 | tail -1 | sed 's/^/head /'
done
