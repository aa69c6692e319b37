# A/B: plain SpMV with y stored st.global.cs (exp/ycs) vs default (exp/base)
cd $GRAFT_REPO_ROOT
for i in 1 2; do for v in base ycs; do
  for a in "24 f32 50 1 0" "24 f64 50 1 0" "24 f64 50 1 1" "24 f32 50 1 1" "20 f32 200 0 0"; do
    MBX_LIB_PATH=exp/$v/libmerbit_b200.so python scripts/prof/spmv_iter.py $a 2>&1 | tail -1 | sed "s/^/$v /"
  done
done; done
