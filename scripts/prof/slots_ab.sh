# slot copy A/B: working tree vs HEAD (exp/head)
cd $GRAFT_REPO_ROOT
for i in 1 2; do
  python scripts/prof/preproc.py s24 s24r c5 c5f64 2>&1 | sed 's/^/tree /'
  MBX_LIB_PATH=exp/head/libmerbit_b200.so python scripts/prof/preproc.py s24 s24r c5 c5f64 2>&1 | sed 's/^/head /'
done
