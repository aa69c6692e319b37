# K3 serial fold run length A/B (exp/fr<N>)
cd $GRAFT_REPO_ROOT
for i in 1 2 3; do for v in fr32 fr8 fr4; do
  MBX_LIB_PATH=exp/$v/libmerbit_b200.so python scripts/prof/pr_iter.py 24 100 3 2>&1 | tail -1 | sed "s/^/$v /"
done; done
