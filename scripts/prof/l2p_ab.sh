# experiment: L2 persisting window over the head of x (exp/l2p, MBX_L2_PERSIST bytes)
cd $GRAFT_REPO_ROOT
L=exp/l2p/libmerbit_b200.so
for pb in 0 33554432 67108864; do
  MBX_L2_PERSIST=$pb MBX_LIB_PATH=$L python scripts/prof/pr_iter.py 27 20 2 2>&1 | tail -2 | sed "s/^/persist $pb /"
done
for pb in 0 33554432; do
  MBX_L2_PERSIST=$pb MBX_LIB_PATH=$L python scripts/prof/pr_iter.py 24 50 2 2>&1 | tail -2 | sed "s/^/persist $pb /"
done
