# K1 A/B: working tree vs HEAD (exp/head)
cd $GRAFT_REPO_ROOT
for i in 1 2; do
  TAG=tree python scripts/prof/k1_time.py 2>&1 | grep tile
  TAG=head MBX_LIB_PATH=exp/head/libmerbit_b200.so python scripts/prof/k1_time.py 2>&1 | grep tile
done
