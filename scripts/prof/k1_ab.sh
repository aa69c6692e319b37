# K1 CTA shape A/B (exp/k1_<threads>_<lanes per thread>)
cd $GRAFT_REPO_ROOT
for i in 1 2; do for v in k1_256_4 k1_128_4 k1_512_4 k1_128_8; do
  TAG=$v MBX_LIB_PATH=exp/$v/libmerbit_b200.so python scripts/prof/k1_time.py 2>&1 | grep tile
done; done
