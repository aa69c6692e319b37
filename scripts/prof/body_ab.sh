# WHILE-body iterations A/B (MBX_BODY_ITERS)
cd $GRAFT_REPO_ROOT
for i in 1 2 3; do for k in 2 4 10; do
  MBX_BODY_ITERS=$k python scripts/prof/pr_iter.py 24 100 3 2>&1 | tail -1 | sed "s/^/body$k /"
done; done
