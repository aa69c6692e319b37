# s24 fp64 SpMV (natural order, transition matrix): K2 shared-memory budget x staging mode
cd $GRAFT_REPO_ROOT
python scripts/prof/spmv_iter.py 24 f64 50 1 0
for sm in 98304 131072 163840 196608; do for md in 0 1 2; do
  SMEM=$sm MODE=$md python scripts/prof/spmv_iter.py 24 f64 50 1 0
done; done
python scripts/prof/spmv_iter.py 24 f64 50 1 0
