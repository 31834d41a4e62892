# counting-array step time for each library variant scripts/libpc_*.so
cd $GRAFT_REPO_ROOT
for so in scripts/libpc_*.so; do
  echo "== $so"
  PAIRCOUNT_LIB=$PWD/$so python scripts/profile_kernels.py lattice --reps 8 | tail -3
done
