# time the direct/gram kernels for each library variant scripts/libpc_*.so
cd $GRAFT_REPO_ROOT
for so in scripts/libpc_*.so; do
  echo "== $so"
  PAIRCOUNT_LIB=$PWD/$so python scripts/profile_kernels.py direct --reps 2
  PAIRCOUNT_LIB=$PWD/$so python scripts/profile_kernels.py gram --reps 2
done
