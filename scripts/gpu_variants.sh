# kernel times for each library variant scripts/libpc_*.so (args: profile_kernels cases, default "gram cfg2")
cd $GRAFT_REPO_ROOT
cases=${@:-gram cfg2}
for so in scripts/libpc_*.so; do
  echo "== $so"
  for c in $cases; do
    if [ "$c" = comp ]; then PAIRCOUNT_LIB=$PWD/$so python scripts/time_comp.py | tail -1;
    else PAIRCOUNT_LIB=$PWD/$so python scripts/profile_kernels.py $c --reps 3 | tail -1; fi
  done
done
