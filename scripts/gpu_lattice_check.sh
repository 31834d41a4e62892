# dense-regime counting array: parity tests, then step time + per-kernel times for each scripts/libpc_*.so
cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_parity.py -q -m gpu -k "dense_regime or config5 or lattice or batch" -p no:cacheprovider 2>&1 | tail -2
for so in scripts/libpc_*.so; do
  echo "== $so"
  PAIRCOUNT_LIB=$PWD/$so python scripts/profile_kernels.py lattice --reps 6 | tail -2
  PAIRCOUNT_LIB=$PWD/$so ncu --metrics gpu__time_duration.sum --clock-control none -k regex:lat_ --csv \
    python scripts/profile_kernels.py lattice --reps 1 2>/dev/null | grep lat_ | awk -F'","' '{print $5, $NF}' | tail -7 | sed 's/(.*)//'
done
