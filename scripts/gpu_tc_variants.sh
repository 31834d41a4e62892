cd $GRAFT_REPO_ROOT
for so in scripts/libpc_E*.so; do echo "== $so"; PAIRCOUNT_LIB=$PWD/$so timeout 120 python scripts/profile_kernels.py tc --reps 3 2>&1 | tail -2 | cut -c1-150; done
