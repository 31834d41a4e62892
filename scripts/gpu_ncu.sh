# usage: bash scripts/gpu_ncu.sh <case> [<case> ...]   (cases of scripts/profile_kernels.py)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in "$@"; do
  python scripts/profile_kernels.py $c --reps 1 > gpurun_out/prof_${c}_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:pairs_kernel -s 1 -c 1 -o gpurun_out/prof_$c \
      python scripts/profile_kernels.py $c --reps 1 > gpurun_out/ncu_$c.log 2>&1
  echo "$c rc=$?"
done
