# ncu --set full of the headline kernel on sorted points (after a clean plain run) + DRAM bytes
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python scripts/profile_kernels.py sorted --reps 1 > gpurun_out/prof_sorted_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:pairs_kernel -s 1 -c 1 -o gpurun_out/prof_sorted \
    python scripts/profile_kernels.py sorted --reps 1 > gpurun_out/ncu_sorted.log 2>&1
echo "sorted rc=$?"
