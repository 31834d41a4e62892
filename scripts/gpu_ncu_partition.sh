# ncu --set full with source of the two partition kernels (second lattice step)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
P="python scripts/profile_kernels.py lattice --reps 1"
$P > gpurun_out/prof_part_plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:lat_partition -s 2 -c 2 -o gpurun_out/prof_part $P > gpurun_out/ncu_part.log 2>&1
echo "rc=$?"
