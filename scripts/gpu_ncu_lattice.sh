cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
P="python scripts/profile_kernels.py lattice --reps 1"
$P > gpurun_out/prof_lattice_plain.log 2>&1 && \
ncu --set full --clock-control none -k regex:lat_ -s 7 -c 7 -o gpurun_out/prof_lattice $P > gpurun_out/ncu_lattice.log 2>&1
echo "rc=$?"
