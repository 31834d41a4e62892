# ncu evidence for the hot kernels (each ncu run directly follows a clean plain run of the same command)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
P="python scripts/profile_kernels.py"
$P all --reps 2 > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $P all --reps 2 > gpurun_out/ncu_launch.log 2>&1
$P direct --reps 1 > gpurun_out/prof_direct_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:pairs_kernel -s 1 -c 1 -o gpurun_out/prof_direct $P direct --reps 1 > gpurun_out/ncu_direct.log 2>&1
$P gram --reps 1 > gpurun_out/prof_gram_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:pairs_kernel -s 1 -c 1 -o gpurun_out/prof_gram $P gram --reps 1 > gpurun_out/ncu_gram.log 2>&1
$P lattice --reps 1 > gpurun_out/prof_lattice_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:lat_ -s 3 -c 3 -o gpurun_out/prof_lattice $P lattice --reps 1 > gpurun_out/ncu_lattice.log 2>&1
echo done
