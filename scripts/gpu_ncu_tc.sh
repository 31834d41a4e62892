# ncu --set full of the tensor-core count kernel at N = 2^20 and 65,536 (after a clean plain run)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python scripts/profile_kernels.py tc --reps 1 > gpurun_out/prof_tc_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:pairs_tc_kernel -s 1 -c 2 -o gpurun_out/prof_tc \
    python scripts/profile_kernels.py tc --reps 1 > gpurun_out/ncu_tc.log 2>&1
echo "tc rc=$?"
ncu -i gpurun_out/prof_tc.ncu-rep --page raw --csv > gpurun_out/prof_tc_raw.csv 2>&1
grep -i "tmem\|tensor\|utc" gpurun_out/prof_tc_raw.csv | head -3 > /dev/null
