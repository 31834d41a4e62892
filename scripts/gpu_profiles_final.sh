# Round-end evidence: bench launch list + ncu --set full of every hot kernel (each after a clean plain run)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
$B > gpurun_out/bench_small.json 2> gpurun_out/bench_small.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv $B > gpurun_out/ncu_bench.log 2>&1
echo "launch list rc=$?"
for c in direct gram cfg2; do
  python scripts/profile_kernels.py $c --reps 1 > gpurun_out/prof_${c}_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:pairs_kernel -s 1 -c 1 -o gpurun_out/prof_$c \
      python scripts/profile_kernels.py $c --reps 1 > gpurun_out/ncu_$c.log 2>&1
  echo "$c rc=$?"
done
bash scripts/gpu_ncu_lattice.sh
