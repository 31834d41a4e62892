#!/bin/bash
# round-2 soak (new claim order, parts, key kernel) + reference arm + launch list retry
mkdir -p gpurun_out
timeout 1500 python scripts/parity_soak.py --minutes 18 --seed 7 --sorted > gpurun_out/r2_soak.log 2>&1; echo "soak rc=$?"; tail -16 gpurun_out/r2_soak.log
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_ref.json 2> gpurun_out/r2_ref.err; echo "ref rc=$?"
B="python bench.py --steps 2 --warmup 3 --no-secondary --no-cpu-baseline"
$B > gpurun_out/r2_short2.json 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv $B > gpurun_out/r2_launches_stdout.csv 2> gpurun_out/r2_launches.err; echo "launch rc=$?"; ls -la gpurun_out/r2_launches_stdout.csv
