#!/bin/bash
# Round-2 evidence on one B200: full bench line, launch list of a short bench, ncu of the sorted kernel
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 > gpurun_out/r2_final_bench.json 2> gpurun_out/r2_final_bench.err; echo "bench rc=$?"
python bench.py --steps 2 --warmup 3 --no-secondary --no-cpu-baseline > gpurun_out/r2_short.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-secondary --no-cpu-baseline > gpurun_out/r2_ncu_launches.log 2>&1; echo "launches rc=$?"
python scripts/one_sorted.py > gpurun_out/r2_one_sorted.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:pairs_kernel -c 1 -o gpurun_out/r2_prof_sorted \
    python scripts/one_sorted.py > gpurun_out/r2_ncu_sorted.log 2>&1; echo "ncu sorted rc=$?"
