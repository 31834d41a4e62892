#!/bin/bash
# Round-2 evidence for the tensor-core build on one B200: full bench line, the launch list of a short
# bench, ncu --set full of pairs_tcs_kernel and of the sorted FFMA kernel (scripts/one_tcs.py)
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err; echo "bench rc=$?"
python bench.py --steps 2 --warmup 3 --no-secondary --no-cpu-baseline > gpurun_out/r2f_short.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/r2f_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-secondary --no-cpu-baseline > gpurun_out/r2f_ncu_launches.log 2>&1; echo "launches rc=$?"
python scripts/one_tcs.py > gpurun_out/r2f_one_tcs.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:pairs_tcs -c 1 -o gpurun_out/r2f_prof_tcs \
    python scripts/one_tcs.py > gpurun_out/r2f_ncu_tcs.log 2>&1; echo "ncu tcs rc=$?"
ncu --set full --import-source on --clock-control none -k regex:pairs_kernel -c 1 -o gpurun_out/r2f_prof_ffma \
    python scripts/one_tcs.py > gpurun_out/r2f_ncu_ffma.log 2>&1; echo "ncu ffma rc=$?"
