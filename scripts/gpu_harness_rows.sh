# The reference harness's experiments with GPU rows (bench_cli), CSVs into gpurun_out/
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
M="python -m paper_1901_11204_b200.bench_cli"
$M bench linear-vs-quadratic --out gpurun_out/h_lvq.csv > gpurun_out/h.log 2>&1; echo "lvq rc=$?"
$M bench spi --out gpurun_out/h_spi.csv >> gpurun_out/h.log 2>&1; echo "spi rc=$?"
$M bench realloc --out gpurun_out/h_realloc.csv >> gpurun_out/h.log 2>&1; echo "realloc rc=$?"
$M bench locality --out gpurun_out/h_locality.csv >> gpurun_out/h.log 2>&1; echo "locality rc=$?"
$M verify full --out gpurun_out/h_verify_full.csv >> gpurun_out/h.log 2>&1; echo "verify full rc=$?"
$M stats --in gpurun_out/h_lvq.csv --out gpurun_out/h_stats.csv >> gpurun_out/h.log 2>&1; echo "stats rc=$?"
