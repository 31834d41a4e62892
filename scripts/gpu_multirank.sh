# N>1 code paths on ONE GPU: two ranks with the gloo backend sharing cuda:0 (timings meaningless)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 2 --steps 2 --warmup 1 --dist-backend gloo --shared-gpu > gpurun_out/bench_2rank.json 2> gpurun_out/bench_2rank.err
echo "bench 2-rank rc=$?"
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --impl reference --gpus 2 --steps 1 --warmup 0 > gpurun_out/bench_ref_2rank.json 2> gpurun_out/bench_ref_2rank.err
echo "ref 2-rank rc=$?"
python -m pytest tests/test_distributed.py -m gpu -q -p no:cacheprovider 2>&1 | tail -3
