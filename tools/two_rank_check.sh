# Plumbing check of the multi-rank bench paths on a ONE-GPU box: two ranks on device 0
# over gloo (host-side exchange; no kernel of one rank waits on the other). Not a
# measurement — it only shows that the slab / shard drivers run to completion.
# usage: bash tools/two_rank_check.sh [ranks]
W=${1:-2}
for c in 0 3 2; do
  NAU_BENCH_DEVICE=0 NAU_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 \
    --nproc-per-node $W --master-addr 127.0.0.1 --master-port $((29530 + c)) bench.py --gpus $W \
    --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/two_rank_cfg$c.json 2> gpurun_out/two_rank_cfg$c.err
  echo "cfg$c world $W rc=$?"; tail -c 600 gpurun_out/two_rank_cfg$c.json | head -c 600; echo
  tail -3 gpurun_out/two_rank_cfg$c.err
done
