# Round evidence on one B200: ncu launch lists and full captures first (they refresh
# profiles/traffic.json, which the bench lines quote), then bench lines for every
# BASELINE config, cfg2 EXACT, the reference arm and the one-rank slab run.
# usage: bash tools/measure_round.sh TAG   (outputs in gpurun_out/TAG_*)
T=${1:-r2f}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_throttle_reasons.active --format=csv,noheader
# every profiled command first runs clean without ncu
timeout 600 python tools/profile_step.py --config 2 --steps 1 && \
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"k_reorder|k_hash|k_scatter|k_nlist_pair|k_wcsph_density_pair|k_wcsph_momentum_pair|k_symplectic" -c 7 \
  -o /tmp/${T}_full_cfg2 python tools/profile_step.py --config 2 --steps 1 > gpurun_out/${T}_ncu_full2.log 2>&1
echo "full2 rc=$?"
timeout 600 python tools/profile_step.py --config 4 --steps 1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${T}_launches_cfg4.csv python tools/profile_step.py --config 4 --steps 1 > gpurun_out/${T}_ncu_launch4.log 2>&1
echo "launches4 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gravity_fast -c 1 \
  -o /tmp/${T}_full_cfg4 python tools/profile_step.py --config 4 --steps 1 > gpurun_out/${T}_ncu_full4.log 2>&1
echo "full4 rc=$?"
timeout 600 python tools/profile_step.py --config 1 --steps 1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${T}_launches_cfg1.csv python tools/profile_step.py --config 1 --steps 1 > gpurun_out/${T}_ncu_launch1.log 2>&1
echo "launches1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sph_fast -c 2 \
  -o /tmp/${T}_full_cfg1 python tools/profile_step.py --config 1 --steps 1 > gpurun_out/${T}_ncu_full1.log 2>&1
echo "full1 rc=$?"
# reports stay on the box (gpurun returns <= 64 MiB): summaries + raw metric pages come back
for k in cfg1 cfg2 cfg4; do
  python tools/summarize_ncu.py full /tmp/${T}_full_$k.ncu-rep > gpurun_out/${T}_ncu_full_$k.md 2>/dev/null
  ncu -i /tmp/${T}_full_$k.ncu-rep --page raw --csv > gpurun_out/${T}_ncu_raw_$k.csv 2>/dev/null
done
python tools/make_traffic.py $T > /dev/null && cp profiles/traffic.json gpurun_out/${T}_traffic.json
for c in 2 0 1 3 4; do
  timeout 900 python bench.py --config $c > gpurun_out/${T}_bench_cfg$c.json 2> gpurun_out/${T}_bench_cfg$c.err
  echo "cfg$c rc=$?"; tail -c 300 gpurun_out/${T}_bench_cfg$c.json
done
timeout 900 python bench.py --config 2 --mode exact --no-cpu-baseline > gpurun_out/${T}_bench_cfg2_exact.json 2> gpurun_out/${T}_bench_cfg2_exact.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${T}_reference_cfg2.json 2> gpurun_out/${T}_reference_cfg2.err
echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${T}_launches_cfg2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${T}_ncu_launch2.log 2>&1
echo "launches2 rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
  --master-port 29517 bench.py --gpus 1 --steps 3 --warmup 3 --slab --no-cpu-baseline > gpurun_out/${T}_slab_cfg2.json 2> gpurun_out/${T}_slab_cfg2.err
echo "slab rc=$?"; tail -c 400 gpurun_out/${T}_slab_cfg2.json
du -sh gpurun_out
