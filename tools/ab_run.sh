# A/B timing of library variants on one bench config, then (optionally) GPU tests.
# usage: [BENCH_ARGS=..] [TESTS=-k expr|all] bash tools/ab_run.sh tag variant...   ("new" = in-tree build)
tag=$1; shift
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
for rep in 1 2; do
for v in "$@"; do
  if [ $v = new ]; then L=""; else L="NAU_LIB=build/var/$v/libnau_b200.so"; fi
  env $L timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/${tag}_${v}_$rep.json 2>gpurun_out/${tag}_${v}_$rep.err
done
done
python tools/abjson.py gpurun_out/${tag}_*.json
if [ "$TESTS" = all ]; then timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -15;
elif [ -n "$TESTS" ]; then timeout 1200 python -m pytest tests -m gpu -x -q $TESTS 2>&1 | tail -15; fi
