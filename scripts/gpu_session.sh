#!/bin/bash
# One gpurun session: GPU tests, smoke, bench, ncu launch list + one full capture of the
# top kernel.  Every step has its own timeout so nothing can hang the box.
set -u
mkdir -p gpurun_out
OUT=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $OUT/gpu.txt 2>&1
nproc >> $OUT/gpu.txt
STEPS=${STEPS:-tests,smoke,bench,ncu}
if [[ $STEPS == *tests* ]]; then
  timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/gpu_tests.log 2>&1; echo "tests rc=$?" >> $OUT/gpu_tests.log
  tail -5 $OUT/gpu_tests.log
fi
if [[ $STEPS == *smoke* ]]; then
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
  tail -3 $OUT/smoke.log
fi
if [[ $STEPS == *bench* ]]; then
  timeout 900 python bench.py ${BENCH_ARGS:-} > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
  tail -c 3000 $OUT/bench.json; tail -5 $OUT/bench.err
fi
if [[ $STEPS == *ncu* ]]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
      python bench.py --profile --steps 1 --warmup 1 > $OUT/ncu_launch.log 2>&1; echo "ncu-launch rc=$?" >> $OUT/ncu_launch.log
  tail -3 $OUT/ncu_launch.log
  # the bench configuration itself (64 requests, M = 17.4k tokens): one layer's four GEMM launches
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:umma_gemm -s 96 -c 4 -o $OUT/prof_gemm -f \
      python bench.py --profile --steps 1 --warmup 1 > $OUT/ncu_full.log 2>&1; echo "ncu-full rc=$?" >> $OUT/ncu_full.log
  python scripts/gemm_traffic.py $OUT/prof_gemm.ncu-rep > $OUT/gemm_traffic.json
  tail -3 $OUT/ncu_full.log
  # one attention launch of the bench configuration (layer 5)
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:attention -s 4 -c 1 -o $OUT/prof_attn -f \
      python bench.py --profile --steps 1 --warmup 1 > $OUT/ncu_attn.log 2>&1; echo "ncu-attn rc=$?" >> $OUT/ncu_attn.log
  tail -2 $OUT/ncu_attn.log
fi
if [[ $STEPS == *configs* ]]; then
  timeout 900 python scripts/bench_configs.py ${CONFIGS:-2,3,4} > $OUT/configs.log 2>&1; echo "configs rc=$?" >> $OUT/configs.log
  tail -8 $OUT/configs.log
fi
