# A/B of an experiment knob on the GEMM sweep: bash scripts/exp_ab.sh VAR "v0 v1" Ms out
set -u
VAR=$1; VALS=$2; MS=$3; OUT=$4
mkdir -p gpurun_out
for v in $VALS; do
  env $VAR=$v timeout 600 python scripts/gemm_sweep.py --Ms $MS --tag "$VAR=$v" --out $OUT > /dev/null 2>&1
done
echo done
