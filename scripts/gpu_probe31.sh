set -u
mkdir -p gpurun_out; O=gpurun_out; F=$O/ln_ab.txt; rm -f $F
run() {  # tag, env...
  local tag=$1; shift
  env "$@" timeout 600 python bench.py --steps 20 --warmup 3 > $O/b_$tag.json 2>/dev/null
  python -c "
import json; d=json.loads(open('$O/b_$tag.json').read().strip().splitlines()[-1]); print('$tag', round(d['value'],1), round(d['ms_per_step'],3), d['roofline']['frac'], d['clocks']['sm_mhz'])" >> $F
}
for i in 1 2; do
  run default NIMBLE_DUMMY=1
  run unfused NIMBLE_FUSED_LN=0
  run ln1fused NIMBLE_LN_MIN_K=1024
done
cat $F
