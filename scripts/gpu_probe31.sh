set -u
mkdir -p gpurun_out; O=gpurun_out; F=$O/lnk_ab.txt; rm -f $F
for i in 1 2; do
  for k in 2048 1024; do
    NIMBLE_LN_MIN_K=$k timeout 600 python bench.py --steps 20 --warmup 3 > $O/b_lnk$k.json 2>/dev/null
    python -c "
import json; d=json.loads(open('$O/b_lnk$k.json').read().strip().splitlines()[-1]); print('min_k $k', round(d['value'],1), round(d['ms_per_step'],3), d['clocks']['sm_mhz'])" >> $F
  done
done
cat $F
