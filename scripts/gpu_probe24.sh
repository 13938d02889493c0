set -u
mkdir -p gpurun_out; O=gpurun_out
OLD=$PWD/paper_2006_03031_b200/libnimble_mw.so
rm -f $O/attn_ab.txt
for i in 1 2; do
  echo "old(lane0 attention MMA issuer)" >> $O/attn_ab.txt; NIMBLE_LIB=$OLD python scripts/attn_balance.py 2>&1 | tail -1 >> $O/attn_ab.txt
  echo "new(converged warp)" >> $O/attn_ab.txt; python scripts/attn_balance.py 2>&1 | tail -1 >> $O/attn_ab.txt
done
cat $O/attn_ab.txt
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest_gpu_r2f.txt 2>&1; tail -2 $O/pytest_gpu_r2f.txt
timeout 900 python bench.py > $O/bench_r2f.json 2> $O/bench_r2f.err; python -c "
import json; d=json.loads(open('$O/bench_r2f.json').read().strip().splitlines()[-1]); print('bench', d['value'], d['e2e']['value'], d['roofline']['frac'], d['vs_static']['worst_ratio'], d['clocks'])"
rm -f $O/sweep_r2f.jsonl
timeout 900 python scripts/gemm_sweep.py --Ms 1,16,64,128,256,512,1024,2048,4096,8192,17448 --tag r2f --out $O/sweep_r2f.jsonl > /dev/null 2>&1
echo done
