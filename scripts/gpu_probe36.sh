set -u
mkdir -p gpurun_out; O=gpurun_out
rm -f $O/parity_report.jsonl
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gpu_tests_last.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests_last.log; tail -2 $O/gpu_tests_last.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_last.log 2>&1; echo "smoke rc=$?" >> $O/smoke_last.log; tail -2 $O/smoke_last.log
timeout 900 python bench.py > $O/bench_last.json 2> $O/bench_last.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('$O/bench_last.json').read().strip().splitlines()[-1]); print('bench', d['value'], d['e2e']['value'], d['batch1']['value'], d['roofline']['frac'], d['vs_static']['worst_ratio'], d['vs_static']['all_bitwise_equal'], d['clocks'])"
rm -f $O/sweep_last.jsonl
timeout 900 python scripts/gemm_sweep.py --Ms 1,16,64,128,256,512,1024,2048,4096,8192,17448 --tag last --out $O/sweep_last.jsonl > /dev/null 2>&1; echo sweep $(wc -l < $O/sweep_last.jsonl)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_last.csv \
    python bench.py --profile --steps 1 --warmup 1 > $O/ncu_launch_last.log 2>&1; echo "ncu-launch rc=$?"
python scripts/launch_shares.py $O/launches_last.csv > $O/launch_shares_last.txt 2>&1; head -8 $O/launch_shares_last.txt
