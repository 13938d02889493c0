set -u
mkdir -p gpurun_out; O=gpurun_out
rm -f $O/parity_report.jsonl
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gpu_tests_final.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests_final.log; tail -2 $O/gpu_tests_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_final.log 2>&1; echo "smoke rc=$?" >> $O/smoke_final.log; tail -2 $O/smoke_final.log
timeout 900 python bench.py > $O/bench_final.json 2> $O/bench_final.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('$O/bench_final.json').read().strip().splitlines()[-1]); print('bench', d['value'], d['e2e']['value'], d['batch1']['value'], d['roofline']['frac'], d['vs_static']['worst_ratio'], d['clocks'])"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"; tail -c 600 $O/bench_ref.json
