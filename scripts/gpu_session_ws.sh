set -u
mkdir -p gpurun_out; O=gpurun_out
rm -f $O/parity_report.jsonl
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests.log; tail -4 $O/gpu_tests.log
timeout 900 python scripts/bench_configs.py 3 > $O/configs3.log 2>&1; echo "configs rc=$?"; cat $O/configs3.log | cut -c1-400
cp $O/configs_report.json $O/configs3_report.json 2>/dev/null
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err; python -c "
import json; d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['batch1']['value'], d['roofline']['frac'])"
