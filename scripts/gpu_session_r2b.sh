# Round-2 (second session) evidence on one B200: tests, smoke, configs 2-4, bench, GEMM sweeps.
set -u
mkdir -p gpurun_out; O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $O/gpu.txt 2>&1; nproc >> $O/gpu.txt
rm -f $O/parity_report.jsonl
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests.log; tail -3 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log; tail -2 $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
python -c "
import json; d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]); print('bench', d['value'], d['e2e']['value'], d['batch1']['value'], d['roofline']['frac'], d['vs_static']['worst_ratio'], d['vs_static']['all_bitwise_equal'])"
timeout 1200 python scripts/bench_configs.py 2,3,4 > $O/configs.log 2>&1; echo "configs rc=$?"; grep -v '^{"T"' $O/configs.log | cut -c1-300
rm -f $O/gemm_sweep_final.jsonl
timeout 900 python scripts/gemm_sweep.py --Ms 1,16,64,128,256,512,1024,2048,4096,17448 --tag m_sweep --out $O/gemm_sweep_final.jsonl > /dev/null 2>&1
timeout 600 python scripts/gemm_sweep.py --shapes base --Ms 1,16,64,128,512,2048 --tag base --out $O/gemm_sweep_final.jsonl > /dev/null 2>&1
echo sweep lines $(wc -l < $O/gemm_sweep_final.jsonl)
