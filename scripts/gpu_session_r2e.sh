# Round-2 final evidence on one B200 (third session): tests, smoke, bench, configs 2-4, GEMM sweep,
# ncu launch list + full captures (bench GEMMs, attention, family 4), compute-sanitizer.
set -u
mkdir -p gpurun_out; O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $O/gpu.txt 2>&1; nproc >> $O/gpu.txt
rm -f $O/parity_report.jsonl
timeout 900 python scripts/tune_symbolic.py > $O/tune.log 2>&1; echo "tune rc=$?"; tail -8 $O/tune.log
python scripts/exp/tuned_from_record.py $O/symbolic_tuning.json profiles/r02e_symbolic_tuning.json paper_2006_03031_b200/tuned/bert_dense_schedules.json > /dev/null
cp paper_2006_03031_b200/tuned/bert_dense_schedules.json $O/bert_dense_schedules.json
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests.log; tail -2 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log; tail -2 $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
python -c "
import json; d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]); print('bench', d['value'], d['e2e']['value'], d['batch1']['value'], d['roofline']['frac'], d['vs_static']['worst_ratio'], d['vs_static']['all_bitwise_equal'], d['clocks'])"
timeout 1200 python scripts/bench_configs.py 2,3,4 > $O/configs.log 2>&1; echo "configs rc=$?"
rm -f $O/gemm_sweep_final.jsonl
timeout 900 python scripts/gemm_sweep.py --Ms 1,16,64,128,256,512,1024,2048,4096,8192,17448 --tag m_sweep --out $O/gemm_sweep_final.jsonl > /dev/null 2>&1
timeout 600 python scripts/gemm_sweep.py --shapes base --Ms 1,16,64,128,512,2048 --tag base --out $O/gemm_sweep_final.jsonl > /dev/null 2>&1
timeout 900 python scripts/gemm_sweep.py --residues 512,1024,2048 --tag residues --out $O/gemm_sweep_final.jsonl > /dev/null 2>&1
echo sweep lines $(wc -l < $O/gemm_sweep_final.jsonl)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python bench.py --profile --steps 1 --warmup 1 > $O/ncu_launch.log 2>&1; echo "ncu-launch rc=$?"
python scripts/launch_shares.py $O/launches.csv > $O/launch_shares.txt 2>&1; head -9 $O/launch_shares.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:umma_gemm -s 96 -c 4 -o $O/prof_gemm -f \
    python bench.py --profile --steps 1 --warmup 1 > $O/ncu_full.log 2>&1; echo "ncu-gemm rc=$?"
python scripts/gemm_traffic.py $O/prof_gemm.ncu-rep > $O/gemm_traffic.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attention -s 4 -c 1 -o $O/prof_attn -f \
    python bench.py --profile --steps 1 --warmup 1 > $O/ncu_attn.log 2>&1; echo "ncu-attn rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ws_gemm -s 40 -c 4 -o $O/prof_ws -f \
    python scripts/config3_launches.py 64 > $O/ncu_ws.log 2>&1; echo "ncu-ws rc=$?"
bash scripts/sanitize.sh
for r in prof_gemm prof_attn prof_ws; do python scripts/ncu_summary.py $O/$r.ncu-rep > $O/${r}_summary.txt 2>&1; done
python scripts/sass_histogram.py > $O/sass_histogram.txt 2>&1
echo session-done
