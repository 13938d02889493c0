set -u
mkdir -p gpurun_out; O=gpurun_out
timeout 900 python scripts/tune_symbolic.py > $O/tune_r2e.log 2>&1; tail -8 $O/tune_r2e.log
python scripts/exp/tuned_from_record.py $O/symbolic_tuning.json profiles/r02e_symbolic_tuning.json paper_2006_03031_b200/tuned/bert_dense_schedules.json
cp paper_2006_03031_b200/tuned/bert_dense_schedules.json $O/bert_dense_schedules.json
timeout 900 python scripts/bench_configs.py 2,3,4 > $O/configs_r2e.json 2> $O/configs_r2e.err; tail -c 1500 $O/configs_r2e.json
