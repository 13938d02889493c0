set -u
mkdir -p gpurun_out; O=gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity_r2.py -q -x -p no:cacheprovider -k "family3" > $O/pytest_f3.txt 2>&1; tail -3 $O/pytest_f3.txt
F=$O/newrule.jsonl; rm -f $F
timeout 400 python scripts/exp/pair_medium.py new 512,768,1024,1536,2048,2304,2560,3072,4096 >> $F 2> $O/nr_err.txt
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest_gpu_r2e.txt 2>&1; tail -3 $O/pytest_gpu_r2e.txt
timeout 900 python bench.py > $O/bench_r2e.json 2> $O/bench_r2e.err; tail -c 400 $O/bench_r2e.json
