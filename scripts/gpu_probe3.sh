set -u
mkdir -p gpurun_out; O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_ws.py -x -q -p no:cacheprovider > $O/ws_tests.log 2>&1; echo "rc=$?" >> $O/ws_tests.log; tail -30 $O/ws_tests.log
rm -f $O/sweep_ws.jsonl
timeout 600 python scripts/gemm_sweep.py --Ms 1,16,64,128 --tag ws --out $O/sweep_ws.jsonl > /dev/null 2>&1; echo "sweep rc=$?"
timeout 600 python scripts/gemm_sweep.py --shapes base --Ms 1,16,64,128 --tag ws_base --out $O/sweep_ws.jsonl > /dev/null 2>&1; echo "sweep rc=$?"
