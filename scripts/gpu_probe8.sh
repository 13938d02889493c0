set -u
mkdir -p gpurun_out; O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_ws.py -x -q -p no:cacheprovider > $O/ws_tests.log 2>&1; echo "rc=$?" >> $O/ws_tests.log; tail -3 $O/ws_tests.log
rm -f $O/sweep_ws2.jsonl
timeout 600 python scripts/gemm_sweep.py --Ms 1,16,128,129,256,384,512,1024 --tag ws2 --out $O/sweep_ws2.jsonl > /dev/null 2>&1; echo "sweep rc=$?"
timeout 600 python scripts/gemm_sweep.py --shapes base --Ms 1,16,128,256,512 --tag ws2_base --out $O/sweep_ws2.jsonl > /dev/null 2>&1; echo "sweep rc=$?"
