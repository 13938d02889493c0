set -u
mkdir -p gpurun_out; O=gpurun_out
rm -f $O/sweep_c8.jsonl
for v in "" _c8 "" _c8; do
  NIMBLE_LIB=paper_2006_03031_b200/libnimble$v.so timeout 600 python scripts/gemm_sweep.py --Ms 1,16,128,512 --tag "c$v" --out $O/sweep_c8.jsonl > /dev/null 2>&1
  NIMBLE_LIB=paper_2006_03031_b200/libnimble$v.so timeout 600 python scripts/gemm_sweep.py --shapes base --Ms 1,16,128 --tag "c$v" --out $O/sweep_c8.jsonl > /dev/null 2>&1
done
NIMBLE_LIB=paper_2006_03031_b200/libnimble_c8.so compute-sanitizer --tool synccheck python scripts/exp/ws_sync.py 40x1024x1024 2>&1 | grep -E "^ok|ERROR SUMMARY"
timeout 600 python -m pytest tests/test_gpu_models.py -q -x -p no:cacheprovider -k "lstm" 2>&1 | tail -2
timeout 300 python scripts/exp/lstm_t1.py
