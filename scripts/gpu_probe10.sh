set -u
mkdir -p gpurun_out; O=gpurun_out
for v in "" _rcp _nr; do
  echo "== variant $v"
  NIMBLE_LIB=paper_2006_03031_b200/libnimble$v.so python scripts/trace_stages.py 17448x4096x1024 2>&1 | grep 'within'
  NIMBLE_LIB=paper_2006_03031_b200/libnimble$v.so timeout 600 python scripts/gemm_sweep.py --Ms 2048,17448 --tag "gelu$v" --out $O/sweep_gelu.jsonl > /dev/null 2>&1
done
NIMBLE_LIB=paper_2006_03031_b200/libnimble_nr.so timeout 600 python -m pytest tests/test_gpu_parity_r2.py -x -q -p no:cacheprovider -k gelu 2>&1 | tail -2
