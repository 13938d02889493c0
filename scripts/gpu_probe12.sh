set -u
mkdir -p gpurun_out; O=gpurun_out
rm -f $O/sweep_lsu.jsonl
for d in 0 64 0 64; do
  NIMBLE_DBG=$d timeout 600 python scripts/gemm_sweep.py --Ms 4096,17448 --tag "dbg$d" --out $O/sweep_lsu.jsonl > /dev/null 2>&1
done
sed -i 's/os.environ\["NIMBLE_DBG"\] = "32"/os.environ["NIMBLE_DBG"] = os.environ.get("TS_DBG", "32")/' scripts/trace_stages.py
TS_DBG=96 python scripts/trace_stages.py 17448x3072x1024 2>&1 | grep -E 'within'
NIMBLE_DBG=64 timeout 600 python -m pytest tests/test_gpu_parity_r2.py tests/test_gpu_dense_ln.py -x -q -p no:cacheprovider 2>&1 | tail -2
