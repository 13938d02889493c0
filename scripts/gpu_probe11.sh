set -u
mkdir -p gpurun_out; O=gpurun_out
python scripts/trace_stages.py 17448x3072x1024,17448x1024x4096 2>&1 | grep -E 'tile|within'
rm -f $O/sweep_bnd.jsonl
timeout 600 python scripts/gemm_sweep.py --Ms 2048,4096,17448 --tag bnd --out $O/sweep_bnd.jsonl > /dev/null 2>&1; echo "sweep rc=$?"
timeout 600 python -m pytest tests/test_gpu_parity_r2.py tests/test_gpu_dense_ln.py tests/test_gpu_dense_bmm.py -x -q -p no:cacheprovider 2>&1 | tail -2
