set -u
mkdir -p gpurun_out; O=gpurun_out
timeout 600 python scripts/trace_kblocks.py 128x1024x1024,1024x1024x1024,16x2304x768,2048x3072x1024,17448x1024x1024 > $O/trace_medium2.txt 2>&1; echo "rc=$?" >> $O/trace_medium2.txt
timeout 600 python scripts/gemm_sweep.py --Ms 16,128,512,1024,2048,17448 --tag relaxed --out $O/sweep_relaxed.jsonl > /dev/null 2>&1; echo "sweep rc=$?"
