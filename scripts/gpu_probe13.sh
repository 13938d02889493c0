set -u
mkdir -p gpurun_out; O=gpurun_out
NIMBLE_T3=192 python scripts/exp/t3_check.py
rm -f $O/sweep_t3.jsonl
for t in 256 192 224 160; do
  NIMBLE_T3=$t timeout 600 python scripts/gemm_sweep.py --Ms 2048,3072,4096,8192,17448 --tag "t$t" --out $O/sweep_t3.jsonl > /dev/null 2>&1
done
echo done
