set -u
mkdir -p gpurun_out; O=gpurun_out
NIMBLE_EXP_WS2=1 python scripts/exp/ws2_check.py
rm -f $O/sweep_ws2x.jsonl
for v in 0 1 0 1; do
  NIMBLE_EXP_WS2=$v timeout 600 python scripts/gemm_sweep.py --Ms 129,256,384,512,768,1024 --tag "ws2_$v" --out $O/sweep_ws2x.jsonl > /dev/null 2>&1
  NIMBLE_EXP_WS2=$v timeout 600 python scripts/gemm_sweep.py --shapes base --Ms 256,512 --tag "ws2_$v" --out $O/sweep_ws2x.jsonl > /dev/null 2>&1
done
echo done
