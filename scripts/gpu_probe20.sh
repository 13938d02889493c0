set -u
mkdir -p gpurun_out; O=gpurun_out; F=$O/pair_medium.jsonl; rm -f $F
MS=512,768,1024,1536,2048,3072
timeout 300 python scripts/exp/pair_medium.py def $MS >> $F 2> $O/pm_err.txt
for t in 64 128 256; do
  NIMBLE_EXP_PAIR_FROM=256 NIMBLE_EXP_T3=$t timeout 300 python scripts/exp/pair_medium.py p$t $MS >> $F 2>> $O/pm_err.txt
done
NIMBLE_EXP_PAIR_FROM=256 NIMBLE_EXP_T3=64 python scripts/trace_phases.py 512x1024x1024,1024x1024x1024,2048x1024x1024,1024x3072x1024 > $O/trace_phases_p64.txt 2>&1
python - <<'PY'
import torch
for M,N,K in [(17448,3072,1024),(17448,1024,1024),(17448,4096,1024),(17448,1024,4096)]:
    x=torch.randn((M,K),device="cuda",dtype=torch.bfloat16); W=torch.randn((N,K),device="cuda",dtype=torch.bfloat16)
    for _ in range(3): y=x@W.t()
torch.cuda.synchronize()
PY
ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__cluster_dim_x,launch__cluster_dim_y,launch__shared_mem_per_block_dynamic --clock-control none --csv --log-file $O/cublas_big.csv python -c "
import torch
for M,N,K in [(17448,3072,1024),(17448,1024,1024),(17448,4096,1024),(17448,1024,4096)]:
    x=torch.randn((M,K),device='cuda',dtype=torch.bfloat16); W=torch.randn((N,K),device='cuda',dtype=torch.bfloat16)
    for _ in range(2): y=x@W.t()
torch.cuda.synchronize()
" > /dev/null 2>&1
