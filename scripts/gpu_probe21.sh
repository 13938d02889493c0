set -u
mkdir -p gpurun_out; O=gpurun_out; F=$O/f1_vs_f3.jsonl; rm -f $F
MS=1536,2048,2304,2560,3072,4096,5120,6144,8192
timeout 400 python scripts/exp/pair_medium.py def $MS >> $F 2> $O/f13_err.txt
NIMBLE_EXP_PAIR_FROM=1000000 timeout 400 python scripts/exp/pair_medium.py f1 $MS >> $F 2>> $O/f13_err.txt
