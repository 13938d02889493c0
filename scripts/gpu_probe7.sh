set -u
mkdir -p gpurun_out; O=gpurun_out
rm -f $O/ab_kd.jsonl
bash scripts/exp_ab.sh NIMBLE_KD "2 1" 2048,4096,17448 $O/ab_kd.jsonl
bash scripts/exp_ab.sh NIMBLE_KD "2 1" 2048,4096,17448 $O/ab_kd.jsonl
