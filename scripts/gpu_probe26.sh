set -u
mkdir -p gpurun_out; O=gpurun_out
timeout 600 python scripts/exp/ws_vs_f1.py > $O/ws_vs_f1.jsonl 2> $O/ws_vs_f1.err
timeout 600 python scripts/exp/epi_cost.py > $O/epi_cost.jsonl 2> $O/epi_cost.err
cat $O/epi_cost.jsonl
