set -u
mkdir -p gpurun_out; O=gpurun_out
timeout 120 ./scripts/exp/pdl_floor > $O/pdl_floor.txt 2>&1; cat $O/pdl_floor.txt
timeout 300 python scripts/trace_ws.py > $O/trace_ws.txt 2>&1; cat $O/trace_ws.txt
