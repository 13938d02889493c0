set -u
mkdir -p gpurun_out; O=gpurun_out
timeout 300 ./scripts/exp/tma_issue > $O/tma_issue.txt 2>&1; echo "rc=$?" >> $O/tma_issue.txt
timeout 600 python scripts/trace_kblocks.py 128x1024x1024,1024x1024x1024,512x3072x1024,2048x3072x1024,16x2304x768,128x3072x768 > $O/trace_medium.txt 2>&1; echo "rc=$?" >> $O/trace_medium.txt
