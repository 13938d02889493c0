set -u
mkdir -p gpurun_out; O=gpurun_out
rm -f $O/sweep_wsx.jsonl
for v in "0 libnimble.so" "1 libnimble.so" "2 libnimble.so" "3 libnimble.so" "0 libnimble_lb1.so" "1 libnimble_lb1.so"; do
  set -- $v
  NIMBLE_WS_FLAGS=$1 NIMBLE_LIB=paper_2006_03031_b200/$2 timeout 600 python scripts/gemm_sweep.py --Ms 1,16,128 --tag "f$1_$2" --out $O/sweep_wsx.jsonl > /dev/null 2>&1
  NIMBLE_WS_FLAGS=$1 NIMBLE_LIB=paper_2006_03031_b200/$2 timeout 600 python scripts/gemm_sweep.py --shapes base --Ms 1,16,128 --tag "f$1_$2" --out $O/sweep_wsx.jsonl > /dev/null 2>&1
done
echo done
