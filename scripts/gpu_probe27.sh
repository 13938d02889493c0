set -u
mkdir -p gpurun_out; O=gpurun_out; F=$O/gelu_ab.jsonl; rm -f $F
L=$PWD/paper_2006_03031_b200
for i in 1 2; do
  for v in base rcp2 nr; do
    if [ $v = base ]; then lib=$L/libnimble.so; else lib=$L/libnimble_$v.so; fi
    NIMBLE_LIB=$lib timeout 300 python scripts/exp/epi_cost.py | sed "s/^{/{\"v\": \"$v\", /" >> $F
  done
done
cat $F
for v in rcp2 nr; do
NIMBLE_LIB=$L/libnimble_$v.so timeout 600 python -m pytest tests/test_gpu_parity_r2.py -q -x -p no:cacheprovider -k "gelu or family3_bench" > $O/pytest_gelu_$v.txt 2>&1; tail -1 $O/pytest_gelu_$v.txt
done
