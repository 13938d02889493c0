set -u
mkdir -p gpurun_out; O=gpurun_out; F=$O/poly_ab.txt; rm -f $F
L=$PWD/paper_2006_03031_b200
for i in 1 2 3; do
  echo -n "poly2 " >> $F; python scripts/attn_balance.py 2>&1 | tail -1 >> $F
  echo -n "poly3 " >> $F; NIMBLE_LIB=$L/libnimble_p3.so python scripts/attn_balance.py 2>&1 | tail -1 >> $F
done
cat $F
