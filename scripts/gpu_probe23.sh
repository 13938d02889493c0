set -u
mkdir -p gpurun_out; O=gpurun_out
M=$PWD/paper_2006_03031_b200/libnimble_mw.so
python scripts/trace_phases.py 1024x1024x1024,2048x1024x1024,1024x3072x1024 > $O/tp_base.txt 2>&1
NIMBLE_LIB=$M python scripts/trace_phases.py 1024x1024x1024,2048x1024x1024,1024x3072x1024 > $O/tp_mw.txt 2>&1
F=$O/mw_ab.jsonl; rm -f $F
for i in 1 2; do
timeout 300 python scripts/exp/pair_medium.py base$i 512,1024,2048,4096 >> $F 2> $O/mw_err.txt
NIMBLE_LIB=$M timeout 300 python scripts/exp/pair_medium.py mw$i 512,1024,2048,4096 >> $F 2>> $O/mw_err.txt
done
G=$O/mw_big.jsonl; rm -f $G
for i in 1 2; do
timeout 600 python scripts/gemm_sweep.py --Ms 17448 --tag base$i --out $G > /dev/null 2>&1
NIMBLE_LIB=$M timeout 600 python scripts/gemm_sweep.py --Ms 17448 --tag mw$i --out $G > /dev/null 2>&1
done
NIMBLE_LIB=$M timeout 600 python -m pytest tests/test_gpu_parity_r2.py tests/test_gpu_dense_bmm.py -q -x -p no:cacheprovider > $O/pytest_mw.txt 2>&1; tail -2 $O/pytest_mw.txt
