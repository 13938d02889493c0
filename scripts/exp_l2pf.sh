set -u
mkdir -p gpurun_out
for pf in 0 1; do
  NIMBLE_L2PF=$pf timeout 600 python scripts/gemm_sweep.py --Ms 128,512,1024,2048 --tag pf$pf --out gpurun_out/exp_l2pf.jsonl > /dev/null 2>&1
  NIMBLE_L2PF=$pf timeout 600 python scripts/gemm_sweep.py --Ms 128,512,1024,2048 --hot --tag pf$pf --out gpurun_out/exp_l2pf.jsonl > /dev/null 2>&1
done
echo sweeps done
timeout 1200 python -m pytest tests/test_gpu_parity_r2.py tests/test_gpu_dense_bmm.py tests/test_gpu_packed.py tests/test_gpu_dense_ln.py -q -m gpu -x -p no:cacheprovider > gpurun_out/tests_r2.log 2>&1; echo tests rc=$?
tail -30 gpurun_out/tests_r2.log
