# A/B of the two-warp, two-k-block producer (NIMBLE_KD=1 forces one k-block per stage)
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dense_bmm.py tests/test_gpu_parity_r2.py tests/test_gpu_dense_ln.py tests/test_gpu_devdispatch.py -q -m gpu -x -p no:cacheprovider > gpurun_out/tests_kd.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/tests_kd.log
for kd in 1 2; do
  NIMBLE_KD=$kd timeout 600 python scripts/gemm_sweep.py --Ms 128,512,1024,2048,4096,17448 --tag kd$kd --out gpurun_out/exp_kd.jsonl > /dev/null 2>&1
done
echo sweeps done
