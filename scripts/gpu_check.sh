set -u
mkdir -p gpurun_out; O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $O/gpu.txt 2>&1; nproc >> $O/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests.log; tail -3 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log; tail -2 $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err; tail -c 3000 $O/bench.json
