set -u
mkdir -p gpurun_out; O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_models.py tests/test_gpu_ws.py -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 300 python scripts/exp/lstm_t1.py
python scripts/trace_lstm.py
for s in 40x1024x1024 40x768x3072; do compute-sanitizer --tool synccheck python scripts/exp/ws_sync.py $s 2>&1 | grep -E "^ok|ERROR SUMMARY"; done
