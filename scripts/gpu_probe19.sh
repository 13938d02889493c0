set -u
mkdir -p gpurun_out; O=gpurun_out
python scripts/exp/cublas_kernels.py > $O/cublas_plain.txt 2>&1
ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,launch__cluster_dim_x,launch__cluster_dim_y,launch__shared_mem_per_block_dynamic,launch__registers_per_thread \
  --clock-control none --csv --log-file $O/cublas_kernels.csv python scripts/exp/cublas_kernels.py > /dev/null 2>&1
python scripts/trace_phases.py 512x1024x1024,1024x1024x1024,2048x1024x1024,1024x3072x1024 > $O/trace_phases_r2e.txt 2>&1
