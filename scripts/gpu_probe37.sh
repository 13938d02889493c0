set -u
mkdir -p gpurun_out; O=gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:umma_gemm -s 96 -c 4 -o $O/prof_gemm_final -f \
    python bench.py --profile --steps 1 --warmup 1 > $O/ncu_full_final.log 2>&1; echo "ncu-gemm rc=$?"
python scripts/gemm_traffic.py $O/prof_gemm_final.ncu-rep > $O/gemm_traffic_final.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attention -s 4 -c 1 -o $O/prof_attn_final -f \
    python bench.py --profile --steps 1 --warmup 1 > $O/ncu_attn_final.log 2>&1; echo "ncu-attn rc=$?"
for r in prof_gemm_final prof_attn_final; do python scripts/ncu_summary.py $O/$r.ncu-rep > $O/${r}_summary.txt 2>&1; done
python scripts/sass_histogram.py > $O/sass_histogram_final.txt 2>&1
grep -E "Kernel Name|tensor_cycles|duration" $O/prof_gemm_final_summary.txt | head -12
