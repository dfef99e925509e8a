set -x
python -c "from paper_2508_13386_b200 import build as b; b.build(force=False)"
timeout 600 python bench.py --steps 6 --warmup 4 --no-cpu-baseline > gpurun_out/r2_bench5_x.json 2> gpurun_out/r2_bench5_x.err; echo "bench rc=$?"
MSIM_COARSE_ORDER=nd timeout 600 python bench.py --steps 6 --warmup 4 --no-cpu-baseline > gpurun_out/r2_bench5_nd.json 2> gpurun_out/r2_bench5_nd.err; echo "bench rc=$?"
MSIM_GAL_FUSED=1 MSIM_COARSE_ORDER=nd timeout 600 python bench.py --steps 6 --warmup 4 --no-cpu-baseline > gpurun_out/r2_bench5_ndf.json 2> gpurun_out/r2_bench5_ndf.err; echo "bench rc=$?"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_2508_13386_b200/csrc tools/bench_diag.cu -o /tmp/bench_diag && /tmp/bench_diag > gpurun_out/r2_bench_diag.txt 2>&1; cat gpurun_out/r2_bench_diag.txt
