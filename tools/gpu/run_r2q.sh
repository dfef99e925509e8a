set -x
python -c "from paper_2508_13386_b200 import build as b; b.build(force=False)"
timeout 900 python tools/freerun_log.py 4 gpurun_out/r02_freerun_C4.json > gpurun_out/r02_freerun_C4.log 2>&1; echo "rc=$?"
grep -E "worst|newton_counts_equal|steps_compared" gpurun_out/r02_freerun_C4.json
timeout 600 python bench.py --steps 10 --warmup 5 --no-cpu-baseline > gpurun_out/r2_bench13.json 2> gpurun_out/r2_bench13.err; echo "bench rc=$?"
timeout 600 python bench.py --steps 10 --warmup 5 --no-cpu-baseline --cubature --lag > gpurun_out/r2_bench13_next2.json 2> gpurun_out/r2_bench13_next2.err; echo "bench rc=$?"
timeout 600 python bench.py --steps 10 --warmup 5 --no-cpu-baseline --cubature > gpurun_out/r2_bench13_cub.json 2> gpurun_out/r2_bench13_cub.err; echo "bench rc=$?"
timeout 600 python bench.py --steps 10 --warmup 5 --no-cpu-baseline --integrator bdf2 > gpurun_out/r2_bench13_bdf2.json 2> gpurun_out/r2_bench13_bdf2.err; echo "bench rc=$?"
tail -3 gpurun_out/r2_bench13_next2.err
