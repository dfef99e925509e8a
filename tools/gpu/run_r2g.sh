set -x
python -c "from paper_2508_13386_b200 import build as b; b.build(force=False)"
timeout 1200 python -m pytest tests/test_gpu_coarse_pcg.py -q -x -p no:cacheprovider --durations=5 > gpurun_out/r2_pytest6.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/r2_pytest6.log
timeout 600 python bench.py --steps 6 --warmup 4 --no-cpu-baseline --coarse pcg > gpurun_out/r2_bench6_pcg.json 2> gpurun_out/r2_bench6_pcg.err; echo "bench rc=$?"
tail -c 300 gpurun_out/r2_bench6_pcg.err
