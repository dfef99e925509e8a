set -x
python -c "from paper_2508_13386_b200 import build as b; b.build(force=False)"
timeout 1200 python -m pytest tests/test_gpu_two_level.py tests/test_gpu_multirank.py -x -q -p no:cacheprovider --durations=10 > gpurun_out/r2s_pytest.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/r2s_pytest.log
timeout 600 python bench.py --steps 10 --warmup 5 --no-cpu-baseline --refine two_level > gpurun_out/r2s_bench_tl.json 2> gpurun_out/r2s_bench_tl.err; echo "bench rc=$?"
tail -c 2500 gpurun_out/r2s_bench_tl.json; tail -5 gpurun_out/r2s_bench_tl.err
