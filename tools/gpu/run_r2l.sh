set -x
python -c "from paper_2508_13386_b200 import build as b; b.build(force=False)"
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=8 > gpurun_out/r2_pytest10.log 2>&1; echo "pytest rc=$?"
tail -14 gpurun_out/r2_pytest10.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench10.json 2> gpurun_out/r2_bench10.err; echo "bench rc=$?"
tail -c 1500 gpurun_out/r2_bench10.json
