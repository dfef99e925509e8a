set -x
python -c "from paper_2508_13386_b200 import build as b; b.build(force=False)"
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "coarse or fullsize_coarse or basis_coarse or newton_bootstrapped" > gpurun_out/r2_pytest8.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r2_pytest8.log
timeout 600 python bench.py --steps 6 --warmup 4 --no-cpu-baseline > gpurun_out/r2_bench8.json 2> gpurun_out/r2_bench8.err; echo "bench rc=$?"
