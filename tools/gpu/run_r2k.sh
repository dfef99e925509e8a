set -x
python -c "from paper_2508_13386_b200 import build as b; b.build(force=False)"
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "element or fullsize_hessian or newton_bootstrapped or free_running" > gpurun_out/r2_pytest9.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r2_pytest9.log
timeout 600 python bench.py --steps 6 --warmup 4 --no-cpu-baseline > gpurun_out/r2_bench9.json 2> gpurun_out/r2_bench9.err; echo "bench rc=$?"
MSIM_DEBUG_HESS=1 timeout 600 python bench.py --steps 2 --warmup 4 --no-cpu-baseline 2>&1 | grep "hess:" | tail -8
