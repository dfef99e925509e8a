set -x
python -c "from paper_2508_13386_b200 import build as b; b.build(force=False)"
timeout 600 python bench.py --steps 6 --warmup 4 --no-cpu-baseline > gpurun_out/r2_bench11_split.json 2> gpurun_out/r2_bench11_split.err; echo "bench rc=$?"
MSIM_GAL_SPLIT=0 timeout 600 python bench.py --steps 6 --warmup 4 --no-cpu-baseline > gpurun_out/r2_bench11_nosplit.json 2> gpurun_out/r2_bench11_nosplit.err; echo "bench rc=$?"
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "fullsize_coarse or basis_coarse" > gpurun_out/r2_pytest11.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_pytest11.log
