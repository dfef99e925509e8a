set -x
python -c "from paper_2508_13386_b200 import build as b; b.build(force=False)"
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "fullsize or dataflow or parity or basis" > gpurun_out/r2_pytest3.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/r2_pytest3.log
timeout 600 python bench.py --steps 10 --warmup 5 --no-cpu-baseline > gpurun_out/r2_bench3_fused.json 2> gpurun_out/r2_bench3_fused.err; echo "bench rc=$?"
MSIM_GAL_FUSED=0 timeout 600 python bench.py --steps 10 --warmup 5 --no-cpu-baseline > gpurun_out/r2_bench3_unfused.json 2> gpurun_out/r2_bench3_unfused.err; echo "bench rc=$?"
tail -c 600 gpurun_out/r2_bench3_fused.err
