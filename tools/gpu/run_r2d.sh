set -x
python -c "from paper_2508_13386_b200 import build as b; b.build(force=False)"
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "fullsize or dataflow or parity or basis" > gpurun_out/r2_pytest4.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r2_pytest4.log
timeout 600 python bench.py --steps 10 --warmup 5 --no-cpu-baseline > gpurun_out/r2_bench4_fused.json 2> gpurun_out/r2_bench4_fused.err; echo "bench rc=$?"
MSIM_GAL_FUSED=0 timeout 600 python bench.py --steps 10 --warmup 5 --no-cpu-baseline > gpurun_out/r2_bench4_unfused.json 2> gpurun_out/r2_bench4_unfused.err; echo "bench rc=$?"
tail -c 400 gpurun_out/r2_bench4_fused.err
export MSIM_GAL_FUSED=0
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_galerkin_fused --launch-skip 6 --launch-count 1 -o gpurun_out/r2_ncu_gal2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2_ncu_gal2.log 2>&1; echo "ncu rc=$?"
