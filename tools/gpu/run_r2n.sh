set -x
python -c "from paper_2508_13386_b200 import build as b; b.build(force=False)"
./tools/bench_diag_bin
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "dataflow or fullsize_coarse or basis_coarse or newton_bootstrapped or subspace or coarse_pcg_fixed" > gpurun_out/r2_pytest12.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_pytest12.log
timeout 600 python bench.py --steps 6 --warmup 4 --no-cpu-baseline > gpurun_out/r2_bench12.json 2> gpurun_out/r2_bench12.err; echo "bench rc=$?"
