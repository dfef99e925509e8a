mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g1_gpu.txt 2>&1
timeout 60 ./tools/bench_diag_bin > gpurun_out/g1_diag.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_dataflow.py tests/test_gpu_parity.py "tests/test_gpu_fullsize.py" -k "not C5" -x -q > gpurun_out/g1_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g1_pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/g1_bench.json 2> gpurun_out/g1_bench.err
echo done
