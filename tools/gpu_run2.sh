mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-g2}
timeout 60 ./tools/bench_diag_bin > gpurun_out/${T}_diag.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_dataflow.py "tests/test_gpu_fullsize.py" -k "not C5" -x -q > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
MSIM_NVCC_EXTRA=-DMSIM_CHAIN_PROF python -c "from paper_2508_13386_b200 import build as b; b.build(force=True, verbose=False)" > gpurun_out/${T}_prof_build.log 2>&1
timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${T}_chainprof.txt 2>&1
echo done
