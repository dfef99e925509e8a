#!/bin/bash
# Full GPU suite + smoke + default bench (+ optional ncu launch list).  usage: TAG=x tools/gpu_suite.sh
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
T=${TAG:-suite}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/${T}_gpu.txt 2>&1
python -c "from paper_2508_13386_b200 import build as b; b.build()" > gpurun_out/${T}_build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q ${PYTEST_EXTRA} > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${T}_smoke.log
if [ -z "$NO_BENCH" ]; then
timeout 900 python bench.py ${BENCH_ARGS:---steps 20 --warmup 5} > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?" >> gpurun_out/${T}_bench.err
fi
echo done
