set -x
python -c "from paper_2508_13386_b200 import build as b; b.build(force=False)"
timeout 900 python -m pytest tests/test_gpu_dataflow.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider > gpurun_out/r2u_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r2u_pytest.log
timeout 600 python bench.py --steps 10 --warmup 5 --no-cpu-baseline > gpurun_out/r2u_bench.json 2> gpurun_out/r2u_bench.err; echo "bench rc=$?"
python -c "
import json; l=json.loads(open('gpurun_out/r2u_bench.json').read().strip().splitlines()[-1])
print(l['value'], l['phase_ms_per_newton'], l['roofline']['frac'])"
