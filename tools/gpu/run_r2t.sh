set -x
python -c "from paper_2508_13386_b200 import build as b; b.build(force=False)"
timeout 900 python -m pytest tests/test_gpu_next3.py -x -q -p no:cacheprovider > gpurun_out/r2t_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r2t_pytest.log
timeout 900 python tools/next3_compare.py > gpurun_out/r2t_next3.json 2> gpurun_out/r2t_next3.err; echo "compare rc=$?"
cat gpurun_out/r2t_next3.err | tail -5
