set -x
python -c "from paper_2508_13386_b200 import build as b; b.build(force=False)"
timeout 900 python -m pytest tests/test_gpu_bdf2.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/r2_pytest13.log 2>&1; echo "pytest rc=$?"; tail -20 gpurun_out/r2_pytest13.log
