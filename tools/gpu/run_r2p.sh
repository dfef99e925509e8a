set -x
python -c "from paper_2508_13386_b200 import build as b; b.build(force=False)"
timeout 900 python -m pytest tests/test_gpu_next2.py tests/test_gpu_multirank.py tests/test_gpu_fullsize.py tests/test_gpu_parity.py tests/test_gpu_coarse_pcg.py tests/test_gpu_bdf2.py -q -x -p no:cacheprovider > gpurun_out/r2_pytest14.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/r2_pytest14.log
