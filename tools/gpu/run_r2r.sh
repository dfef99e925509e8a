set -x
python -c "from paper_2508_13386_b200 import build as b; b.build(force=False)"
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=12 > gpurun_out/r2_pytest15.log 2>&1; echo "pytest rc=$?"
tail -22 gpurun_out/r2_pytest15.log
