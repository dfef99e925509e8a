set -x
nvidia-smi --query-gpu=name,memory.total --format=csv
python -c "from paper_2508_13386_b200 import build as b; b.build(force=False)"
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/r2_pytest2.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/r2_pytest2.log
