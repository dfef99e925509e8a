set -x
python -c "from paper_2508_13386_b200 import build as b; b.build(force=False)"
mkdir -p gpurun_out
timeout 900 python tools/freerun_log.py 3 gpurun_out/r02_freerun_C3.json > gpurun_out/r02_freerun_C3.log 2>&1; echo "rc=$?"
timeout 900 python tools/freerun_log.py 1 gpurun_out/r02_freerun_C1.json > gpurun_out/r02_freerun_C1.log 2>&1; echo "rc=$?"
grep -E "worst|newton_counts_equal|steps_compared" gpurun_out/r02_freerun_C3.json gpurun_out/r02_freerun_C1.json
tail -3 gpurun_out/r02_freerun_C3.log
