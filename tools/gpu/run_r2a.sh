set -x
nvidia-smi --query-gpu=name,memory.total --format=csv
python -c "from paper_2508_13386_b200 import build as b; b.build(force=False)"
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=15 > gpurun_out/r2_pytest1.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/r2_pytest1.log
timeout 900 python bench.py --steps 10 --warmup 5 > gpurun_out/r2_bench1.json 2> gpurun_out/r2_bench1.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/r2_bench1.json
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2_ref1.json 2> gpurun_out/r2_ref1.err; echo "ref rc=$?"
cat gpurun_out/r2_ref1.json
nproc; lscpu | head -20
