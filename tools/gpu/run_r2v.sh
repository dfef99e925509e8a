python -c "from paper_2508_13386_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_galerkin_fused --csv python tools/gal_time.py 4 2>/dev/null | grep k_galerkin_fused | awk -F'","' '{print "gal", $NF}' | tail -3
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_coarse_pcg.py tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "not C5" 2>&1 | tail -3
timeout 600 python bench.py --steps 10 --warmup 5 --no-cpu-baseline > gpurun_out/r2v_bench.json 2> gpurun_out/r2v_bench.err; echo "bench rc=$?"
python -c "
import json; l=json.loads(open('gpurun_out/r2v_bench.json').read().strip().splitlines()[-1])
print(l['value'], l['phase_ms_per_newton'], l['roofline']['frac'])"
