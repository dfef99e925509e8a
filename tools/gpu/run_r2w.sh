python -c "from paper_2508_13386_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_galerkin_fused --csv python tools/gal_time.py 4 2>/dev/null | grep k_galerkin_fused | awk -F'","' '{print "gal", $NF}' | tail -3
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -p no:cacheprovider -k "coarse and not C5" 2>&1 | tail -2
