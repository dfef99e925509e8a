set -x
python -c "from paper_2508_13386_b200 import build as b; b.build(force=False)"
export MSIM_GAL_FUSED=0
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_galerkin_fused --launch-skip 6 --launch-count 1 -o gpurun_out/r2_ncu_gal python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2_ncu_gal.log 2>&1; echo "ncu rc=$?"
tail -5 gpurun_out/r2_ncu_gal.log
