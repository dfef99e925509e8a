for v in "" "-DMSIM_GAL_SKIP_A" "-DMSIM_GAL_SKIP_B"; do
  MSIM_NVCC_EXTRA="$v" python -c "from paper_2508_13386_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_galerkin_fused --csv python tools/gal_time.py 4 2>/dev/null | grep k_galerkin_fused | awk -F'","' -v V="$v" '{print V, $NF}' | tail -3
done
