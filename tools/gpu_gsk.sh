for f in "" "-DMSIM_GAL_SKIP_A" "-DMSIM_GAL_SKIP_B"; do
  MSIM_NVCC_EXTRA="$f" python -c "from paper_2508_13386_b200 import build as b; b.build(force=True, verbose=False)" > /dev/null 2>&1
  echo "== $f" >> gpurun_out/gsk2.txt
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:galerkin --csv python tools/gal_time.py 4 2>/dev/null | grep -i "galerkin" | awk -F'","' '{print $5, $NF}' >> gpurun_out/gsk2.txt
done
python -c "from paper_2508_13386_b200 import build as b; b.build(force=True, verbose=False)"
