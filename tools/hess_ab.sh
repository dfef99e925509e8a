for mb in 2 3; do
  MSIM_NVCC_EXTRA="-DMSIM_HESS_MINB=$mb" python -c "from paper_2508_13386_b200 import build as b; b.build(force=True, verbose=False)"
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/hessab_$mb.json 2>/dev/null
done
