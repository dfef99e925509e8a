# Round-2 profiling pass (run under gpurun, one GPU): the bench's launch list and one ncu --set full
# capture per hot kernel in a contact step of C4; the CSV exports are kept, the .ncu-rep dropped.
set -x
python -c "from paper_2508_13386_b200 import build as b; b.build(force=False)"
OUT=gpurun_out/prof_r02
mkdir -p $OUT
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file $OUT/launches.csv \
  python bench.py --steps 2 --warmup 6 --no-cpu-baseline > $OUT/launches_bench.log 2>&1; echo "launch list rc=$?"
python tools/launch_summary.py $OUT/launches.csv $OUT/launches_summary.txt | head -30
for k in k_chol_dataflow k_galerkin_fused k_elem_hess k_assemble k_pcg_spmv k_pcg_update; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$k\$" -s 25 -c 1 -o $OUT/$k \
    python bench.py --steps 2 --warmup 6 --no-cpu-baseline > $OUT/$k.log 2>&1
  echo "$k rc=$?"
  ncu -i $OUT/$k.ncu-rep --page raw --csv > $OUT/${k}_raw.csv 2>/dev/null
  ncu -i $OUT/$k.ncu-rep --page details --csv > $OUT/${k}_details.csv 2>/dev/null
  rm -f $OUT/$k.ncu-rep
done
ls -la $OUT
