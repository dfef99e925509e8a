# Round-2 final pass on HEAD (one B200): full GPU suite, smoke, driver-format C4 bench (both arms),
# launch list and one ncu --set full capture per hot kernel (contact step of C4).
export PYTHONUNBUFFERED=1
O=gpurun_out/r2final; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/gpu.txt 2>&1
python -c "from paper_2508_13386_b200 import build as b; b.build(force=False)" > $O/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench_c4.json 2> $O/bench_c4.err; echo "bench rc=$?" >> $O/bench_c4.err
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref rc=$?" >> $O/bench_reference.err
timeout 600 python bench.py --nccl1 --steps 10 --warmup 5 --no-cpu-baseline > $O/bench_c4_nccl1.json 2> $O/bench_c4_nccl1.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 6 --no-cpu-baseline > $O/launches_bench.log 2>&1; echo "launch list rc=$?" >> $O/launches_bench.log
python tools/launch_summary.py $O/launches.csv $O/launches_summary.txt > /dev/null 2>&1
for k in k_chol_dataflow k_galerkin_fused k_elem_hess k_assemble k_pcg_spmv k_pcg_update; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"^$k\$" -s 25 -c 1 -o $O/$k \
    python bench.py --steps 2 --warmup 6 --no-cpu-baseline > $O/$k.log 2>&1
  echo "$k rc=$?" >> $O/ncu_rc.txt
  if [ -f $O/$k.ncu-rep ]; then
    ncu -i $O/$k.ncu-rep --page raw --csv > $O/${k}_raw.csv 2>/dev/null
    ncu -i $O/$k.ncu-rep --page details --csv > $O/${k}_details.csv 2>/dev/null
    rm -f $O/$k.ncu-rep
  fi
done
python tools/ncu_summarise.py $O $O/traffic.json $O/ncu_summary.md > /dev/null 2>&1
ls -la $O
tail -3 $O/pytest_gpu.log; cat $O/smoke.log | tail -2; cat $O/bench_c4.json | cut -c1-400
