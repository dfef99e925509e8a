# assembly split (off-diagonal / diagonal parts) + compact 640-byte stage record: parity + C4 bench + ncu
mkdir -p gpurun_out; O=gpurun_out/r2x
python -c "from paper_2508_13386_b200 import build as b; b.build(force=False)" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > ${O}_parity.log 2>&1; echo "parity rc=$?" >> ${O}_parity.log
timeout 600 python bench.py --config 4 --steps 20 --warmup 5 --no-cpu-baseline > ${O}_bench_c4.json 2> ${O}_bench_c4.err
for k in k_assemble k_elem_hess; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"$k\$" -s 25 -c 1 -o ${O}_$k \
    python bench.py --steps 2 --warmup 6 --no-cpu-baseline > ${O}_$k.log 2>&1
  ncu -i ${O}_$k.ncu-rep --page raw --csv > ${O}_${k}_raw.csv 2>/dev/null
  ncu -i ${O}_$k.ncu-rep --page details --csv > ${O}_${k}_details.csv 2>/dev/null
  rm -f ${O}_$k.ncu-rep
done
timeout 1200 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_newton_fullsize.py -q -p no:cacheprovider -k "not C5" > ${O}_fullsize.log 2>&1; echo "fullsize rc=$?" >> ${O}_fullsize.log
