export PYTHONUNBUFFERED=1
O=gpurun_out/dbg6; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_coarse_pcg.py -q -p no:cacheprovider > $O/cpcg.log 2>&1; echo "rc=$?" >> $O/cpcg.log
MSIM_POISON=1 MSIM_NANCHECK=1 timeout 200 python -m pytest tests/test_gpu_coarse_pcg.py -q -x -p no:cacheprovider -k "not c4 and not c2" > $O/cpcg_poison.log 2>&1; echo "rc=$?" >> $O/cpcg_poison.log
for f in test_gpu_parity test_gpu_two_level test_gpu_bdf2 test_gpu_next2 test_gpu_multirank test_gpu_next3; do
  MSIM_POISON=1 timeout 240 python -m pytest tests/$f.py -q -p no:cacheprovider -k "not c4 and not C4 and not c2 and not C2" > $O/poison_$f.log 2>&1; echo "rc=$?" >> $O/poison_$f.log
done
tail -3 $O/cpcg.log; tail -3 $O/cpcg_poison.log; for f in $O/poison_*.log; do echo == $f; tail -4 $f | cut -c1-200; done
