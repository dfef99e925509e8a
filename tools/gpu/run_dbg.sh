export PYTHONUNBUFFERED=1
O=gpurun_out/r2traj; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_newton_fullsize.py -q -rA -p no:cacheprovider -k "free_running" > $O/traj.log 2>&1; echo "rc=$?" >> $O/traj.log
tail -12 $O/traj.log
