# C5 free-running parity on the paper's basis: GPU basis build (partition from .cache), oracle
# trajectory of 1 timestep on the box's CPU, GPU free-running log + the suite's C5x1 test.
export PYTHONUNBUFFERED=1
O=gpurun_out/c5fr; mkdir -p $O
python -c "from paper_2508_13386_b200 import build as b; b.build(force=False)" > $O/build.log 2>&1
timeout 2400 python tools/c5_basis_gpu.py /tmp/c5basis > $O/basis.log 2>&1 || { echo "basis failed" >> $O/basis.log; tail -5 $O/basis.log; exit 1; }
timeout 2700 python tools/oracle_fixtures.py traj 5 1 > $O/traj_fix.log 2>&1; echo "traj rc=$?" >> $O/traj_fix.log
timeout 600 python tools/freerun_log.py 5 $O/freerun_C5.json > $O/freerun.log 2>&1; echo "freerun rc=$?" >> $O/freerun.log
timeout 900 python -m pytest tests/test_gpu_newton_fullsize.py -k "C5x1" -q -rA -p no:cacheprovider > $O/pytest_fr.log 2>&1; echo "rc=$?" >> $O/pytest_fr.log
cp .cache/fixtures/traj_C5_1_v2.npz $O/ 2>/dev/null
tail -3 $O/basis.log; tail -3 $O/traj_fix.log; tail -5 $O/freerun.log; tail -3 $O/pytest_fr.log
