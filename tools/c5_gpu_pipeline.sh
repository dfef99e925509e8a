#!/bin/bash
# One GPU-box session for C5 with the paper's basis: GPU basis build, oracle fixtures (box CPU),
# parity tests, bench line, free-running log.  Results under gpurun_out/c5p_*; basis chunks in
# /tmp/c5basis (fetched by follow-up calls).
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
O=gpurun_out/c5p
timeout 4000 python tools/c5_basis_gpu.py /tmp/c5basis > ${O}_basis.log 2>&1 || { echo "basis failed" >> ${O}_basis.log; exit 1; }
timeout 1200 python tools/oracle_fixtures.py newton 5 > ${O}_newton_fix.log 2>&1
cp .cache/fixtures/newton_C5_v2.npz gpurun_out/ 2>/dev/null
timeout 1200 python -m pytest tests/test_gpu_newton_fullsize.py tests/test_gpu_fullsize.py -k "C5 and not standin" -q -rA > ${O}_pytest.log 2>&1; echo "rc=$?" >> ${O}_pytest.log
timeout 900 python bench.py --config 5 --steps 4 --warmup 1 > ${O}_bench.json 2> ${O}_bench.err
timeout 2400 python tools/oracle_fixtures.py traj 5 1 > ${O}_traj_fix.log 2>&1
cp .cache/fixtures/traj_C5_1_v2.npz gpurun_out/ 2>/dev/null
timeout 600 python tools/freerun_log.py 5 gpurun_out/c5p_freerun_C5.json > ${O}_freerun.log 2>&1
timeout 900 python -m pytest tests/test_gpu_newton_fullsize.py -k "C5x1" -q -rA > ${O}_pytest_fr.log 2>&1
cp /tmp/c5basis/*.part0 gpurun_out/ 2>/dev/null
ls -la /tmp/c5basis > ${O}_chunks.txt
echo done
