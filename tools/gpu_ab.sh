#!/bin/bash
# A/B of library build flags: parity subset, Galerkin launch times under ncu, short bench.
# usage: TAG=x TESTS="pytest args" tools/gpu_ab.sh "flags A" "flags B" ...
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
i=0
for flags in "$@"; do
  MSIM_NVCC_EXTRA="$flags" python -c "from paper_2508_13386_b200 import build as b; b.build(force=True, verbose=False)" > gpurun_out/${TAG}_${i}_build.log 2>&1 || { echo "$i BUILD FAILED" >> gpurun_out/${TAG}_summary.txt; i=$((i+1)); continue; }
  echo "== $i: $flags" >> gpurun_out/${TAG}_summary.txt
  if [ -n "$TESTS" ]; then timeout 900 python -m pytest $TESTS -x -q > gpurun_out/${TAG}_${i}_pytest.log 2>&1; tail -1 gpurun_out/${TAG}_${i}_pytest.log >> gpurun_out/${TAG}_summary.txt; fi
  if [ -n "$KREGEX" ]; then timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:$KREGEX --csv python tools/gal_time.py 4 2>/dev/null | grep -i "$KREGEX" | awk -F'","' '{print $5, $NF}' | sort | uniq -c | head -8 >> gpurun_out/${TAG}_summary.txt; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_${i}_bench.json 2> gpurun_out/${TAG}_${i}_bench.err
  python -c "
import json; d=json.loads(open('gpurun_out/${TAG}_${i}_bench.json').read()); print('bench', round(d['value'],2), {k: round(v,3) for k,v in d['phase_ms_per_newton'].items()})" >> gpurun_out/${TAG}_summary.txt 2>&1
  i=$((i+1))
done
python -c "from paper_2508_13386_b200 import build as b; b.build(force=True, verbose=False)"
