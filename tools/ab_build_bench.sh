#!/bin/bash
# A/B tuning: build the library with each set of extra nvcc flags and run a short bench.
# usage: tools/ab_build_bench.sh tag "flags A" "flags B" ...
TAG=$1; shift
i=0
for flags in "$@"; do
  rm -f paper_2508_13386_b200/lib/libmsim.so
  MSIM_NVCC_EXTRA="$flags" python -c "from paper_2508_13386_b200 import build as b; b.build(force=True, verbose=False)" || { echo "$i: BUILD FAILED $flags" >> gpurun_out/${TAG}_flags.txt; i=$((i+1)); continue; }
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_$i.json 2>/dev/null
  echo "$i: $flags" >> gpurun_out/${TAG}_flags.txt
  i=$((i+1))
done
