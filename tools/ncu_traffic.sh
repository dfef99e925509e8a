#!/bin/bash
# One ncu --set full capture per listed kernel (C4 bench, after warm-up) -> gpurun_out/<tag>_<kernel>.ncu-rep
TAG=$1; shift
for k in "$@"; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"^$k\$" -s 2 -c 1 -o gpurun_out/${TAG}_$k \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_$k.log 2>&1
done
