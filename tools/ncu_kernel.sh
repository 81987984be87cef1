#!/bin/bash
# ncu --set full capture of one launch of a kernel (regex) on a config.
# Usage: bash tools/ncu_kernel.sh <kernel-regex> <config> <points> <out-name>
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:$1 -c 1 -o gpurun_out/$4 -f \
  python tools/profile_run.py $2 $3 1 > gpurun_out/$4.log 2>&1
ncu -i gpurun_out/$4.ncu-rep --page raw --csv > gpurun_out/$4_raw.csv 2>/dev/null
ncu -i gpurun_out/$4.ncu-rep --page source --csv > gpurun_out/$4_source.csv 2>/dev/null
ls -la gpurun_out/$4*
