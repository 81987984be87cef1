#!/bin/bash
# ncu --set full capture of the tile-staged plain kernel on config 2 or 3.
# Usage: bash tools/ncu_tiled.sh <config> <points> <out-name>
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:tiled_kernel -c 1 -o gpurun_out/$3 -f \
  python tools/profile_run.py $1 $2 1 > gpurun_out/$3.log 2>&1
ncu -i gpurun_out/$3.ncu-rep --page raw --csv > gpurun_out/$3_raw.csv 2>/dev/null
ncu -i gpurun_out/$3.ncu-rep --page source --csv > gpurun_out/$3_source.csv 2>/dev/null
ls -la gpurun_out/$3*
