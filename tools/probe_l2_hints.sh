#!/bin/bash
# DRAM traffic and time of one config-5 slot-kernel launch (447,392 points) per
# library build variant (DDSG_B200_LIB): L2 eviction-priority hints
# (build.py DDSG_BUILD_DEFS=-DDDSG_SLOT_L2HINT=bits).
# Usage: bash tools/probe_l2_hints.sh libddsg_b200.so libddsg_b200_h3.so ...
mkdir -p gpurun_out
for lib in "$@"; do
  echo "== $lib"
  DDSG_B200_LIB=$lib python tools/probe_perf.py 5:447392 2>&1 | grep exact
  DDSG_B200_LIB=$lib ncu --clock-control none -k regex:fast_hdmr_kernel -c 1 \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_bytes.sum \
    python tools/profile_run.py 5 447392 1 2>&1 | grep -E "dram__|gpu__time|lts__"
done
