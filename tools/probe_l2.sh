#!/bin/bash
# DRAM traffic and time of one config-5 slot-kernel launch per column-block
# group budget (DDSG_CB_BUDGET_MB).  Usage: bash tools/probe_l2.sh 16 32 64
mkdir -p gpurun_out
for b in "$@"; do
  echo "== budget ${b} MB"
  DDSG_CB_BUDGET_MB=$b python tools/probe_perf.py 5:447392 2>&1 | grep exact
  DDSG_CB_BUDGET_MB=$b ncu --clock-control none -k regex:fast_hdmr_kernel -c 1 \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
    python tools/profile_run.py 5 447392 1 2>&1 | grep -E "dram__|gpu__time|lts__"
done
