#!/bin/bash
# Rebuild (abort loudly on failure), then run a command on the B200 via gpurun.
set -e
cd /root/repo
python paper_2202_06555_b200/build.py > /tmp/ddsg_build.log 2>&1 || { grep -E "error" -A3 /tmp/ddsg_build.log | head -30; echo "BUILD FAILED"; exit 1; }
exec /usr/local/graft/bin/gpurun --timeout "${GPU_TIMEOUT:-900}" -- "$@"
