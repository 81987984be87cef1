#!/bin/bash
# Round-end measurement pass on the GPU box (run via gpurun from the repo root):
# GPU tests, the default bench line, the reference arm, the ncu launch list of
# the bench command and one full ncu capture of the slot kernel at the bench's
# launch size, the IRBC caller workloads.  Outputs land in gpurun_out/;
# tools/summarize_profiles.py <round> turns them into profiles/<round>_*.json.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.txt 2>&1; tail -1 gpurun_out/pytest_gpu.txt
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 300 gpurun_out/bench_default.json
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -c 200 gpurun_out/bench_ref.json
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-refine > gpurun_out/ncu_launch.log 2>&1; echo "launch list rc=$?"
timeout 300 python tools/profile_run.py 5 447392 1 > /dev/null 2>&1 && \
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:fast_hdmr_kernel -c 1 \
  -o gpurun_out/prof_final_config5 python tools/profile_run.py 5 447392 1 > gpurun_out/ncu_full.log 2>&1; echo "full capture rc=$?"
timeout 900 python bench.py --workload euler > gpurun_out/bench_euler.json 2> gpurun_out/bench_euler.err; tail -c 200 gpurun_out/bench_euler.json
timeout 900 python bench.py --workload jacobian > gpurun_out/bench_jacobian.json 2> gpurun_out/bench_jacobian.err; tail -c 200 gpurun_out/bench_jacobian.json
