#!/bin/bash
# Sweep-kernel check: GPU parity suite with the default (k_pd_sweep) and an
# A/B of the default bench against the tile kernel and sweep segment sizes.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
ARGS=${ARGS:-"FT_PD_SWEEP=0 FT_PD_SWEEP=1 FT_SWEEP_SEG=32 FT_SWEEP_SEG=96 FT_SWEEP_SEG=144"}
for c in $ARGS; do env $c timeout 300 python bench.py --no-cpu-baseline > gpurun_out/ab.log 2>&1; tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$c', d['value'], d['e2e']['value'], r['ms_per_launch'], r['frac'], r['share_of_step'])" || tail -3 gpurun_out/ab.log; done
