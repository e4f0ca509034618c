#!/bin/bash
# k_pd_sweep: GPU parity, A/B bench, ncu --set full of one finest-level
# middle launch (frame 1, level 0) of the default bench command.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log

for c in ${ARGS:-FT_PD_SWEEP=0 FT_PD_SWEEP=1}; do env $c timeout 300 python bench.py --no-cpu-baseline > gpurun_out/ab.log 2>&1; tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$c', d['value'], d['e2e']['value'], r['ms_per_launch'], r['frac'], r['share_of_step'])" || tail -3 gpurun_out/ab.log; done
CMD="python bench.py --no-cpu-baseline --steps 2 --warmup 3"
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"k_pd_sweep<\\(int\\)8" -s ${SKIP:-230} -c 1 -o gpurun_out/sweep_full -f $CMD > gpurun_out/ncu_sweep.log 2>&1; echo "ncu rc=$?"
