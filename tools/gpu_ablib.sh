#!/bin/bash
# A/B of two builds on one box: default lib vs $BASE (FT_LIB), alternating,
# for each bench argument set in $SETS (";"-separated).
mkdir -p gpurun_out
BASE=${BASE:-paper_1910_06017_b200/libbase.so}
SETS=${SETS:-"--no-cpu-baseline"}
IFS=';' read -ra SA <<< "$SETS"
for args in "${SA[@]}"; do
  for v in new base new base; do
    if [ $v = base ]; then export FT_LIB=$PWD/$BASE; else unset FT_LIB; fi
    timeout 300 python bench.py $args > gpurun_out/ab.log 2>&1
    tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$v [$args]', d['value'], r['ms_per_launch'], r['frac'])" || tail -3 gpurun_out/ab.log
  done
done
