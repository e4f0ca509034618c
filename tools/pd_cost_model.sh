#!/bin/bash
# PD kernel cost model: ms per finest-level launch vs PD iterations per launch
# (FT_PD_PROFILE_ITERS), for the tile configs / halos given.
for cfg in ${CFGS:-1}; do for halo in ${HALOS:-3}; do for it in ${ITERS:-0 1 2 3}; do
  out=$(FT_PD_CFG=$cfg FT_PD_HALO=$halo FT_PD_PROFILE_ITERS=$it timeout 300 python bench.py --steps 1 --warmup 1 --streams ${STREAMS:-8} --no-cpu-baseline 2>&1 | tail -1)
  python -c "import json,sys; d=json.loads(sys.argv[1]); r=d['roofline']; print('cfg=$cfg halo=$halo iters=$it ms_per_launch=%.4f' % r['ms_per_launch'])" "$out" || echo "cfg=$cfg halo=$halo iters=$it FAILED"
done; done; done
