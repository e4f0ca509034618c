#!/bin/bash
# PD kernel cost model: ms per finest-level launch (timed alone by
# ft_tracker_profile_pd over the final state) vs PD iterations per launch
# (FT_PD_PROFILE_ITERS), for the tile configs / halos given.
for cfg in ${CFGS:-1}; do for halo in ${HALOS:-4}; do for it in ${ITERS:-0 1 2 3 4}; do
  out=$(FT_PD_CFG=$cfg FT_PD_HALO=$halo FT_PD_PROFILE_ITERS=$it timeout 300 python bench.py --steps 3 --warmup 3 --streams ${STREAMS:-32} --no-cpu-baseline 2>&1 | tail -1)
  python -c "import json,sys; d=json.loads(sys.argv[1]); r=d['roofline']['alone']; print('cfg=$cfg halo=$halo iters=$it ms_per_launch=%.4f' % r['ms_per_launch'])" "$out" || echo "cfg=$cfg halo=$halo iters=$it FAILED"
done; done; done
