# A/B/C... of several library builds (FT_LIB), alternating, same box:
# default bench (64 SD streams).  usage: bash tools/ab_multi.sh a.so b.so ...
for r in 1 2; do
  for lib in "$@"; do
    export FT_LIB=$PWD/$lib
    tag=$(basename $lib .so)
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/abm_$tag.$r.json 2>gpurun_out/abm_$tag.$r.err
    python -c "
import json; d=json.loads(open('gpurun_out/abm_$tag.$r.json').read().strip().splitlines()[-1]); p=d['phases_ms']; r=d['roofline'] or {}
print('$tag', d['value'], d['e2e']['value'], r.get('ms_per_launch'), [round(p['flow level %d' % l],2) for l in range(6)], round(p['structure_texture'],3))"
  done
done
unset FT_LIB
