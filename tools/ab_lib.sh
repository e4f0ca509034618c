# A/B of the current library against $OLD (FT_LIB), alternating, same box:
# default bench (64 SD streams), phases per level.
OLD=${OLD:-build_old.so}
for r in 1 2; do
  for v in new old; do
    if [ $v = old ]; then export FT_LIB=$PWD/$OLD; else unset FT_LIB; fi
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_$v.$r.json 2>gpurun_out/ab_$v.$r.err
    python -c "
import json; d=json.loads(open('gpurun_out/ab_$v.$r.json').read().strip().splitlines()[-1]); p=d['phases_ms']; r=d['roofline'] or {}
print('$v', d['value'], d['e2e']['value'], r.get('ms_per_launch'), [round(p['flow level %d' % l],2) for l in range(6)], round(p['structure_texture'],3))"
  done
done
unset FT_LIB
