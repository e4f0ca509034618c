# A/B of env settings on the default bench, same box: ARGS="FT_X=1 FT_X=0 ..."
for c in $ARGS; do env $c python bench.py --no-cpu-baseline > gpurun_out/ab.log 2>&1; tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$c', d['value'], d['e2e']['value'], r['ms_per_launch'], r['frac'], r['share_of_step'])" || tail -3 gpurun_out/ab.log; done
