# A/B of library builds on the light-params bench (ROF-heavy), same box
for c in $ARGS; do env $c python bench.py --flow light --no-cpu-baseline --steps 20 > gpurun_out/ab.log 2>&1; tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['value'], d['e2e']['value'])" || tail -3 gpurun_out/ab.log; done
