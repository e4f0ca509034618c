# halo sweep with the shrinking cone (same box, back to back)
for h in 4 3 5 6 4; do FT_PD_HALO=$h python bench.py --no-cpu-baseline > gpurun_out/halo$h.log 2>&1; tail -1 gpurun_out/halo$h.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('halo=$h', d['value'], d['e2e']['value'], r['ms_per_launch'], r['frac'], r['share_of_step'])"; done
