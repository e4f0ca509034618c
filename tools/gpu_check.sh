# quick GPU check: parity suite (default + FT_PD_CQ=0) + A/B of a PD switch on the default bench
VAR=${VAR:-FT_PD_CQ}
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for c in 1 0 1; do env $VAR=$c python bench.py --no-cpu-baseline > gpurun_out/ab$c.log 2>&1; tail -1 gpurun_out/ab$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$VAR=$c', d['value'], d['e2e']['value'], r['ms_per_launch'], r['frac'], r['share_of_step'])"; done
