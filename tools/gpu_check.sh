# quick GPU check: parity suite + cone A/B on the default bench
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for c in 1 0; do FT_PD_CONE=$c python bench.py --no-cpu-baseline > gpurun_out/cone$c.log 2>&1; tail -1 gpurun_out/cone$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('cone=$c', d['value'], d['e2e']['value'], r['ms_per_launch'], r['frac'], r['share_of_step'], r['alone'])"; done
