#!/bin/bash
# A/B of the 64x32 ROF tiles (FT_ROF_WIDE=1) against the default 32x32 tiles,
# back to back on one box, plus the kernel-variant parity tests.
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -m gpu -q -k "variants" > gpurun_out/ab_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/ab_pytest.log
for r in 1 2; do
  for v in 0 1; do
    FT_ROF_WIDE=$v python bench.py --no-cpu-baseline > gpurun_out/ab_wide$v.$r.log 2>&1
    echo "wide=$v run=$r $(tail -1 gpurun_out/ab_wide$v.$r.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["e2e"]["value"])')"
  done
done
for v in 0 1; do
  FT_ROF_WIDE=$v python bench.py --no-cpu-baseline --flow light > gpurun_out/ab_light$v.log 2>&1
  echo "light wide=$v $(tail -1 gpurun_out/ab_light$v.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["e2e"]["value"])')"
done
