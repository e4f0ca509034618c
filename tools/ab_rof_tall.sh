#!/bin/bash
# A/B: ROF 64x64 tiles (FT_ROF_TALL=1, 1024 threads) vs the default 64x32.
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -m gpu -q -k "variants" > gpurun_out/ab_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/ab_pytest.log
for r in 1 2; do
  for v in 0 1; do
    FT_ROF_TALL=$v python bench.py --no-cpu-baseline --flow light > gpurun_out/ab_tall$v.$r.log 2>&1
    echo "light tall=$v run=$r $(tail -1 gpurun_out/ab_tall$v.$r.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["e2e"]["value"])')"
  done
done
for v in 0 1; do
  FT_ROF_TALL=$v python bench.py --no-cpu-baseline > gpurun_out/ab_tdef$v.log 2>&1
  echo "default tall=$v $(tail -1 gpurun_out/ab_tdef$v.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["e2e"]["value"])')"
done
