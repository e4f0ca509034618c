#!/bin/bash
# A/B: ROF interior-tile specialisation (default build) vs a build with
# -DFT_ROF_NO_IN, back to back on one box; parity suite of the default build.
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -m gpu -q > gpurun_out/ab_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/ab_pytest.log
NOIN=$PWD/paper_1910_06017_b200/libomnitrack_noin.so
for r in 1 2; do
  for v in in noin; do
    if [ $v = noin ]; then export FT_LIB=$NOIN; else unset FT_LIB; fi
    python bench.py --no-cpu-baseline --flow light > gpurun_out/ab_$v.$r.log 2>&1
    echo "light $v run=$r $(tail -1 gpurun_out/ab_$v.$r.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["e2e"]["value"])')"
  done
done
for v in in noin; do
  if [ $v = noin ]; then export FT_LIB=$NOIN; else unset FT_LIB; fi
  python bench.py --no-cpu-baseline > gpurun_out/ab_d$v.log 2>&1
  echo "default $v $(tail -1 gpurun_out/ab_d$v.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["e2e"]["value"])')"
done
