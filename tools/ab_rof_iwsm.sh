#!/bin/bash
# A/B: ROF img/weight in shared memory (-DFT_ROF_IWSM build, no spills) vs the
# default build (img/weight in registers), back to back; parity of the alt build.
mkdir -p gpurun_out
ALT=$PWD/paper_1910_06017_b200/libomnitrack_iwsm.so
FT_LIB=$ALT python -m pytest tests/test_gpu_parity.py -m gpu -q > gpurun_out/ab_pytest.log 2>&1; echo "pytest(alt) rc=$?"; tail -1 gpurun_out/ab_pytest.log
for r in 1 2; do
  for v in reg sm; do
    if [ $v = sm ]; then export FT_LIB=$ALT; else unset FT_LIB; fi
    python bench.py --no-cpu-baseline --flow light > gpurun_out/ab_$v.$r.log 2>&1
    echo "light $v run=$r $(tail -1 gpurun_out/ab_$v.$r.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["e2e"]["value"])')"
  done
done
for v in reg sm; do
  if [ $v = sm ]; then export FT_LIB=$ALT; else unset FT_LIB; fi
  python bench.py --no-cpu-baseline > gpurun_out/ab_d$v.log 2>&1
  echo "default $v $(tail -1 gpurun_out/ab_d$v.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["e2e"]["value"])')"
done
