#!/bin/bash
# Final round-1 check: GPU parity suite, smoke, and the bench lines (headline,
# reference arm, light, KLT, C3 / C4 non-headline configs).
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"
python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
python bench.py --flow light > gpurun_out/bench_light.log 2>&1; echo "light rc=$?"
python bench.py --motion klt > gpurun_out/bench_klt.log 2>&1; echo "klt rc=$?"
python bench.py --config c3 --streams 32 > gpurun_out/bench_c3.log 2>&1; echo "c3 rc=$?"
python bench.py --config c4 --streams 8 > gpurun_out/bench_c4.log 2>&1; echo "c4 rc=$?"
