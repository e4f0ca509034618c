#!/bin/bash
# Evidence refresh after the 64x32 ROF tiles became the default: GPU suite,
# smoke, bench lines (default / light / KLT / C3 / C4), the launch list of the
# default command and one `ncu --set full` capture of a k_rof_tile launch.
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"
python bench.py --flow light > gpurun_out/bench_light.log 2>&1; echo "light rc=$?"
python bench.py --motion klt > gpurun_out/bench_klt.log 2>&1; echo "klt rc=$?"
python bench.py --config c3 --streams 32 > gpurun_out/bench_c3.log 2>&1; echo "c3 rc=$?"
python bench.py --config c4 --streams 8 > gpurun_out/bench_c4.log 2>&1; echo "c4 rc=$?"
CMD="python bench.py --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    $CMD > gpurun_out/ncu_launch.log 2>&1; echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_rof_tile -s 40 -c 1 \
    -o gpurun_out/rof_full $CMD > gpurun_out/ncu_rof.log 2>&1; echo "rof full rc=$?"
