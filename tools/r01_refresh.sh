#!/bin/bash
# Round-1 evidence refresh (run under gpurun): GPU parity suite, default
# bench line, reference arm, KLT bench line, launch list of the default
# command and one `ncu --set full` capture of a finest-level PD launch of the
# same command (after it exited 0 without ncu).
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"
python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
python bench.py --motion klt > gpurun_out/bench_klt.log 2>&1; echo "klt rc=$?"
CMD="python bench.py --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    $CMD > gpurun_out/ncu_launch.log 2>&1; echo "launch list rc=$?"
S=$(python tools/summarize_ncu.py --pick gpurun_out/launches.csv); echo "skip=$S"
ncu --set full --clock-control none --import-source on -k regex:k_pd_tile -s $S -c 1 \
    -o gpurun_out/pd_full $CMD > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"
KCMD="python bench.py --motion klt --no-cpu-baseline"
$KCMD > gpurun_out/kplain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_klt_points -s 2 -c 1 \
    -o gpurun_out/klt_full $KCMD > gpurun_out/ncu_klt.log 2>&1; echo "klt full rc=$?"
python bench.py --flow light > gpurun_out/bench_light.log 2>&1; echo "light rc=$?"
python bench.py --flow light --impl reference > gpurun_out/bench_light_ref.log 2>&1; echo "light ref rc=$?"
bash tools/gpu_pyr_profile.sh
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
