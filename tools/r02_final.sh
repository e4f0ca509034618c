# Round-2 evidence run on one B200: GPU suite, bench lines (headline, light,
# KLT, C3, C4, single stream, strong-scaling split), reference arm, ncu launch
# list and full captures of the dominant kernels.  Outputs in gpurun_out/r02_*.
set -u
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $O/r02_gpu.txt
timeout 1500 python -m pytest tests -m gpu -q > $O/r02_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/r02_pytest_gpu.log
timeout 900 python bench.py > $O/r02_bench_default.jsonl 2> $O/r02_bench_default.err; echo "default rc=$?"
timeout 600 python bench.py --flow light --no-cpu-baseline > $O/r02_bench_light.jsonl 2>&1; echo "light rc=$?"
timeout 900 python bench.py --motion klt > $O/r02_bench_klt.jsonl 2>&1; echo "klt rc=$?"
timeout 600 python bench.py --config c3 --streams 32 --no-cpu-baseline > $O/r02_bench_c3.jsonl 2>&1; echo "c3 rc=$?"
timeout 600 python bench.py --config c4 --streams 8 --no-cpu-baseline > $O/r02_bench_c4.jsonl 2>&1; echo "c4 rc=$?"
timeout 600 python bench.py --streams 1 --steps 20 --no-cpu-baseline > $O/r02_bench_single.jsonl 2>&1; echo "single rc=$?"
timeout 600 python bench.py --total-streams 64 --no-cpu-baseline > $O/r02_bench_total64.jsonl 2>&1; echo "total64 rc=$?"
timeout 120 python bench.py --gpus 2 > $O/r02_bench_gpus2.txt 2>&1; echo "gpus2 rc=$? (one-GPU box: must refuse)"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 --ref-budget-s 120 > $O/r02_bench_reference.jsonl 2>&1; echo "reference rc=$?"
# launch list of one default step (ncu serialises; shares only)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2300 --csv \
  --log-file $O/r02_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/r02_ncu_list.log 2>&1; echo "ncu list rc=$?"
# full captures: a finest-level middle primal-dual launch, a ROF launch
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_pd_tile -s 300 -c 1 \
  -o $O/r02_pd_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/r02_ncu_pd.log 2>&1; echo "ncu pd rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_rof_tile -s 30 -c 1 \
  -o $O/r02_rof_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/r02_ncu_rof.log 2>&1; echo "ncu rof rc=$?"
