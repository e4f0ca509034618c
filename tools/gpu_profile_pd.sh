# ncu --set full of the finest-level PD launch and of one ROF launch of the
# default bench command (run after the same command exited 0 without ncu)
CMD="python bench.py --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_pd_tile -s ${SKIP:-266} -c 1 \
    -o gpurun_out/pd_full $CMD > gpurun_out/ncu_full.log 2>&1; echo "pd full rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_rof_tile -s 13 -c 1 \
    -o gpurun_out/rof_full $CMD > gpurun_out/ncu_rof.log 2>&1; echo "rof full rc=$?"
