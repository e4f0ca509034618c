# ncu of the pyramid / ingest stencil kernels of the default bench command
# (duration + DRAM bytes per launch), after the command ran clean without ncu.
CMD="python bench.py --no-cpu-baseline --steps 3 --warmup 3"
$CMD > gpurun_out/pyr_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"k_blur|k_gray8|k_scale_copy|k_central_grad|k_st_combine|k_upsample|k_median|k_warp_setup" \
    --csv --log-file gpurun_out/pyr.csv $CMD > gpurun_out/pyr_ncu.log 2>&1; echo "pyr ncu rc=$?"
