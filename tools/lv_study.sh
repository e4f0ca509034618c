# Whole-level PD kernel study: default vs no-exchange timing build (FT_LIB),
# then ncu of one finest-level k_pd_level launch.
set -x
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/lv_a.json 2>gpurun_out/lv_a.err
FT_LIB=$PWD/build_nosync.so python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/lv_b.json 2>gpurun_out/lv_b.err
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --pd-kernel tiled > gpurun_out/lv_c.json 2>gpurun_out/lv_c.err
for f in a b c; do python -c "
import json; d=json.loads(open('gpurun_out/lv_$f.json').read().strip().splitlines()[-1]); p=d['phases_ms']; print('$f', d['value'], p['flow level 0'], p['flow level 1'], p['flow level 2'], p['flow level 3'])"; done
timeout 600 ncu --set full --import-source on -k regex:k_pd_level -s 40 -c 1 -o gpurun_out/lv_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline --streams 4 > gpurun_out/lv_ncu.log 2>&1
tail -3 gpurun_out/lv_ncu.log
