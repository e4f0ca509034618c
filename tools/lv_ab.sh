# A/B of the PD kernels on the default bench: whole-level (auto), its
# no-exchange timing build (FT_LIB, wrong results), and the tile kernel.
for f in a b c; do
  case $f in
    a) python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ab_$f.json 2>gpurun_out/ab_$f.err ;;
    b) FT_LIB=$PWD/build_nosync.so python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ab_$f.json 2>gpurun_out/ab_$f.err ;;
    c) python bench.py --steps 3 --warmup 3 --no-cpu-baseline --pd-kernel tiled > gpurun_out/ab_$f.json 2>gpurun_out/ab_$f.err ;;
  esac
  python -c "
import json; d=json.loads(open('gpurun_out/ab_$f.json').read().strip().splitlines()[-1]); p=d['phases_ms']; print('$f', d['value'], [round(p['flow level %d' % l],2) for l in range(6)])"
done
