#!/bin/bash
# Sweep the PD tile configuration / halo on one GPU (FT_PD_CFG, FT_PD_HALO).
mkdir -p gpurun_out
for cfg in ${CFGS:-0 1 2 3}; do
  for halo in ${HALOS:-4 6}; do
    out=$(FT_PD_CFG=$cfg FT_PD_HALO=$halo timeout 300 python bench.py --steps ${STEPS:-3} --warmup 1 --streams ${STREAMS:-8} --no-cpu-baseline 2>&1 | tail -1)
    python - "$cfg" "$halo" "$out" <<'PY'
import json, sys
cfg, halo, line = sys.argv[1], sys.argv[2], sys.argv[3]
try:
    d = json.loads(line)
    r = d["roofline"]
    print(f"cfg={cfg} halo={halo} fps={d['value']:.1f} e2e={d['e2e']['value']:.1f} ms/step={d['ms_per_step']:.2f} pd_ms={r['ms_per_launch']:.4f} iters={r['iters_per_launch']} frac={r['frac']}")
except Exception as e:
    print(f"cfg={cfg} halo={halo} FAILED: {line[-300:]}")
PY
  done
done
