#!/bin/bash
# A/B timing of native-library variants (tools/variants.py) on the GPU box:
#   VARIANTS="default head" CONFIGS="blast512 mag160" PREC="fast strict" bash tools/cmp_variants.sh
for cfg in ${CONFIGS:-blast512 mag160}; do
for prec in ${PREC:-fast}; do
for v in ${VARIANTS:-default}; do
  if [ "$v" = default ]; then unset PPMLR_LIB; else export PPMLR_LIB=variants/$v/libppmlr_b200.so; fi
  printf "%-10s %-7s %-10s " "$cfg" "$prec" "$v"
  timeout 300 python bench.py --config "$cfg" --precision "$prec" --steps 10 --warmup 3 \
      --no-e2e --no-cpu-baseline --no-secondary 2>/dev/null | python -c "
import json, sys
d = json.loads(sys.stdin.read()); r = d['roofline']
print(f\"{d['value']/1e9:.4f} Gcu/s  {d['ms_per_step']:.3f} ms/step  sweep {r['per_launch']['avg_ms']:.3f} ms  frac {r['frac']:.4f}\")"
done; done; done
