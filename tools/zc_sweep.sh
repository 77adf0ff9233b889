for zc in 0 32 24 16 12 8; do
  for cfg in mag160 ot512; do
  printf "zc=%-3s %-8s " $zc $cfg
  PPMLR_SRC_ZCHUNK=$zc timeout 300 python bench.py --config $cfg --precision fast --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary 2>/dev/null | python -c "
import json, sys
d = json.loads(sys.stdin.read()); r = d['roofline']
print(f\"{d['value']/1e9:.4f} Gcu/s  {d['ms_per_step']:.4f} ms/step  sweep {r['per_launch']['avg_ms']:.4f}\")"
  done
done
