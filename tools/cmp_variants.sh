set -x
for cfg in blast512 mag160; do
for v in default cs0mb3 cs1mb2 cs0mb2; do
  if [ $v = default ]; then unset PPMLR_LIB; else export PPMLR_LIB=variants/$v/libppmlr_b200.so; fi
  echo "== $cfg $v"; timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['value']/1e9, d['ms_per_step'], r['per_launch']['avg_ms'], r['frac'])"
done; done
