#!/bin/bash
# One GPU session on the box (run through gpurun from the repo root):
#   TAG=r02a TESTS=1 BENCH=1 PROFILE=1 bash tools/gpu_session.sh
# Writes logs/reports under gpurun_out/$TAG/.
set -u
TAG=${TAG:-s}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $OUT/smi.txt 2>&1
if [ "${TESTS:-0}" = 1 ]; then
  timeout ${TEST_TIMEOUT:-1800} python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > $OUT/gpu_tests.log 2>&1
  echo "tests rc=$?" >> $OUT/gpu_tests.log
  tail -3 $OUT/gpu_tests.log
fi
if [ "${SMOKE:-0}" = 1 ]; then
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
  tail -2 $OUT/smoke.log
fi
if [ "${BENCH:-0}" = 1 ]; then
  for cfg in ${BENCH_CONFIGS:-blast512}; do
    timeout 900 python bench.py --config $cfg --steps ${STEPS:-20} --warmup 5 ${BENCH_ARGS:-} > $OUT/bench_$cfg.json 2> $OUT/bench_$cfg.err
    echo "bench $cfg rc=$?"; tail -c 600 $OUT/bench_$cfg.json
  done
fi
if [ "${LAUNCHES:-0}" = 1 ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c ${NLAUNCH:-200} \
    ${LKERNEL:+-k regex:$LKERNEL} --csv \
    --log-file $OUT/launches.csv python bench.py --config ${LCFG:-blast512} --steps 2 --warmup 3 \
    --no-e2e --no-cpu-baseline --no-secondary > $OUT/launches.log 2>&1
  python tools/launch_shares.py $OUT/launches.csv > $OUT/launch_shares.txt 2>&1; cat $OUT/launch_shares.txt | head -12
fi
if [ "${PROFILE:-0}" = 1 ]; then
  timeout 1500 ncu --set full --import-source on --clock-control none -k regex:${PKERNEL:-sweep_kernel} \
    --launch-skip ${PSKIP:-18} --launch-count ${PCOUNT:-6} -o $OUT/prof -f \
    python bench.py --config ${PCFG:-blast256} --precision ${PPREC:-fast} --steps 3 --warmup 5 \
    --no-e2e --no-cpu-baseline --no-secondary > $OUT/prof.log 2>&1
  echo "profile rc=$?"; tail -3 $OUT/prof.log
fi
exit 0
