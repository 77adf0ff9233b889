#!/bin/bash
# A/B of native-library variants on the GPU box: parity subset, then timing.
#   VARIANTS="default tl96" CONFIGS="blast512 mag160" PREC="fast strict" bash tools/ab.sh
mkdir -p gpurun_out/ab
for v in ${VARIANTS:-default}; do
  if [ "$v" = default ]; then unset PPMLR_LIB; else export PPMLR_LIB=variants/$v/libppmlr_b200.so; fi
  if [ "${PARITY:-1}" = 1 ]; then
    timeout 900 python -m pytest -q -x tests/test_gpu_baseline.py tests/test_gpu_parity.py \
      -k "${PARITY_K:-not slow and not c2_ and not c3_ and not division}" > gpurun_out/ab/parity_$v.log 2>&1
    echo "$v parity: $(tail -1 gpurun_out/ab/parity_$v.log)"
  fi
done
unset PPMLR_LIB
bash tools/cmp_variants.sh
