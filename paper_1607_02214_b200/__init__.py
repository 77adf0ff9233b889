"""B200-native PPMLR-MHD time-step hot path (arXiv 1607.02214 reference).

The numerics live in ``libppmlr_b200.so`` (hand-written sm_100a FP64 CUDA
kernels behind the C-ABI in ``include/ppmlr_gpu.h``); this package is the
thin host-side mirror of the reference's API.  Importing it fails loudly if
the native library has not been built — there is no CPU fallback.
"""
from .api import (FAST, IC_BLAST, IC_BRIOWU, IC_GAUSSIAN, IC_ORSZAG_TANG, IC_PARTITION,  # noqa
                  IC_SMOOTH, IC_UNIFORM, MAGNETOSPHERE, OUTFLOW, PERIODIC, STRICT, Axis,
                  AxisSpec, Block, BlockInfo, Error, Harness, HarnessOptions, InvalidSpec,
                  OutOfRange, RuntimeFailure, SolarWindParams, StepRejected, UnphysicalState,
                  build_axis, device_count, exchanged_bytes, host_block_state, layout,
                  strip_max_dt, sweep_strips, tde_units, version)

__all__ = [n for n in dir() if not n.startswith("_")]
