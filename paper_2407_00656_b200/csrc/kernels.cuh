// sm_100a kernels of the HGKS hot path.
//
// common.cuh: fp64 step control (Ctrl, CFL bound, min, time bookkeeping).
// hot.cuh:    the hot path, compiled for fp64 (p64, the parity path) and for
//             fp32 (p32, the FP32 variant of P:1098-1183).
// No tensor cores: there is no dense contraction on this path.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace hgks {
namespace p64 {
using Real = double;
using R2 = double2;
#include "hot.cuh"
}  // namespace p64
namespace p32 {
using Real = float;
using R2 = float2;
#include "hot.cuh"
}  // namespace p32
}  // namespace hgks
