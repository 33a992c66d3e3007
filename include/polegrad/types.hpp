// polegrad/types.hpp — element type of every tensor in this build.
//
// Source-compatible with the reference's types.hpp:5-11: `real` is double by
// default and float under POLEGRAD_SINGLE_PRECISION.  The B200 library ships
// both builds (libpolegrad_b200_f64.so / _f32.so); float runs on the tcgen05
// TF32 tensor-core path, double on the SIMT FP64 path.
#pragma once

#include "cudadnn.h"

namespace polegrad {

#ifdef POLEGRAD_SINGLE_PRECISION
using real = float;
inline constexpr int kRealDtype = CDNN_F32;
#else
using real = double;
inline constexpr int kRealDtype = CDNN_F64;
#endif

}  // namespace polegrad
