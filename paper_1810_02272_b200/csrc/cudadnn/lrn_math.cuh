// lrn_math.cuh — the arithmetic of LRN (ACROSS_CHANNELS, Caffe), written with
// explicitly rounded intrinsics so every kernel that evaluates it (the unfused
// ops_layers.cu kernels and the fused LRN + pooling kernels of ops_lrnpool.cu)
// performs the same operations in the same order: no FMA contraction choice is
// left to the compiler, so the results are bit-identical across kernels.
//
//   scale = k + alpha/n * sum_{window} x^2         (sum in window order)
//   y     = x * scale^-beta
//   dx    = dy * scale^-beta - (2 alpha beta / n) * x * sum_{c': c in window(c')} dy' y' / scale'
#pragma once

namespace cdnn {
namespace lrn {

__device__ __forceinline__ float fma_(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double fma_(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ float mul_(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float add_(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float sub_(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double sub_(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float div_(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double div_(double a, double b) { return __ddiv_rn(a, b); }

// running sum of squares: s + x*x (one rounding)
template <typename T>
__device__ __forceinline__ T sq_acc(T s, T x) { return fma_(x, x, s); }
// scale = k + aN * sum
template <typename T>
__device__ __forceinline__ T scale(T sum, T aN, T k) { return fma_(aN, sum, k); }
// float: the SFU's approximate base-2 logarithm / exponential / reciprocal (relative
// error ~2^-22; scale >= k > 0, so no denormal inputs) -- deterministic single
// instructions, where the IEEE-exact powf / division cost a function call each
__device__ __forceinline__ float lg2_(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float ex2_(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ double rcp_(double x) { return __drcp_rn(x); }
// scale^-beta
__device__ __forceinline__ float neg_pow(float sc, float beta) { return ex2_(mul_(-beta, lg2_(sc))); }
__device__ __forceinline__ double neg_pow(double sc, double beta) { return pow(sc, -beta); }
// forward top
template <typename T>
__device__ __forceinline__ T top(T x, T np) { return mul_(x, np); }
// backward window term dy * y / scale
__device__ __forceinline__ float term(float dy, float y, float sc) { return mul_(mul_(dy, y), rcp_(sc)); }
__device__ __forceinline__ double term(double dy, double y, double sc) { return div_(mul_(dy, y), sc); }
// backward: dy * np - coef * x * acc
template <typename T>
__device__ __forceinline__ T grad(T dy, T np, T coef, T x, T acc) { return sub_(mul_(dy, np), mul_(mul_(coef, x), acc)); }

}  // namespace lrn
}  // namespace cdnn
