// Shared device helpers for the denseprop B200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/denseprop_b200.h"

namespace dp {

// ---------------------------------------------------------------------------
// Exact-order arithmetic.  The reference builds with -ffp-contract=off
// (pkg/setup.py:15): every multiply and add rounds separately.  The _rn
// intrinsics are never contracted into FFMA/DFMA regardless of -fmad.
// ---------------------------------------------------------------------------
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float div_rn(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }

// tanh: fp32 evaluates in fp64 and rounds once (<= 0.5 ulp + tiny), so it is
// within 2 ulp of numpy's float32 tanh (reference forward.py:71).
__device__ __forceinline__ float dp_tanh(float x) { return (float)tanh((double)x); }
__device__ __forceinline__ double dp_tanh(double x) { return tanh(x); }

// relu == np.maximum(x, 0) bit for bit: x when x > 0 or x is NaN, else +0.0
// (numpy returns the second operand on ties, so maximum(-0.0, 0) is +0.0).
template <typename T>
__device__ __forceinline__ T dp_relu(T x) { return (x > T(0) || x != x) ? x : T(0); }

// fast tier: tanh(x) = 1 - 2 / (1 + 2^(2 x log2 e)) from the MUFU ex2 / rcp approximations,
// x - x^3/3 below |x| = 1/16 (where the subtraction cancels): <= 3e-6 relative, ~10
// instructions against tanhf's ~18 (the pool forwards that fuse it are issue bound)
__device__ __forceinline__ float dp_tanh_fast(float x) {
    float e, r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(x * 2.8853900817779268f));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(1.0f + e));
    const float big = fmaf(-2.0f, r, 1.0f);
    const float small = fmaf(x * (x * x), -0.333333343f, x);
    return fabsf(x) < 0.0625f ? small : big;
}
__device__ __forceinline__ double dp_tanh_fast(double x) { return tanh(x); }

template <typename T>
__device__ __forceinline__ T apply_nonlin(T v, int kind) {
    if (kind == DP_TANH) return dp_tanh(v);
    if (kind == DP_TANH_FAST) return dp_tanh_fast(v);
    if (kind == DP_RELU) return dp_relu(v);
    return v;
}

// Derivative factor from the nonlinearity OUTPUT t (the engine caches outputs):
// tanh' = 1 - t*t (backward.py:176-177 computes it from t = tanh(x_in)),
// relu' = (x_in > 0) == (t > 0) (backward.py:179).
template <typename T>
__device__ __forceinline__ T gate_from_output(T delta, T t, int kind) {
    if (kind == DP_TANH || kind == DP_TANH_FAST)
        return mul_rn(delta, add_rn(T(1), -mul_rn(t, t)));
    if (kind == DP_RELU) return mul_rn(delta, t > T(0) ? T(1) : T(0));
    return delta;
}

template <typename T>
__device__ __forceinline__ T neg_inf();
template <>
__device__ __forceinline__ float neg_inf<float>() { return __int_as_float(0xff800000); }
template <>
__device__ __forceinline__ double neg_inf<double>() {
    return __longlong_as_double(0xfff0000000000000ULL);
}

inline int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }

}  // namespace dp

// error state + launch checking, implemented in capi.cu
namespace dp {
int set_error(int code, const char *fmt, ...);
int check_launch(const char *what);
}  // namespace dp
