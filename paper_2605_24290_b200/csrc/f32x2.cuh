// Packed FP32 (sm_100a FFMA2 / FADD2 / FMUL2) and packed-bf16 helpers.
//
// Blackwell issues two FP32 lanes per instruction with the .f32x2 forms:
// one issue slot for two fused multiply-adds, each rounded exactly like the
// scalar fmaf / __fadd_rn / __fmul_rn.  ptxas folds scalar broadcast
// (make_float2(x, x)), operand swaps and per-lane negation into the SASS
// operand modifiers, so the helpers below cost one instruction each.
#pragma once

#include <cstdint>

#ifndef RXGS_RELU_CVT
#define RXGS_RELU_CVT 1
#endif

namespace rxgs_b200 {
namespace x2 {

__device__ __forceinline__ unsigned long long u64(float2 v) {
    return (static_cast<unsigned long long>(__float_as_uint(v.y)) << 32) | __float_as_uint(v.x);
}
__device__ __forceinline__ float2 f2(unsigned long long r) {
    return make_float2(__uint_as_float(static_cast<uint32_t>(r)), __uint_as_float(static_cast<uint32_t>(r >> 32)));
}

// a * b + c, per lane, round to nearest even
__device__ __forceinline__ float2 fma(float2 a, float2 b, float2 c) {
    unsigned long long r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(u64(a)), "l"(u64(b)), "l"(u64(c)));
    return f2(r);
}
__device__ __forceinline__ float2 add(float2 a, float2 b) {
    unsigned long long r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(u64(a)), "l"(u64(b)));
    return f2(r);
}
__device__ __forceinline__ float2 sub(float2 a, float2 b) {
    unsigned long long r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(u64(a)), "l"(u64(b)));
    return f2(r);
}
__device__ __forceinline__ float2 mul(float2 a, float2 b) {
    unsigned long long r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(u64(a)), "l"(u64(b)));
    return f2(r);
}
__device__ __forceinline__ float2 bc(float x) { return make_float2(x, x); }

// ReLU'd bf16 hi/lo split of two FP32 values, packed as bf16x2 (low half =
// a).  hi = a truncated to bf16 (same sign as a, |hi| <= |a|), lo = the exact
// FP32 remainder a - hi rounded to bf16 (same sign again), so max(., 0) on
// the packed halves is ReLU(a) split: hi + lo = relu(a) within 2^-16 |a|.
// The ReLU of lo rides on the conversion (F2FP.RELU): 6 instructions per
// pair (PRMT, 2 LOP3, FADD2, F2FP.RELU, HMNMX2).
__device__ __forceinline__ void relu_split_bf16(float a, float b, uint32_t& hi, uint32_t& lo) {
    uint32_t h;
    asm("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(h) : "r"(__float_as_uint(a)), "r"(__float_as_uint(b)));
    const float2 t = make_float2(__uint_as_float(__float_as_uint(a) & 0xFFFF0000u),
                                 __uint_as_float(__float_as_uint(b) & 0xFFFF0000u));
    const float2 r = sub(make_float2(a, b), t);
#if RXGS_RELU_CVT
    asm("cvt.rn.relu.bf16x2.f32 %0, %1, %2;" : "=r"(lo) : "f"(r.y), "f"(r.x));
#else
    uint32_t l;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(l) : "f"(r.y), "f"(r.x));
    asm("max.bf16x2 %0, %1, %2;" : "=r"(lo) : "r"(l), "r"(0u));
#endif
    asm("max.bf16x2 %0, %1, %2;" : "=r"(hi) : "r"(h), "r"(0u));
}

// Same split without the ReLU (layer-1 features).
__device__ __forceinline__ void split_bf16(float a, float b, uint32_t& hi, uint32_t& lo) {
    asm("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(hi) : "r"(__float_as_uint(a)), "r"(__float_as_uint(b)));
    const float2 t = make_float2(__uint_as_float(__float_as_uint(a) & 0xFFFF0000u),
                                 __uint_as_float(__float_as_uint(b) & 0xFFFF0000u));
    const float2 r = sub(make_float2(a, b), t);
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(lo) : "f"(r.y), "f"(r.x));
}

}  // namespace x2
}  // namespace rxgs_b200
