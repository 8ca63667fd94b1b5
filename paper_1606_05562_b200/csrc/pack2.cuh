// pack2.cuh — two float32 lanes processed by one FADD2/FFMA2 (sm_100): the
// butterfly networks of net16.cuh run on F2 values to transform two blocks
// with one instruction per addition.
#pragma once

namespace dct16a {

struct F2 {
    float2 v;
};
__device__ __forceinline__ F2 operator+(F2 a, F2 b) { return F2{__fadd2_rn(a.v, b.v)}; }
__device__ __forceinline__ F2 operator-(F2 a, F2 b) { return F2{__fadd2_rn(a.v, make_float2(-b.v.x, -b.v.y))}; }
__device__ __forceinline__ F2 operator-(F2 a) { return F2{make_float2(-a.v.x, -a.v.y)}; }
__device__ __forceinline__ F2 fma2(F2 a, F2 b, F2 c) { return F2{__ffma2_rn(a.v, b.v, c.v)}; }

}  // namespace dct16a
