// Device helpers shared by the quantization kernels (prologue.cu, weights.cu).
// Rounding replicates the reference bit-for-bit (quantize.py:26-29, 115-117,
// 168-171): every float64 op is an explicit __dmul_rn / __dadd_rn / IEEE
// division, so nvcc cannot contract into FMA.
#pragma once
#include <cuda_fp16.h>
#include <cstdint>

namespace i8mm {

__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }

__device__ __forceinline__ uint4 ld_stream_u4(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ bool h_is_nonfinite(__half h) {
    return (__half_as_ushort(h) & 0x7C00u) == 0x7C00u;
}

// quantize.py:26-29 + 115-117: clip(copysign(floor(fl64(|p|+0.5)), p), +-127)
__device__ __forceinline__ int8_t code_of(float x, double s) {
    double p = __dmul_rn(static_cast<double>(x), s);
    double t = __dadd_rn(fabs(p), 0.5);
    double r = copysign(floor(t), p);
    r = fmin(fmax(r, -127.0), 127.0);
    return static_cast<int8_t>(static_cast<int>(r));
}

// quantize.py:168-171: scale = 127 / amax, all-zero slice -> scale 1.
__device__ __forceinline__ double scale_of(float amax) {
    return 127.0 / (amax == 0.0f ? 127.0 : static_cast<double>(amax));
}

// Fast exact quantization of one element. p32 = x * fl32(s) differs from the
// exact product P = x*s by < 127 * 2^-23 < 2^-16 (two f32 roundings), and the
// reference's f64 result differs from P by < 2^-45. So whenever p32 is more
// than 2^-14 away from a half-integer, round-to-nearest of p32 equals the
// reference's floor(|p64| + 0.5) with sign (quantize.py:26-29); otherwise
// (~1e-4 of elements) the exact f64 formulation decides.
__device__ __forceinline__ int code_fast(float x, float s32, double s) {
    constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23: t - kMagic = rint(pf)
    const float pf = x * s32;
    const float t = pf + kMagic;
    const float r = t - kMagic;
    if (fabsf(pf - r) < 0.5f - 6.103515625e-05f)
        return static_cast<int>(__float_as_int(t) - 0x4B400000);
    return static_cast<int>(code_of(x, s));
}


inline int grid_rows_chunk(int64_t M, int64_t col_blocks, int64_t target_blocks,
                                  int64_t* rows_per_block) {
    int64_t chunks = (target_blocks + col_blocks - 1) / col_blocks;
    if (chunks < 1) chunks = 1;
    if (chunks > M) chunks = M;
    int64_t rpb = (M + chunks - 1) / chunks;
    if (rpb < 1) rpb = 1;
    *rows_per_block = rpb;
    return static_cast<int>((M + rpb - 1) / rpb);
}


}  // namespace i8mm
