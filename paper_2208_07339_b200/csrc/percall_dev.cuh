// Device pieces of the weight-stationary per-call work (W[O, :] gather, column
// fixup, patched-column codes), shared by their own kernels (weights.cu) and
// the fused prologue kernels (prologue.cu).
#pragma once
#include <cuda_fp16.h>
#include <cstdint>

#include "kernels.cuh"
#include "quant_common.cuh"

namespace i8mm {

constexpr int TOPT = kTopT;

__device__ __forceinline__ bool row_is_out(const uint32_t* mask, int64_t k) {
    return mask != nullptr && ((mask[k >> 5] >> (k & 31)) & 1u);
}

__device__ __forceinline__ float half_bits_to_float(uint32_t b) {
    return __half2float(__ushort_as_half(static_cast<unsigned short>(b)));
}

// block (bx of gx) of row t
__device__ __forceinline__ void gather_rows_block(const __half* __restrict__ w, int64_t ldw, int64_t N,
                                                  const int32_t* __restrict__ idx,
                                                  const int32_t* __restrict__ count, int64_t cap,
                                                  __half* __restrict__ out, int64_t ldo, int vec,
                                                  int64_t t, int64_t bx, int64_t gx) {
    const int64_t n = imin64(static_cast<int64_t>(*count), cap);
    if (t >= n) return;
    const __half* src = w + static_cast<int64_t>(idx[t]) * ldw;
    __half* dst = out + t * ldo;
    if (vec) {
        for (int64_t v = bx * blockDim.x + threadIdx.x; v < (N >> 3); v += gx * blockDim.x)
            reinterpret_cast<uint4*>(dst)[v] = ld_stream_u4(src + (v << 3));
    } else {
        for (int64_t j = bx * blockDim.x + threadIdx.x; j < N; j += gx * blockDim.x) dst[j] = src[j];
    }
}

__device__ __forceinline__ void fixup_column(const __half* __restrict__ w, int64_t K, int64_t N, int64_t ldw,
                                             const uint32_t* __restrict__ mask,
                                             const float* __restrict__ amax_full,
                                             const uint16_t* __restrict__ cand_v,
                                             const int32_t* __restrict__ cand_r,
                                             int32_t* __restrict__ p_count, int32_t* __restrict__ p_idx,
                                             float* __restrict__ p_amax, int32_t* __restrict__ p_src,
                                             int64_t j) {
    if (j >= N) return;
    const int32_t r0 = cand_r[j];
    if (r0 < 0 || !row_is_out(mask, r0)) return;  // cached maximiser is a keep row
    float a_new = -1.0f;
    bool exhausted = true;
    int src = 0;  // 1: the new amax is candidate 1's, so the cached q2 codes apply
#pragma unroll
    for (int i = 1; i < TOPT; ++i) {
        const int32_t r = cand_r[i * N + j];
        if (r < 0) {  // fewer than T rows exist: every row was listed
            exhausted = false;
            a_new = 0.0f;
            src = i == 1;
            break;
        }
        if (!row_is_out(mask, r)) {
            exhausted = false;
            a_new = half_bits_to_float(cand_v[i * N + j]);
            src = i == 1;
            break;
        }
    }
    if (exhausted) {  // all T candidates are outlier rows: rescan the column
        uint32_t m = 0;
        for (int64_t k = 0; k < K; ++k)
            if (!row_is_out(mask, k))
                m = max(m, static_cast<uint32_t>(__half_as_ushort(w[k * ldw + j])) & 0x7FFFu);
        a_new = half_bits_to_float(m);
    }
    if (a_new != amax_full[j]) {
        const int32_t p = atomicAdd(p_count, 1);
        p_idx[p] = static_cast<int32_t>(j);
        p_amax[p] = a_new;
        p_src[p] = src;
        atomicOr(reinterpret_cast<uint32_t*>(p_count) + 4 + (j >> 5), 1u << (j & 31));
    }
}

// codes of patched column p for rows [k0, k0 + 8) (one 8-byte store of WqP)
__device__ __forceinline__ void patch_chunk(const __half* __restrict__ w, int64_t K, int64_t ldw,
                                            const uint32_t* __restrict__ mask,
                                            const int32_t* __restrict__ p_idx,
                                            const float* __restrict__ p_amax,
                                            const int32_t* __restrict__ p_src,
                                            const int8_t* __restrict__ q2, int8_t* __restrict__ wq_p,
                                            int64_t ldq, int32_t p, int64_t k0) {
    const int64_t j = p_idx[p];
    int8_t* dst = wq_p + static_cast<int64_t>(p) * ldq + k0;
    if (p_src[p]) {  // cached second-candidate codes: one contiguous row
        const int8_t* src = q2 + j * ldq + k0;
        if (k0 + 8 <= ldq) *reinterpret_cast<uint2*>(dst) = *reinterpret_cast<const uint2*>(src);
        else for (int e = 0; k0 + e < ldq; ++e) dst[e] = src[e];
        return;
    }
    const double s = scale_of(p_amax[p]);
    const float s32 = static_cast<float>(s);
    __half h[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) h[e] = (k0 + e < K) ? w[(k0 + e) * ldw + j] : __float2half(0.0f);
    uint32_t b[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const int64_t k = k0 + e;
        const int c = (k < K && !row_is_out(mask, k)) ? code_fast(__half2float(h[e]), s32, s) : 0;
        b[e] = static_cast<uint32_t>(c) & 0xFFu;
    }
    if (k0 + 8 <= ldq) {
        *reinterpret_cast<uint2*>(dst) = make_uint2(b[0] | b[1] << 8 | b[2] << 16 | b[3] << 24,
                                                    b[4] | b[5] << 8 | b[6] << 16 | b[7] << 24);
    } else {
        for (int e = 0; k0 + e < ldq; ++e) dst[e] = static_cast<int8_t>(b[e]);
    }
}

}  // namespace i8mm
