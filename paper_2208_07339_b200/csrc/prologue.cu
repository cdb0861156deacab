// Prologue kernels of the LLM.int8() path (CUDA cores, HBM-bound):
//   K1 outlier_scan      -- column mask of |x| >= alpha      (gemm.py:208-210)
//      outlier_compact   -- sorted outlier index list        (gemm.py:211)
//   K2 quantize_rows     -- row absmax over keep columns, f64 round-half-away
//                           codes, outlier gather            (quantize.py:168-179,
//                                                              gemm.py:238,242)
//   K3 quantize_cols_t   -- column absmax over keep rows, codes stored K-major
//                                                             (quantize.py:182-187,
//                                                              gemm.py:243)
//   dequantize_output    -- exact f64 dequantization         (gemm.py:130-147)
//
// Rounding is replicated bit-for-bit: every float64 op is an explicit
// __dmul_rn / __dadd_rn / IEEE division so nvcc cannot contract into FMA.
#include <cuda_fp16.h>
#include <cstdint>
#include <cstdlib>

#include "kernels.cuh"
#include "quant_common.cuh"
#include "sm100_ptx.cuh"
#include "percall_dev.cuh"

namespace i8mm {

// ------------------------------------------------------------------ compact
// One block (any multiple of 32 threads): prefix popcount over the mask words,
// scatter the sorted outlier indices. Mask words are read through L2 (the
// caller may be the scan's last CTA, whose atomics went to L2).
// dgrp (optional, K <= 65536): [count, 32 bitmap words of 64-column groups
// holding an outlier column, then the list of those groups] for row_scale.
__device__ __forceinline__ void compact_block(const uint32_t* __restrict__ col_mask, int64_t K,
                                              int32_t* __restrict__ o_idx, int32_t* __restrict__ o_count,
                                              int32_t* __restrict__ dgrp) {
    __shared__ int32_t warp_sums[32];
    __shared__ uint32_t gbits[32];
    __shared__ int32_t n_dg;
    const int64_t nwords = (K + 31) >> 5;
    const int64_t per = (nwords + blockDim.x - 1) / blockDim.x;
    const int64_t w0 = threadIdx.x * per;
    const int64_t w1 = min(nwords, w0 + per);
    int32_t local = 0;
    for (int64_t w = w0; w < w1; ++w) local += __popc(__ldcg(col_mask + w));
    // block exclusive scan
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int32_t incl = local;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        int32_t t = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += t;
    }
    if (lane == 31) warp_sums[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        const int nw = blockDim.x >> 5;
        int32_t s = lane < nw ? warp_sums[lane] : 0;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            int32_t t = __shfl_up_sync(0xffffffffu, s, d);
            if (lane >= d) s += t;
        }
        if (lane < nw) warp_sums[lane] = s;  // inclusive warp prefix
    }
    __syncthreads();
    int32_t pos = incl - local + (wid > 0 ? warp_sums[wid - 1] : 0);
    for (int64_t w = w0; w < w1; ++w) {
        uint32_t m = __ldcg(col_mask + w);
        while (m) {
            const int b = __ffs(m) - 1;
            m &= m - 1;
            o_idx[pos++] = static_cast<int32_t>((w << 5) + b);
        }
    }
    if (threadIdx.x == blockDim.x - 1) *o_count = pos;
    if (dgrp == nullptr) return;
    if (threadIdx.x < 32) gbits[threadIdx.x] = 0u;
    if (threadIdx.x == 0) n_dg = 0;
    __syncthreads();
    const int64_t ng = (K + 63) >> 6;
    for (int64_t g = threadIdx.x; g < ng; g += blockDim.x) {
        const uint32_t m1 = (2 * g + 1 < nwords) ? __ldcg(col_mask + 2 * g + 1) : 0u;
        if ((__ldcg(col_mask + 2 * g) | m1) != 0u) {
            atomicOr(&gbits[g >> 5], 1u << (g & 31));
            dgrp[33 + atomicAdd(&n_dg, 1)] = static_cast<int32_t>(g);
        }
    }
    __syncthreads();
    if (threadIdx.x < 32) dgrp[1 + threadIdx.x] = static_cast<int32_t>(gbits[threadIdx.x]);
    if (threadIdx.x == 0) dgrp[0] = n_dg;
}

// ------------------------------------------------------------------ K1 scan
// Vector path: each thread owns 8 consecutive columns (one 16-byte load per
// row) for a chunk of rows; 4 adjacent lanes form one 32-bit mask word. The
// threshold test runs on the fp16 bit patterns, two halves per 32-bit SIMD
// compare: for finite fp16 x, |x| >= a  <=>  (bits(x) & 0x7FFF) >= bits(a_h),
// where a_h is the smallest fp16 >= (float)alpha (computed on the host), so
// the test is exactly the reference's float32 comparison (gemm.py:210).
// Per column the kernel keeps max_i (bits(x_ik) & 0x7FFF) with the SIMD
// unsigned max (two halves per 32-bit word); the column is an outlier iff that
// max >= bits(a_h). NaN/Inf patterns are >= 0x7C00, so they surface both as
// outliers and through the nonfinite flag.
template <bool GM>
__global__ void outlier_scan_vec_kernel(const __half* __restrict__ x, int64_t M, int64_t K,
                                        int64_t ldx, uint32_t thr_bits, int64_t rows_per_block,
                                        uint32_t* __restrict__ col_mask,
                                        int32_t* __restrict__ nonfinite,
                                        uint16_t* __restrict__ gmax, int64_t ng,
                                        int32_t* __restrict__ done_ctr, int32_t* __restrict__ o_idx,
                                        int32_t* __restrict__ o_count, int32_t* __restrict__ dgrp) {
    pdl_wait();
    pdl_trigger();
    const int64_t v = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;  // vector col
    const int64_t nvec = K >> 3;
    const int64_t r0 = static_cast<int64_t>(blockIdx.y) * rows_per_block;
    const int64_t r1 = min(M, r0 + rows_per_block);
    const uint32_t lane = threadIdx.x & 31u;
    const bool live = v < nvec;
    uint32_t m[4] = {0, 0, 0, 0};
    // GM: per row, the max |x| bits over each 64-column group (8 adjacent
    // lanes), so the row quantizer needs no second amax pass over X. The
    // row loop is warp-uniform (dead lanes load nothing and feed zeros).
    auto group_max = [&](const uint4& q, int64_t r) {
        if (!GM) return;
        const uint32_t w = __vmaxu2(__vmaxu2(q.x & 0x7FFF7FFFu, q.y & 0x7FFF7FFFu),
                                    __vmaxu2(q.z & 0x7FFF7FFFu, q.w & 0x7FFF7FFFu));
        uint32_t h = max(w & 0xFFFFu, w >> 16);
        h = max(h, __shfl_xor_sync(0xffffffffu, h, 1));
        h = max(h, __shfl_xor_sync(0xffffffffu, h, 2));
        h = max(h, __shfl_xor_sync(0xffffffffu, h, 4));
        if ((lane & 7u) == 0 && live) gmax[r * ng + (v >> 3)] = static_cast<uint16_t>(h);
    };
    if (live || GM) {
        const __half* p = x + r0 * ldx + (live ? (v << 3) : 0);
        int64_t r = r0;
        for (; r + 8 <= r1; r += 8) {
            uint4 q[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) q[u] = live ? ld_stream_u4(p + u * ldx) : make_uint4(0, 0, 0, 0);
            p += 8 * ldx;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                m[0] = __vmaxu2(m[0], q[u].x & 0x7FFF7FFFu);
                m[1] = __vmaxu2(m[1], q[u].y & 0x7FFF7FFFu);
                m[2] = __vmaxu2(m[2], q[u].z & 0x7FFF7FFFu);
                m[3] = __vmaxu2(m[3], q[u].w & 0x7FFF7FFFu);
                group_max(q[u], r + u);
            }
        }
        for (; r < r1; ++r, p += ldx) {
            const uint4 q = live ? ld_stream_u4(p) : make_uint4(0, 0, 0, 0);
            m[0] = __vmaxu2(m[0], q.x & 0x7FFF7FFFu);
            m[1] = __vmaxu2(m[1], q.y & 0x7FFF7FFFu);
            m[2] = __vmaxu2(m[2], q.z & 0x7FFF7FFFu);
            m[3] = __vmaxu2(m[3], q.w & 0x7FFF7FFFu);
            group_max(q, r);
        }
    }
    uint32_t bits = 0, bad = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint32_t lo = m[i] & 0xFFFFu, hi = m[i] >> 16;
        bits |= (lo >= thr_bits ? 1u : 0u) << (2 * i);
        bits |= (hi >= thr_bits ? 1u : 0u) << (2 * i + 1);
        bad |= (lo >= 0x7C00u || hi >= 0x7C00u) ? 1u : 0u;
    }
    uint32_t word = bits << (8u * (lane & 3u));
    word |= __shfl_xor_sync(0xffffffffu, word, 1);
    word |= __shfl_xor_sync(0xffffffffu, word, 2);
    if ((lane & 3u) == 0 && word != 0 && live) atomicOr(col_mask + (v >> 2), word);
    if (nonfinite != nullptr && __any_sync(0xffffffffu, bad != 0) && lane == 0)
        atomicExch(nonfinite, 1);
    if (done_ctr != nullptr) {  // the last CTA to finish compacts the final mask (saves a launch)
        __shared__ int last;
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            last = atomicAdd(done_ctr, 1) == static_cast<int>(gridDim.x * gridDim.y) - 1;
        }
        __syncthreads();
        if (last) {
            __threadfence();
            compact_block(col_mask, K, o_idx, o_count, dgrp);
        }
    }
}

// Scalar path for K % 8 != 0 or unaligned X: one column per thread.
__global__ void outlier_scan_scalar_kernel(const __half* __restrict__ x, int64_t M, int64_t K,
                                           int64_t ldx, float alpha, int64_t rows_per_block,
                                           uint32_t* __restrict__ col_mask,
                                           int32_t* __restrict__ nonfinite) {
    const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t r0 = static_cast<int64_t>(blockIdx.y) * rows_per_block;
    const int64_t r1 = min(M, r0 + rows_per_block);
    bool hit = false, bad = false;
    if (k < K)
        for (int64_t r = r0; r < r1; ++r) {
            __half h = x[r * ldx + k];
            hit |= fabsf(__half2float(h)) >= alpha;
            bad |= h_is_nonfinite(h);
        }
    const uint32_t word = __ballot_sync(0xffffffffu, hit);
    // 32 consecutive threads == 32 consecutive columns == one aligned word
    if ((threadIdx.x & 31u) == 0 && word != 0) atomicOr(col_mask + (k >> 5), word);
    if (nonfinite != nullptr && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31u) == 0)
        atomicExch(nonfinite, 1);
}

__global__ void zero_u32_kernel(uint32_t* p, int64_t n) {
    pdl_wait();
    pdl_trigger();
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        p[i] = 0u;
}

// two ranges in one launch (the mask and the caller's per-call counters)
__global__ void zero2_u32_kernel(uint32_t* p, int64_t n, uint32_t* p2, int64_t n2, uint32_t* one,
                                 uint32_t* p3, int64_t n3, uint32_t* one2) {
    pdl_wait();
    pdl_trigger();
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const int64_t i0 = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i0 == 0) {
        *one = 0u;
        if (one2 != nullptr) *one2 = 0u;
    }
    for (int64_t i = i0; i < n + n2; i += stride) {
        if (i < n) p[i] = 0u;
        else p2[i - n] = 0u;
    }
    // third range (split-K partial sums): 16-byte stores
    uint4* q3 = reinterpret_cast<uint4*>(p3);
    for (int64_t i = i0; i < (n3 >> 2); i += stride) q3[i] = make_uint4(0, 0, 0, 0);
    for (int64_t i = (n3 & ~int64_t(3)) + i0; i < n3; i += stride) p3[i] = 0u;
}

// ------------------------------------------------------------------ compact
// One block: prefix popcount over the mask words, scatter sorted indices.
__global__ void outlier_compact_kernel(const uint32_t* __restrict__ col_mask, int64_t K,
                                       int32_t* __restrict__ o_idx, int32_t* __restrict__ o_count,
                                       int32_t* __restrict__ dgrp) {
    pdl_wait();
    pdl_trigger();
    compact_block(col_mask, K, o_idx, o_count, dgrp);
}

// ------------------------------------------------------------------ K2 rows
__device__ __forceinline__ float block_max(float v, float* red) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, d));
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) red[wid] = v;
    __syncthreads();
    const int nw = blockDim.x >> 5;
    v = lane < nw ? red[lane] : 0.0f;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, d));
    return v;
}

__device__ __forceinline__ uint32_t mask_byte(const uint32_t* mask, int64_t v) {
    // 8 mask bits for vector column v (columns 8v..8v+7)
    return (mask[v >> 2] >> (8u * (v & 3))) & 0xFFu;
}

__device__ __forceinline__ uint32_t keep_word(uint32_t mbyte, int i) {
    // 16-bit lane keep-masks for elements 2i, 2i+1 of a vector (mask bit = outlier)
    return (((mbyte >> (2 * i)) & 1u) ? 0u : 0x0000FFFFu) |
           (((mbyte >> (2 * i + 1)) & 1u) ? 0u : 0xFFFF0000u);
}

__device__ __forceinline__ uint32_t block_max_u32(uint32_t v, uint32_t* red) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, d));
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) red[wid] = v;
    __syncthreads();
    const int nw = blockDim.x >> 5;
    v = lane < nw ? red[lane] : 0u;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, d));
    return v;
}

__device__ __noinline__ int code_of_slow(float x, double s) { return static_cast<int>(code_of(x, s)); }

// Quantize 8 fp16 values (one 16-byte vector) with the row scale: the fp32
// fast path for all 8, one band test for the vector, and the exact f64 rule
// only for elements within 2^-14 of a rounding boundary (see code_fast).
// Rounding uses the 1.5*2^23 magic constant (FADDs on the full-rate FMA pipe,
// not the quarter-rate conversion pipe): t = p + M rounds p to the nearest
// integer and the low byte of bits(t) IS the two's-complement int8 code.
// mbyte bit e set = outlier column -> code 0. Returns the 8 codes packed.
__device__ __forceinline__ uint2 quant8(const uint4& q, uint32_t mbyte, float s32, double s) {
    constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23
    const __half2* h2 = reinterpret_cast<const __half2*>(&q);
    const float2 s2 = make_float2(s32, s32);
    const float2 m2 = make_float2(kMagic, kMagic);
    const float2 nm2 = make_float2(-kMagic, -kMagic);
    float2 pf[4], r[4];
    uint32_t tb[8];
    float dmax = 0.0f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {  // packed f32x2 math (sm_100 FMUL2/FADD2)
        pf[i] = __fmul2_rn(__half22float2(h2[i]), s2);
        const float2 t = __fadd2_rn(pf[i], m2);
        tb[2 * i] = __float_as_uint(t.x);
        tb[2 * i + 1] = __float_as_uint(t.y);
        r[i] = __fadd2_rn(t, nm2);
        const float2 d = __fadd2_rn(pf[i], make_float2(-r[i].x, -r[i].y));
        dmax = fmaxf(dmax, fmaxf(fabsf(d.x), fabsf(d.y)));
    }
    if (dmax >= 0.5f - 6.103515625e-05f) {  // rare: some element near a .5 boundary
        const __half* h = reinterpret_cast<const __half*>(&q);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const float pe = (e & 1) ? pf[e >> 1].y : pf[e >> 1].x;
            const float re = (e & 1) ? r[e >> 1].y : r[e >> 1].x;
            if (fabsf(pe - re) >= 0.5f - 6.103515625e-05f)
                tb[e] = static_cast<uint32_t>(code_of_slow(__half2float(h[e]), s));
        }
    }
    if (mbyte != 0u) {  // vector holds an outlier column
#pragma unroll
        for (int e = 0; e < 8; ++e)
            if ((mbyte >> e) & 1u) tb[e] = 0u;
    }
    const uint32_t a01 = __byte_perm(tb[0], tb[1], 0x0040);
    const uint32_t a23 = __byte_perm(tb[2], tb[3], 0x0040);
    const uint32_t a45 = __byte_perm(tb[4], tb[5], 0x0040);
    const uint32_t a67 = __byte_perm(tb[6], tb[7], 0x0040);
    return make_uint2(__byte_perm(a01, a23, 0x5410), __byte_perm(a45, a67, 0x5410));
}

// One block per row; the row stays in registers (VPT 16-byte vectors/thread).
// amax over keep columns runs on fp16 bit patterns (monotone for |x|) with
// 2-way SIMD max; codes use the fp32 fast path with exact f64 fallback.
template <int VPT>
__global__ void __launch_bounds__(512) quantize_rows_vec_kernel(
    const __half* __restrict__ x, int64_t K, int64_t ldx, const uint32_t* __restrict__ col_mask,
    const int32_t* __restrict__ o_idx, const int32_t* __restrict__ o_count,
    int8_t* __restrict__ xq, int64_t ldq, float* __restrict__ row_amax, __half* __restrict__ xo,
    int64_t o_cap) {
    __shared__ uint32_t red[32];
    const int64_t row = blockIdx.x;
    const int64_t nvec = K >> 3;
    const __half* xr = x + row * ldx;
    uint4 q[VPT];
    uint32_t mb[VPT];
    uint32_t am2 = 0;
#pragma unroll
    for (int j = 0; j < VPT; ++j) {
        const int64_t v = threadIdx.x + static_cast<int64_t>(j) * blockDim.x;
        mb[j] = 0xFFu;
        if (v < nvec) {
            q[j] = ld_stream_u4(xr + (v << 3));
            mb[j] = col_mask ? mask_byte(col_mask, v) : 0u;
        }
    }
#pragma unroll
    for (int j = 0; j < VPT; ++j) {
        const int64_t v = threadIdx.x + static_cast<int64_t>(j) * blockDim.x;
        if (v < nvec) {
            const uint32_t w4[4] = {q[j].x, q[j].y, q[j].z, q[j].w};
            if (mb[j] == 0u) {
#pragma unroll
                for (int i = 0; i < 4; ++i) am2 = __vmaxu2(am2, w4[i] & 0x7FFF7FFFu);
            } else {
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    am2 = __vmaxu2(am2, (w4[i] & 0x7FFF7FFFu) & keep_word(mb[j], i));
            }
        }
    }
    const uint32_t am_bits = block_max_u32(max(am2 & 0xFFFFu, am2 >> 16), red);
    const float amax = __half2float(__ushort_as_half(static_cast<unsigned short>(am_bits)));
    const double s = scale_of(amax);
    const float s32 = static_cast<float>(s);
    int8_t* qr = xq + row * ldq;
#pragma unroll
    for (int j = 0; j < VPT; ++j) {
        const int64_t v = threadIdx.x + static_cast<int64_t>(j) * blockDim.x;
        if (v < nvec) *reinterpret_cast<uint2*>(qr + (v << 3)) = quant8(q[j], mb[j], s32, s);
    }
    if (threadIdx.x == 0) row_amax[row] = amax;
    if (xo != nullptr && o_count != nullptr) {
        const int64_t n = min(static_cast<int64_t>(*o_count), o_cap);
        for (int64_t t = threadIdx.x; t < n; t += blockDim.x) xo[row * o_cap + t] = xr[o_idx[t]];
    }
    // zero the K..ldq padding so the codes buffer is fully defined
    for (int64_t k = K + threadIdx.x; k < ldq; k += blockDim.x) qr[k] = 0;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
                 "l"(gmem)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Rows staged through shared memory with a 2-deep cp.async ring: while a
// block quantizes row r (amax pass + code pass, both from smem), the next
// row's bytes are already in flight, so HBM sees a continuous stream with a
// small register footprint (high occupancy). Dynamic smem: 2 * K * 2 bytes of
// row buffers + the outlier mask words.
__global__ void __launch_bounds__(256) quantize_rows_smem_kernel(
    const __half* __restrict__ x, int64_t M, int64_t K, int64_t ldx,
    const uint32_t* __restrict__ col_mask, const int32_t* __restrict__ o_idx,
    const int32_t* __restrict__ o_count, int8_t* __restrict__ xq, int64_t ldq,
    float* __restrict__ row_amax, __half* __restrict__ xo, int64_t o_cap) {
    extern __shared__ __align__(16) uint8_t qsm[];
    __shared__ uint32_t red[32];
    const int nv = static_cast<int>(K >> 3);
    const int tid = threadIdx.x, bd = blockDim.x;
    uint4* buf0 = reinterpret_cast<uint4*>(qsm);
    uint4* buf1 = buf0 + nv;
    uint32_t* smask = reinterpret_cast<uint32_t*>(buf1 + nv);
    const uint8_t* smask8 = reinterpret_cast<const uint8_t*>(smask);  // one mask byte per vector
    const int nwords = static_cast<int>((K + 31) >> 5);
    for (int i = tid; i < nwords; i += bd) smask[i] = col_mask ? col_mask[i] : 0u;
    const int n_o = (xo != nullptr && o_count != nullptr) ? static_cast<int>(min(static_cast<int64_t>(*o_count), o_cap)) : 0;

    int64_t row = blockIdx.x;
    if (row < M) {
        const uint4* src = reinterpret_cast<const uint4*>(x + row * ldx);
        for (int v = tid; v < nv; v += bd) cp_async16(buf0 + v, src + v);
    }
    cp_async_commit();
    int stage = 0;
    for (; row < M; row += gridDim.x) {
        uint4* cur = stage ? buf1 : buf0;
        uint4* nxt = stage ? buf0 : buf1;
        const int64_t nrow = row + gridDim.x;
        if (nrow < M) {
            const uint4* src = reinterpret_cast<const uint4*>(x + nrow * ldx);
            for (int v = tid; v < nv; v += bd) cp_async16(nxt + v, src + v);
        }
        cp_async_commit();
        cp_async_wait<1>();  // this row's group has landed
        __syncthreads();
        // pass 1: amax over keep columns on fp16 bit patterns
        uint32_t am2 = 0;
        for (int v = tid; v < nv; v += bd) {
            const uint4 q = cur[v];
            const uint32_t mb = smask8[v];
            if (mb == 0u) {
                am2 = __vmaxu2(am2, q.x & 0x7FFF7FFFu);
                am2 = __vmaxu2(am2, q.y & 0x7FFF7FFFu);
                am2 = __vmaxu2(am2, q.z & 0x7FFF7FFFu);
                am2 = __vmaxu2(am2, q.w & 0x7FFF7FFFu);
            } else {
                const uint32_t w4[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
                for (int i = 0; i < 4; ++i) am2 = __vmaxu2(am2, (w4[i] & 0x7FFF7FFFu) & keep_word(mb, i));
            }
        }
        const uint32_t am_bits = block_max_u32(max(am2 & 0xFFFFu, am2 >> 16), red);
        const float amax = __half2float(__ushort_as_half(static_cast<unsigned short>(am_bits)));
        const double s = scale_of(amax);
        const float s32 = static_cast<float>(s);
        uint2* qr = reinterpret_cast<uint2*>(xq + row * ldq);
        // pass 2: codes
#pragma unroll 2
        for (int v = tid; v < nv; v += bd) qr[v] = quant8(cur[v], smask8[v], s32, s);
        if (tid == 0) row_amax[row] = amax;
        const __half* crow = reinterpret_cast<const __half*>(cur);
        for (int t = tid; t < n_o; t += bd) xo[row * o_cap + t] = crow[o_idx[t]];
        int8_t* qb = xq + row * ldq;
        for (int64_t k = K + tid; k < ldq; k += bd) qb[k] = 0;
        __syncthreads();  // everyone is done with `cur` (and `red`) before it is refilled
        stage ^= 1;
    }
    cp_async_wait<0>();
}

// ---------------------------------------------------------- K2 split form
// With the scan's per-row 64-column group maxima (gmax), the row quantizer
// splits into a tiny scale pass and a pure streaming code pass:
//   row_scale    -- amax over keep columns = max of gmax over groups without an
//                   outlier column, plus a direct re-read of the (few) groups that
//                   hold one; writes row_amax, the f64 scale and x[:, O]
//   quantize_bulk -- codes from a cp.async.bulk-fed shared-memory ring
//                   (one 16-byte vector column per consumer thread).
// Same bits as quantize_rows_* (amax on fp16 bit patterns, quant8 codes).
// One warp per row, one memory round trip: the loads of the row's group
// maxima, of the vectors of the dirty groups and of x[row, O] are all issued
// before any is consumed. Dirty groups (64-column groups holding an outlier
// column) come from outlier_compact's dgrp list; K <= 65536 (ng <= 1024).
constexpr int RS_GM = 8;  // group maxima per lane per pass (256 groups = 16384 columns)
struct RowScaleArgs {
    const __half* x;
    int64_t M, K, ldx;
    const uint32_t* col_mask;
    const int32_t* o_idx;
    const int32_t* o_count;
    const uint16_t* gmax;
    int64_t ng;
    const int32_t* dgrp;
    float* row_amax;
    double* row_s;
    __half* xo;
    int64_t o_cap;
};

// block bid of nblk row-scale blocks
__device__ __forceinline__ void row_scale_block(const RowScaleArgs& a, int64_t bid, int64_t nblk) {
    const __half* __restrict__ x = a.x;
    const int64_t M = a.M, K = a.K, ldx = a.ldx, ng = a.ng, o_cap = a.o_cap;
    const uint32_t* __restrict__ col_mask = a.col_mask;
    const int32_t* __restrict__ o_idx = a.o_idx;
    const int32_t* __restrict__ o_count = a.o_count;
    const uint16_t* __restrict__ gmax = a.gmax;
    const int32_t* __restrict__ dgrp = a.dgrp;
    float* __restrict__ row_amax = a.row_amax;
    double* __restrict__ row_s = a.row_s;
    __half* __restrict__ xo = a.xo;
    __shared__ uint32_t sgb[32];
    __shared__ int32_t sdg[1024];
    __shared__ int32_t so[64];
    const int nd = __ldg(dgrp);
    const int n_o = xo != nullptr ? static_cast<int>(min(static_cast<int64_t>(__ldg(o_count)), min(o_cap, static_cast<int64_t>(64)))) : 0;
    if (threadIdx.x < 32) sgb[threadIdx.x] = static_cast<uint32_t>(__ldg(dgrp + 1 + threadIdx.x));
    for (int k = threadIdx.x; k < nd; k += blockDim.x) sdg[k] = __ldg(dgrp + 33 + k);
    for (int k = threadIdx.x; k < n_o; k += blockDim.x) so[k] = __ldg(o_idx + k);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t nvec = K >> 3;
    const int nd8 = nd * 8;
    const int64_t nwarps = blockDim.x >> 5;
    const bool gvec = (ng & 7) == 0 && (reinterpret_cast<uintptr_t>(gmax) & 15u) == 0;
    for (int64_t row = bid * nwarps + (threadIdx.x >> 5); row < M; row += nblk * nwarps) {
        const __half* xr = x + row * ldx;
        const uint16_t* gr = gmax + row * ng;
        // issue: first dirty pair chunk + x[row, O]
        uint4 dq[2];
        uint32_t dmb[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int pidx = lane + 32 * j;
            const int64_t v = pidx < nd8 ? (static_cast<int64_t>(sdg[pidx >> 3]) << 3) + (pidx & 7) : nvec;
            dq[j] = make_uint4(0, 0, 0, 0);
            dmb[j] = 0xFFu;
            if (v < nvec) {
                dq[j] = *reinterpret_cast<const uint4*>(xr + (v << 3));
                dmb[j] = mask_byte(col_mask, v);
            }
        }
        __half ov[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int t = lane + 32 * j;
            if (t < n_o) ov[j] = xr[so[t]];
        }
        uint32_t am = 0;
        if (gvec) {  // 8 group maxima per lane per 16-byte load, dirty groups masked per pair
            for (int g = lane * 8; g < ng; g += 256) {
                const uint4 q = *reinterpret_cast<const uint4*>(gr + g);
                const uint32_t db = (sgb[g >> 5] >> (g & 31)) & 0xFFu;
                const uint32_t w4[4] = {q.x, q.y, q.z, q.w};
                uint32_t m2 = 0;
#pragma unroll
                for (int i = 0; i < 4; ++i) m2 = __vmaxu2(m2, w4[i] & keep_word(db, i));
                am = max(am, max(m2 & 0xFFFFu, m2 >> 16));
            }
        } else
        for (int64_t g0 = 0; g0 < ng; g0 += 32 * RS_GM) {
            uint32_t gm[RS_GM];
#pragma unroll
            for (int j = 0; j < RS_GM; ++j) {
                const int64_t g = g0 + lane + 32 * j;
                gm[j] = g < ng ? static_cast<uint32_t>(gr[g]) : 0u;
            }
#pragma unroll
            for (int j = 0; j < RS_GM; ++j) {
                const int64_t g = g0 + lane + 32 * j;
                if (g < ng && !((sgb[g >> 5] >> (g & 31)) & 1u)) am = max(am, gm[j]);
            }
        }
        auto keep_max = [&](const uint4& q, uint32_t mb) {
            const uint32_t w4[4] = {q.x, q.y, q.z, q.w};
            uint32_t am2 = 0;
#pragma unroll
            for (int i = 0; i < 4; ++i) am2 = __vmaxu2(am2, (w4[i] & 0x7FFF7FFFu) & keep_word(mb, i));
            am = max(am, max(am2 & 0xFFFFu, am2 >> 16));
        };
        keep_max(dq[0], dmb[0]);
        keep_max(dq[1], dmb[1]);
        for (int pidx = lane + 64; pidx < nd8; pidx += 32) {  // > 8 dirty groups
            const int64_t v = (static_cast<int64_t>(sdg[pidx >> 3]) << 3) + (pidx & 7);
            if (v < nvec) keep_max(*reinterpret_cast<const uint4*>(xr + (v << 3)), mask_byte(col_mask, v));
        }
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int t = lane + 32 * j;
            if (t < n_o) xo[row * o_cap + t] = ov[j];
        }
        for (int t = lane + 64; t < min(static_cast<int64_t>(__ldg(o_count)), o_cap) && xo != nullptr; t += 32)
            xo[row * o_cap + t] = xr[o_idx[t]];
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) am = max(am, __shfl_xor_sync(0xffffffffu, am, d));
        if (lane == 0) {
            const float amax = __half2float(__ushort_as_half(static_cast<unsigned short>(am)));
            row_amax[row] = amax;
            row_s[row] = scale_of(amax);
        }
    }
}

__global__ void __launch_bounds__(256) row_scale_kernel(const RowScaleArgs a) {
    pdl_wait();
    pdl_trigger();
    row_scale_block(a, blockIdx.x, gridDim.x);
}

// Row scales + the weight-stationary W[O, :] gather and column fixup in one
// grid (all three only need the compacted outlier set): blocks [0, rs_blocks)
// are row-scale blocks, then o_cap * gx gather blocks, then fixup blocks.
__global__ void __launch_bounds__(256) row_scale_fix_kernel(const RowScaleArgs a, int64_t rs_blocks,
                                                            const PerCallFix f, int vec, int64_t gx) {
    pdl_wait();
    pdl_trigger();
    const int64_t b = blockIdx.x;
    if (b < rs_blocks) {
        row_scale_block(a, b, rs_blocks);
        return;
    }
    const int64_t g = b - rs_blocks, ngath = a.o_cap * gx;
    if (g < ngath) {
        gather_rows_block(f.w, f.ldw, f.N, a.o_idx, a.o_count, a.o_cap, f.wo, f.ldwo, vec, g / gx, g % gx, gx);
        return;
    }
    fixup_column(f.w, f.K, f.N, f.ldw, a.col_mask, f.amax_full, f.cand_v, f.cand_r, f.p_count, f.p_idx,
                 f.p_amax, f.p_src, (g - ngath) * blockDim.x + threadIdx.x);
}

// Bulk-copy fed code pass: persistent CTAs (2 per SM), a producer lane streams
// 8-row x 2048-column tiles of X into a QS_STAGES-deep shared-memory ring with
// cp.async.bulk (the copy engine keeps up to QS_STAGES x 32 KB per CTA in
// flight, independent of the register file); 8 consumer warps quantize one
// 16-byte vector column per thread and store the codes (8 bytes, coalesced).
constexpr int QS_ROWS = 8, QS_VECS = 256, QS_STAGES = 3;
constexpr int QS_STAGE_BYTES = QS_ROWS * QS_VECS * 16;

__global__ void __launch_bounds__(288) quantize_bulk_kernel(
    const __half* __restrict__ x, int64_t M, int64_t K, int64_t ldx,
    const uint32_t* __restrict__ col_mask, const double* __restrict__ row_s,
    int8_t* __restrict__ xq, int64_t ldq, const PerCallFix f, int rev) {
    extern __shared__ __align__(128) uint8_t qb_sm[];
    __shared__ __align__(8) uint64_t full[QS_STAGES], empty[QS_STAGES];
    const int64_t nvec = K >> 3;
    const int64_t ncb = (nvec + QS_VECS - 1) / QS_VECS;
    const int64_t ntiles = ((M + QS_ROWS - 1) / QS_ROWS) * ncb;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < QS_STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 8);
        }
        fence_mbarrier_init();
    }
    __syncthreads();
    pdl_wait();
    pdl_trigger();
    if (warp == 8) {  // producer
        if (lane == 0) {
            int i = 0;
            for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
                const int s = i % QS_STAGES;
                if (i >= QS_STAGES) mbar_wait(&empty[s], ((i / QS_STAGES) - 1) & 1);
                const int64_t tt = rev ? ntiles - 1 - t : t;
                const int64_t r0 = (tt / ncb) * QS_ROWS, v0 = (tt % ncb) * QS_VECS;
                const int rows = static_cast<int>(min(static_cast<int64_t>(QS_ROWS), M - r0));
                const uint32_t seg = static_cast<uint32_t>(min(static_cast<int64_t>(QS_VECS), nvec - v0)) * 16u;
                mbar_arrive_expect_tx(&full[s], seg * rows);
                uint8_t* dst = qb_sm + s * QS_STAGE_BYTES;
                for (int u = 0; u < rows; ++u)
                    bulk_load_1d(dst + u * QS_VECS * 16, x + (r0 + u) * ldx + (v0 << 3), seg, &full[s]);
            }
        }
        return;
    }
    if (f.p_count != nullptr) {  // weight-stationary: patched columns' codes first (the ring fills meanwhile)
        const int32_t np = *f.p_count;
        for (int32_t p = blockIdx.x; p < np; p += gridDim.x)
            for (int64_t k0 = threadIdx.x * 8; k0 < ldq; k0 += 256 * 8)
                patch_chunk(f.w, f.K, f.ldw, col_mask, f.p_idx, f.p_amax, f.p_src, f.q2, f.wq_p, ldq, p, k0);
    }
    int i = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
        const int s = i % QS_STAGES;
        const int64_t tt = rev ? ntiles - 1 - t : t;
        const int64_t r0 = (tt / ncb) * QS_ROWS, v = (tt % ncb) * QS_VECS + threadIdx.x;
        const int rows = static_cast<int>(min(static_cast<int64_t>(QS_ROWS), M - r0));
        double sc[QS_ROWS];
        if (rows == QS_ROWS) {
#pragma unroll
            for (int u = 0; u < QS_ROWS; ++u) sc[u] = __ldg(row_s + r0 + u);
        }
        const uint32_t mb = v < nvec ? mask_byte(col_mask, v) : 0u;
        mbar_wait(&full[s], (i / QS_STAGES) & 1);
        if (v < nvec) {
            const uint4* src = reinterpret_cast<const uint4*>(qb_sm + s * QS_STAGE_BYTES) + threadIdx.x;
            int8_t* o = xq + r0 * ldq + (v << 3);
            if (rows == QS_ROWS) {
                uint4 q[QS_ROWS];
#pragma unroll
                for (int u = 0; u < QS_ROWS; ++u) q[u] = src[u * QS_VECS];
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);
#pragma unroll
                for (int u = 0; u < QS_ROWS; ++u)
                    *reinterpret_cast<uint2*>(o + u * ldq) = quant8(q[u], mb, static_cast<float>(sc[u]), sc[u]);
            } else {
                for (int u = 0; u < rows; ++u) {
                    const double su = __ldg(row_s + r0 + u);
                    *reinterpret_cast<uint2*>(o + u * ldq) =
                        quant8(src[u * QS_VECS], mb, static_cast<float>(su), su);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);
            }
            if (v == nvec - 1 && ldq > K)
                for (int u = 0; u < rows; ++u)
                    for (int64_t k = K; k < ldq; ++k) xq[(r0 + u) * ldq + k] = 0;
        } else {
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
    }
}

// Generic path (any K / alignment): two passes over the row from global.
__global__ void quantize_rows_scalar_kernel(const __half* __restrict__ x, int64_t K, int64_t ldx,
                                            const uint32_t* __restrict__ col_mask,
                                            const int32_t* __restrict__ o_idx,
                                            const int32_t* __restrict__ o_count,
                                            int8_t* __restrict__ xq, int64_t ldq,
                                            float* __restrict__ row_amax, __half* __restrict__ xo,
                                            int64_t o_cap) {
    __shared__ float red[32];
    const int64_t row = blockIdx.x;
    const __half* xr = x + row * ldx;
    float amax = 0.0f;
    for (int64_t k = threadIdx.x; k < K; k += blockDim.x) {
        const bool out = col_mask && ((col_mask[k >> 5] >> (k & 31)) & 1u);
        if (!out) amax = fmaxf(amax, fabsf(__half2float(xr[k])));
    }
    amax = block_max(amax, red);
    const double s = scale_of(amax);
    int8_t* qr = xq + row * ldq;
    for (int64_t k = threadIdx.x; k < ldq; k += blockDim.x) {
        int8_t c = 0;
        if (k < K) {
            const bool out = col_mask && ((col_mask[k >> 5] >> (k & 31)) & 1u);
            if (!out) c = code_of(__half2float(xr[k]), s);
        }
        qr[k] = c;
    }
    if (threadIdx.x == 0) row_amax[row] = amax;
    if (xo != nullptr && o_count != nullptr) {
        const int64_t n = min(static_cast<int64_t>(*o_count), o_cap);
        for (int64_t t = threadIdx.x; t < n; t += blockDim.x) xo[row * o_cap + t] = xr[o_idx[t]];
    }
}

// ------------------------------------------------------------------ dequant
__global__ void dequantize_output_kernel(const int32_t* __restrict__ c, int64_t M, int64_t N,
                                         int64_t ldc, const double* __restrict__ sx,
                                         const double* __restrict__ sw, float* __restrict__ out,
                                         int64_t ldo) {
    const int64_t total = M * N;
    for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = t / N, j = t - (t / N) * N;
        const double d = __dmul_rn(sx[i], sw[j]);
        out[i * ldo + j] = __double2float_rn(__ddiv_rn(static_cast<double>(c[i * ldc + j]), d));
    }
}

__global__ void transpose_i8_kernel(const int8_t* __restrict__ src, int64_t rows, int64_t cols,
                                    int64_t lds, int8_t* __restrict__ dst, int64_t ldd) {
    __shared__ int8_t t[32][33];
    const int64_t r0 = static_cast<int64_t>(blockIdx.y) * 32, c0 = static_cast<int64_t>(blockIdx.x) * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int64_t r = r0 + i, c = c0 + threadIdx.x;
        t[i][threadIdx.x] = (r < rows && c < cols) ? src[r * lds + c] : int8_t(0);
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int64_t c = c0 + i, r = r0 + threadIdx.x;  // dst row = src col
        if (c < cols && r < rows) dst[c * ldd + r] = t[threadIdx.x][i];
    }
}

// ------------------------------------------------------------------ launchers
// smallest fp16 bit pattern h (as |x| bits) with float(h) >= alpha (alpha > 0)
uint32_t alpha_threshold_bits(float alpha) {
    if (!(alpha <= 65504.0f)) return 0x7C00u;  // only +-inf would qualify
    __half h = __float2half_rn(alpha);
    uint32_t b = __half_as_ushort(h) & 0x7FFFu;
    if (__half2float(h) < alpha) b += 1u;
    return b;
}

cudaError_t launch_outlier_scan(const __half* x, int64_t M, int64_t K, int64_t ldx, float alpha,
                                uint32_t* col_mask, int32_t* nonfinite, cudaStream_t st) {
    const int64_t nwords = (K + 31) >> 5;
    zero_u32_kernel<<<static_cast<unsigned>(imin64((nwords + 255) / 256, 1024)), 256, 0, st>>>(
        col_mask, nwords);
    count_launch();
    if (M == 0) return cudaGetLastError();
    const int sms = num_sms();
    const bool vec = (K % 8 == 0) && (ldx % 8 == 0) && ((reinterpret_cast<uintptr_t>(x) & 15u) == 0);
    int64_t rpb;
    if (vec) {
        const int64_t nvec = K >> 3;
        const int64_t cb = (nvec + 255) / 256;
        const int rb = grid_rows_chunk(M, cb, static_cast<int64_t>(sms) * 8, &rpb);
        outlier_scan_vec_kernel<false><<<dim3(static_cast<unsigned>(cb), rb), 256, 0, st>>>(
            x, M, K, ldx, alpha_threshold_bits(alpha), rpb, col_mask, nonfinite, nullptr, 0, nullptr,
            nullptr, nullptr, nullptr);
    } else {
        const int64_t cb = (K + 255) / 256;
        const int rb = grid_rows_chunk(M, cb, static_cast<int64_t>(sms) * 8, &rpb);
        outlier_scan_scalar_kernel<<<dim3(static_cast<unsigned>(cb), rb), 256, 0, st>>>(
            x, M, K, ldx, alpha, rpb, col_mask, nonfinite);
    }
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_outlier_compact(const uint32_t* col_mask, int64_t K, int32_t* o_idx,
                                   int32_t* o_count, cudaStream_t st) {
    outlier_compact_kernel<<<1, 1024, 0, st>>>(col_mask, K, o_idx, o_count, nullptr);
    count_launch();
    return cudaGetLastError();
}

template <int VPT>
static void launch_qrows(int threads, const __half* x, int64_t M, int64_t K, int64_t ldx,
                         const uint32_t* mask, const int32_t* o_idx, const int32_t* o_count,
                         int8_t* xq, int64_t ldq, float* amax, __half* xo, int64_t o_cap,
                         cudaStream_t st) {
    quantize_rows_vec_kernel<VPT><<<static_cast<unsigned>(M), threads, 0, st>>>(
        x, K, ldx, mask, o_idx, o_count, xq, ldq, amax, xo, o_cap);
}

cudaError_t launch_quantize_rows(const __half* x, int64_t M, int64_t K, int64_t ldx,
                                 const uint32_t* mask, const int32_t* o_idx,
                                 const int32_t* o_count, int8_t* xq, int64_t ldq, float* amax,
                                 __half* xo, int64_t o_cap, cudaStream_t st) {
    if (M == 0) return cudaSuccess;
    // register-resident rows up to K = 16 vectors x 8 x 512 threads = 65536
    const size_t smem_bytes = static_cast<size_t>(K) * 4 + static_cast<size_t>((K + 31) / 32) * 4;
    const bool aligned = (K % 8 == 0) && (ldx % 8 == 0) && (ldq % 8 == 0) &&
                         ((reinterpret_cast<uintptr_t>(x) & 15u) == 0) &&
                         ((reinterpret_cast<uintptr_t>(xq) & 7u) == 0);
    if (aligned && smem_bytes <= 200 * 1024) {
        static size_t configured = 0;
        if (smem_bytes > 48 * 1024 && smem_bytes > configured) {
            cudaFuncSetAttribute(quantize_rows_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 200 * 1024);
            configured = 200 * 1024;
        }
        const int per_sm = static_cast<int>(imin64(8, (220 * 1024) / static_cast<int64_t>(smem_bytes + 1024)));
        const int64_t grid = imin64(M, static_cast<int64_t>(num_sms()) * (per_sm > 0 ? per_sm : 1));
        quantize_rows_smem_kernel<<<static_cast<unsigned>(grid), 256, smem_bytes, st>>>(
            x, M, K, ldx, mask, o_idx, o_count, xq, ldq, amax, xo, o_cap);
        count_launch();
        return cudaGetLastError();
    }
    const bool vec = (K % 8 == 0) && (K <= 65536) && (ldx % 8 == 0) && (ldq % 8 == 0) &&
                     ((reinterpret_cast<uintptr_t>(x) & 15u) == 0) &&
                     ((reinterpret_cast<uintptr_t>(xq) & 7u) == 0);
    if (!vec) {
        quantize_rows_scalar_kernel<<<static_cast<unsigned>(M), 256, 0, st>>>(
            x, K, ldx, mask, o_idx, o_count, xq, ldq, amax, xo, o_cap);
        count_launch();
        return cudaGetLastError();
    }
    // ~8 vectors (64 halves) per thread keeps 8 16-byte loads in flight; the
    // block grows with K up to 512 threads, then VPT grows (<= 16).
    const int64_t nvec = K >> 3;
    int64_t threads = ((nvec + 8 * 32 - 1) / (8 * 32)) * 32;
    if (threads < 64) threads = 64;
    if (threads > 512) threads = 512;
    int vpt = 1;
    while (vpt < 16 && static_cast<int64_t>(vpt) * threads < nvec) vpt <<= 1;
    if (static_cast<int64_t>(vpt) * threads < nvec) return cudaErrorInvalidValue;
    const int t = static_cast<int>(threads);
    switch (vpt) {
        case 1: launch_qrows<1>(t, x, M, K, ldx, mask, o_idx, o_count, xq, ldq, amax, xo, o_cap, st); break;
        case 2: launch_qrows<2>(t, x, M, K, ldx, mask, o_idx, o_count, xq, ldq, amax, xo, o_cap, st); break;
        case 4: launch_qrows<4>(t, x, M, K, ldx, mask, o_idx, o_count, xq, ldq, amax, xo, o_cap, st); break;
        case 8: launch_qrows<8>(t, x, M, K, ldx, mask, o_idx, o_count, xq, ldq, amax, xo, o_cap, st); break;
        default: launch_qrows<16>(t, x, M, K, ldx, mask, o_idx, o_count, xq, ldq, amax, xo, o_cap, st); break;
    }
    count_launch();
    return cudaGetLastError();
}

// ------------------------------------------------------- K1+K2 one-read form
// One HBM read of X (SURVEY 8(d) "1-read"): persistent CTAs stream blocks of
// RB whole rows into a shared-memory ring (cp.async.bulk, one copy per row);
// per block the consumer warps
//   1. scan the block's columns (|x| >= alpha on fp16 bits) and publish new
//      outlier columns to the running global mask F (atomicOr only for bits
//      not yet set),
//   2. snapshot F (S_b: it holds every column flagged so far, including the
//      block's own) and store S_b with its popcount,
//   3. quantize the rows against S_b: amax over keep columns, codes (quant8),
//      all from shared memory.
// S_b is a subset of the final mask F, so rows of a block quantized before some
// column was flagged elsewhere are corrected exactly by rp1_finalize_kernel:
// codes at the late columns are zeroed, and a row whose amax may have sat in a
// late column is re-quantized from X. When outlier features show up in most
// row blocks (they do in LLM activations and in planted_pair) S_b == F for
// nearly every block and the finalize pass only gathers x[:, O].
constexpr int RP1_THREADS = 544;  // 16 consumer warps + 1 producer warp
constexpr int RP1_CONSUMERS = 512;
constexpr int RP1_MAX_STAGES = 4;
constexpr int RP1_BLOCK_VECS = 4096;       // 16-byte vectors per block (64 KB)
constexpr int RP1_VPT = RP1_BLOCK_VECS / RP1_CONSUMERS;  // vectors per consumer thread (registers)
constexpr int RP1_SMEM_RING = 200 * 1024;  // ring bytes (row blocks + their mask views)

struct Rp1Geom {
    int rb;          // rows per block (power of two, <= 16)
    int tpr;         // consumer threads per row = RP1_CONSUMERS / rb
    int view_bytes;  // mask view per stage (nwords rounded up to 16 bytes)
    int stage_bytes; // rb rows + view
    int stages;
    int64_t nblk;
};

__host__ __device__ inline Rp1Geom rp1_geom(int64_t M, int64_t K) {
    Rp1Geom g{};
    const int64_t nv = K >> 3;
    int64_t p2 = 1;
    while (p2 < nv) p2 <<= 1;
    int64_t rb = RP1_BLOCK_VECS / p2;
    if (rb < 1) rb = 1;
    if (rb > 16) rb = 16;
    g.rb = static_cast<int>(rb);
    g.tpr = RP1_CONSUMERS / g.rb;
    const int64_t nwords = (K + 31) >> 5;
    g.view_bytes = static_cast<int>(((nwords * 4 + 15) / 16) * 16);
    const int64_t row_part = ((rb * K * 2 + 127) / 128) * 128;
    g.stage_bytes = static_cast<int>(row_part + ((g.view_bytes + 127) / 128) * 128);
    int64_t st = RP1_SMEM_RING / g.stage_bytes;
    if (st > RP1_MAX_STAGES) st = RP1_MAX_STAGES;
    g.stages = static_cast<int>(st);
    g.nblk = (M + rb - 1) / rb;
    return g;
}

// Per block: the producer lands RB rows (one bulk copy each) plus a copy of
// the running mask F (the block's snapshot S_b, taken when the copy is
// issued). Consumers (256 / RB threads per row):
//   pass A: keep amax of the row against S_b; elements >= alpha in a column
//           outside S_b publish that column to F (atomicOr; rare once F holds
//           the layer's outlier features) -- such rows are then corrected by
//           rp1_finalize_kernel, like every row of a block whose S_b missed a
//           column of the final F;
//   pass B: codes (quant8) from shared memory, 8-byte stores.
// S_b and its popcount are stored for the finalize pass.
template <int RB>
__global__ void __launch_bounds__(RP1_THREADS, 1) rp1_stream_kernel(
    const __half* __restrict__ x, int64_t M, int64_t K, int64_t ldx, uint32_t thr_bits,
    uint32_t* __restrict__ fmask, uint32_t* __restrict__ snap, int32_t* __restrict__ snap_cnt,
    int8_t* __restrict__ xq, int64_t ldq, float* __restrict__ row_amax) {
    extern __shared__ __align__(128) uint8_t rp_sm[];
    __shared__ __align__(8) uint64_t full[RP1_MAX_STAGES], empty[RP1_MAX_STAGES];
    __shared__ uint32_t ram[3][16];  // block i uses slot i % 3 (reset two blocks ahead)
    static_assert(RP1_CONSUMERS / 32 <= 16 * 32, "");
    __shared__ int32_t scnt[3];
    constexpr int TPR = RP1_CONSUMERS / RB;  // threads per row (>= 32: whole warps)
    const Rp1Geom g = rp1_geom(M, K);
    const int nwords = static_cast<int>((K + 31) >> 5);
    const int nv = static_cast<int>(K >> 3);
    const int row_part = g.stage_bytes - ((g.view_bytes + 127) / 128) * 128;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < g.stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], RP1_CONSUMERS / 32);
        }
        fence_mbarrier_init();
    }
    if (threadIdx.x < 48) ram[threadIdx.x >> 4][threadIdx.x & 15] = 0u;
    if (threadIdx.x < 3) scnt[threadIdx.x] = 0;
    __syncthreads();
    pdl_wait();
    pdl_trigger();
    if (warp == RP1_CONSUMERS / 32) {  // producer
        if (lane == 0) {
            int i = 0;
            for (int64_t b = blockIdx.x; b < g.nblk; b += gridDim.x, ++i) {
                const int s = i % g.stages;
                if (i >= g.stages)  // back off between polls: the spin would steal issue slots
                    while (!mbar_try_wait(&empty[s], ((i / g.stages) - 1) & 1)) __nanosleep(64);
                const int64_t r0 = b * RB;
                const int rows = static_cast<int>(min(static_cast<int64_t>(RB), M - r0));
                mbar_arrive_expect_tx(&full[s], static_cast<uint32_t>(rows * K * 2 + g.view_bytes));
                uint8_t* dst = rp_sm + static_cast<size_t>(s) * g.stage_bytes;
                bulk_load_1d(dst + row_part, fmask, static_cast<uint32_t>(g.view_bytes), &full[s]);
                for (int u = 0; u < rows; ++u)
                    bulk_load_1d(dst + u * K * 2, x + (r0 + u) * ldx, static_cast<uint32_t>(K * 2), &full[s]);
            }
        }
        return;
    }
    const int tid = threadIdx.x;
    const int rl = tid / TPR, tr = tid % TPR;  // row within the block, thread within the row
    const uint32_t thr2 = thr_bits | (thr_bits << 16);
    int i = 0;
    for (int64_t b = blockIdx.x; b < g.nblk; b += gridDim.x, ++i) {
        // slot (i+1)%3 was last read by block i-2, before block i-1's barrier
        const int s = i % g.stages, par = i % 3, nxt = (i + 1) % 3;
        const int64_t r0 = b * RB;
        const int rows = static_cast<int>(min(static_cast<int64_t>(RB), M - r0));
        if (tid < 16) ram[nxt][tid] = 0u;
        if (tid == 0) scnt[nxt] = 0;
        mbar_wait(&full[s], (i / g.stages) & 1);
        const uint8_t* base = rp_sm + static_cast<size_t>(s) * g.stage_bytes;
        const uint32_t* view = reinterpret_cast<const uint32_t*>(base + row_part);
        const uint4* rowv = reinterpret_cast<const uint4*>(base) + static_cast<int64_t>(rl) * nv;
        const bool live = rl < rows;
        // snapshot S_b -> global (for the finalize pass)
        int32_t pc = 0;
        for (int w = tid; w < nwords; w += RP1_CONSUMERS) {
            const uint32_t f = view[w];
            snap[b * nwords + w] = f;
            pc += __popc(f);
        }
        if (pc) atomicAdd(&scnt[par], pc);
        // the thread's (at most 8) vectors of its row and their mask bytes -> registers
        uint4 q[RP1_VPT];
        uint32_t mbv[RP1_VPT];
#pragma unroll
        for (int j = 0; j < RP1_VPT; ++j) {
            const int v = tr + j * TPR;
            const bool ok = live && v < nv;
            q[j] = ok ? rowv[v] : make_uint4(0, 0, 0, 0);
            mbv[j] = ok ? (view[v >> 2] >> (8 * (v & 3))) & 0xFFu : 0xFFu;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);  // stage consumed: the producer may refill it
        // keep amax + detection of columns outside S_b
        uint32_t am2 = 0;
#pragma unroll
        for (int j = 0; j < RP1_VPT; ++j) {
            const uint32_t w4[4] = {q[j].x & 0x7FFF7FFFu, q[j].y & 0x7FFF7FFFu, q[j].z & 0x7FFF7FFFu,
                                    q[j].w & 0x7FFF7FFFu};
            const uint32_t m = __vmaxu2(__vmaxu2(w4[0], w4[1]), __vmaxu2(w4[2], w4[3]));
            const uint32_t mb = mbv[j];
            uint32_t mk = m;
            if (mb != 0u)
                mk = __vmaxu2(__vmaxu2(w4[0] & keep_word(mb, 0), w4[1] & keep_word(mb, 1)),
                              __vmaxu2(w4[2] & keep_word(mb, 2), w4[3] & keep_word(mb, 3)));
            am2 = __vmaxu2(am2, mk);
            if (max(m & 0xFFFFu, m >> 16) >= thr_bits) {  // an element >= alpha
                uint32_t hit = 0;
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const uint32_t c = __vcmpgeu2(w4[e], thr2);
                    hit |= ((c & 1u) << (2 * e)) | (((c >> 16) & 1u) << (2 * e + 1));
                }
                hit &= ~mb;
                const int v = tr + j * TPR;
                if (hit) atomicOr(fmask + (v >> 2), hit << (8 * (v & 3)));
            }
        }
        uint32_t am = max(am2 & 0xFFFFu, am2 >> 16);
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) am = max(am, __shfl_xor_sync(0xffffffffu, am, d));
        if (live && lane == 0 && am) atomicMax(&ram[par][rl], am);
        named_bar_sync(1, RP1_CONSUMERS);
        if (tid == 0) snap_cnt[b] = scnt[par];
        // codes from registers
        if (live) {
            const float amax = __half2float(__ushort_as_half(static_cast<unsigned short>(ram[par][rl])));
            const double sc = scale_of(amax);
            const float s32 = static_cast<float>(sc);
            int8_t* qr = xq + (r0 + rl) * ldq;
#pragma unroll
            for (int j = 0; j < RP1_VPT; ++j) {
                const int v = tr + j * TPR;
                if (v < nv) *reinterpret_cast<uint2*>(qr + 8 * v) = quant8(q[j], mbv[j], s32, sc);
            }
            if (tr == 0) {
                row_amax[r0 + rl] = amax;
                for (int64_t k = K; k < ldq; ++k) qr[k] = 0;
            }
        }
    }
}

// Final mask F -> sorted o_idx / o_count (block 0), x[:, O] for every row, and
// the exact correction of blocks whose snapshot S_b missed columns of F.
__global__ void __launch_bounds__(256) rp1_finalize_kernel(
    const __half* __restrict__ x, int64_t M, int64_t K, int64_t ldx,
    const uint32_t* __restrict__ fmask, const uint32_t* __restrict__ snap,
    const int32_t* __restrict__ snap_cnt, int rb, int32_t* __restrict__ o_idx,
    int32_t* __restrict__ o_count, int8_t* __restrict__ xq, int64_t ldq,
    float* __restrict__ row_amax, __half* __restrict__ xo, int64_t o_cap) {
    extern __shared__ __align__(16) uint32_t fz_sm[];
    __shared__ int32_t warp_sums[32];
    __shared__ int32_t n_f;
    pdl_wait();
    pdl_trigger();
    const int nwords = static_cast<int>((K + 31) >> 5);
    uint32_t* sf = fz_sm;                                     // F
    int32_t* scol = reinterpret_cast<int32_t*>(fz_sm + nwords);  // sorted columns of F (cap K)
    const int per = (nwords + blockDim.x - 1) / blockDim.x;
    const int w0 = threadIdx.x * per, w1 = min(nwords, w0 + per);
    int32_t local = 0;
    for (int w = w0; w < w1; ++w) {
        const uint32_t f = fmask[w];
        sf[w] = f;
        local += __popc(f);
    }
    // block exclusive scan of the popcounts -> sorted column list
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int32_t incl = local;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int32_t t = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += t;
    }
    if (lane == 31) warp_sums[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        const int nw = blockDim.x >> 5;
        int32_t sum = lane < nw ? warp_sums[lane] : 0;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int32_t t = __shfl_up_sync(0xffffffffu, sum, d);
            if (lane >= d) sum += t;
        }
        if (lane < nw) warp_sums[lane] = sum;
        if (lane == nw - 1) n_f = sum;
    }
    __syncthreads();
    int32_t pos = incl - local + (wid > 0 ? warp_sums[wid - 1] : 0);
    for (int w = w0; w < w1; ++w)
        for (uint32_t m = sf[w]; m; m &= m - 1) {
            const int32_t c = (w << 5) + __ffs(m) - 1;
            scol[pos] = c;
            if (blockIdx.x == 0) o_idx[pos] = c;
            ++pos;
        }
    __syncthreads();
    const int nf = n_f;
    if (blockIdx.x == 0 && threadIdx.x == 0) *o_count = nf;
    const int n_xo = xo != nullptr ? static_cast<int>(min(static_cast<int64_t>(nf), o_cap)) : 0;
    const int64_t nwarps = blockDim.x >> 5;
    for (int64_t row = blockIdx.x * nwarps + wid; row < M; row += static_cast<int64_t>(gridDim.x) * nwarps) {
        const __half* xr = x + row * ldx;
        for (int t = lane; t < n_xo; t += 32) xo[row * o_cap + t] = xr[scol[t]];
        const int64_t b = row / rb;
        if (snap_cnt[b] == nf) continue;  // S_b == F (S_b is a subset of F)
        // late columns: in F, not in S_b
        const uint32_t* sb = snap + b * nwords;
        const uint32_t am_bits = __half_as_ushort(__float2half_rn(row_amax[row]));
        bool requant = false;
        for (int t = lane; t < nf; t += 32) {
            const int32_t c = scol[t];
            if ((sb[c >> 5] >> (c & 31)) & 1u) continue;
            if ((__half_as_ushort(xr[c]) & 0x7FFFu) == am_bits) requant = true;
        }
        requant = __any_sync(0xffffffffu, requant);
        if (!requant) {
            for (int t = lane; t < nf; t += 32) {
                const int32_t c = scol[t];
                if (!((sb[c >> 5] >> (c & 31)) & 1u)) xq[row * ldq + c] = 0;
            }
            continue;
        }
        // the row max may have been in a late column: redo the row against F
        // (K % 8 == 0 and 16-byte aligned rows on this path)
        const int nvr = static_cast<int>(K >> 3);
        uint32_t am2 = 0;
        for (int v = lane; v < nvr; v += 32) {
            const uint4 q = *reinterpret_cast<const uint4*>(xr + 8 * v);
            const uint32_t mb = (sf[v >> 2] >> (8 * (v & 3))) & 0xFFu;
            const uint32_t w4[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) am2 = __vmaxu2(am2, (w4[e] & 0x7FFF7FFFu) & keep_word(mb, e));
        }
        uint32_t am = max(am2 & 0xFFFFu, am2 >> 16);
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) am = max(am, __shfl_xor_sync(0xffffffffu, am, d));
        const float amax = __half2float(__ushort_as_half(static_cast<unsigned short>(am)));
        const double sc = scale_of(amax);
        const float s32 = static_cast<float>(sc);
        for (int v = lane; v < nvr; v += 32) {
            const uint4 q = *reinterpret_cast<const uint4*>(xr + 8 * v);
            const uint32_t mb = (sf[v >> 2] >> (8 * (v & 3))) & 0xFFu;
            *reinterpret_cast<uint2*>(xq + row * ldq + 8 * v) = quant8(q, mb, s32, sc);
        }
        if (lane == 0) row_amax[row] = amax;
    }
}

bool row_prologue_split_ok(int64_t K, int64_t ldx, int64_t ldq, const void* x, const void* xq) {
    static int env = -1;
    if (env < 0) {
        const char* e = getenv("I8MM_QUANT_SPLIT");
        env = (e && e[0] == '0') ? 0 : 1;
    }
    return env == 1 && K % 8 == 0 && ldx % 8 == 0 && ldq % 8 == 0 && K <= 65536 &&
           (reinterpret_cast<uintptr_t>(x) & 15u) == 0 && (reinterpret_cast<uintptr_t>(xq) & 7u) == 0;
}


// 1-read row prologue (rp1_*): scratch = row_prologue_scratch_bytes(M, K).
// Returns cudaErrorNotSupported when the shape is outside its envelope (the
// caller then runs the 2-read form).
static bool rp1_ok(int64_t M, int64_t K, int64_t ldx, int64_t ldq, const void* x, const void* xq) {
    static int env = -1;
    if (env < 0) {
        const char* e = getenv("I8MM_PROLOGUE_1READ");  // opt-in: measured slower
        env = (e && e[0] == '1') ? 1 : 0;
    }
    if (env != 1 || M <= 0 || K % 8 != 0 || ldx % 8 != 0 || ldq % 8 != 0) return false;
    if ((reinterpret_cast<uintptr_t>(x) & 15u) || (reinterpret_cast<uintptr_t>(xq) & 7u)) return false;
    const Rp1Geom g = rp1_geom(M, K);
    // a row fits the consumers' registers (K <= 32768), >= 2 ring stages
    return (K >> 3) <= RP1_BLOCK_VECS && g.stages >= 2;
}

static size_t rp1_scratch_bytes(int64_t M, int64_t K) {
    const Rp1Geom g = rp1_geom(M > 0 ? M : 1, K);
    const int64_t nwords = (K + 31) >> 5;
    return static_cast<size_t>(((g.nblk * nwords * 4 + 255) / 256) * 256 + g.nblk * 4);
}

static cudaError_t launch_rp1(const __half* x, int64_t M, int64_t K, int64_t ldx, float alpha,
                              uint32_t* mask, int32_t* o_idx, int32_t* o_count, int8_t* xq,
                              int64_t ldq, float* row_amax, __half* xo, int64_t o_cap,
                              void* scratch, cudaStream_t st) {
    const Rp1Geom g = rp1_geom(M, K);
    const int64_t nwords = (K + 31) >> 5;
    uint32_t* snap = static_cast<uint32_t*>(scratch);
    int32_t* snap_cnt = reinterpret_cast<int32_t*>(static_cast<char*>(scratch) +
                                                   ((g.nblk * nwords * 4 + 255) / 256) * 256);
    const int sms = num_sms();
    cudaError_t e;
    if ((e = launch_pdl(zero_u32_kernel, dim3(static_cast<unsigned>(imin64((nwords + 255) / 256, 1024))),
                        dim3(256), 0, st, mask, nwords)))
        return e;
    count_launch();
    // seed F with the first rows (systematic outlier features show up at once),
    // so few blocks are quantized against an incomplete snapshot
    {
        const int64_t seed_rows = imin64(M, 64);
        const int64_t nvec = K >> 3, cb = (nvec + 255) / 256;
        const int64_t rpb = 4, rbs = (seed_rows + rpb - 1) / rpb;
        if ((e = launch_pdl(outlier_scan_vec_kernel<false>, dim3(static_cast<unsigned>(cb), static_cast<unsigned>(rbs)),
                            dim3(256), 0, st, x, seed_rows, K, ldx, alpha_threshold_bits(alpha), rpb, mask,
                            static_cast<int32_t*>(nullptr), static_cast<uint16_t*>(nullptr), int64_t(0),
                            static_cast<int32_t*>(nullptr), static_cast<int32_t*>(nullptr),
                            static_cast<int32_t*>(nullptr), static_cast<int32_t*>(nullptr))))
            return e;
        count_launch();
    }
    const size_t smem = static_cast<size_t>(g.stages) * g.stage_bytes;
    const unsigned grid = static_cast<unsigned>(imin64(g.nblk, sms));
    auto go = [&](auto kern) -> cudaError_t {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, RP1_SMEM_RING);
        return launch_pdl(kern, dim3(grid), dim3(RP1_THREADS), smem, st, x, M, K, ldx,
                          alpha_threshold_bits(alpha), mask, snap, snap_cnt, xq, ldq, row_amax);
    };
    switch (g.rb) {
        case 1: e = go(rp1_stream_kernel<1>); break;
        case 2: e = go(rp1_stream_kernel<2>); break;
        case 4: e = go(rp1_stream_kernel<4>); break;
        case 8: e = go(rp1_stream_kernel<8>); break;
        default: e = go(rp1_stream_kernel<16>); break;
    }
    if (e) return e;
    count_launch();
    const size_t fsmem = static_cast<size_t>(nwords) * 4 + static_cast<size_t>(K) * 4;
    static size_t fconfigured = 0;
    if (fsmem > 48 * 1024 && fsmem > fconfigured) {
        cudaFuncSetAttribute(rp1_finalize_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(fsmem));
        fconfigured = fsmem;
    }
    const int64_t fgrid = imin64((M + 7) / 8, static_cast<int64_t>(sms) * 4);
    if ((e = launch_pdl(rp1_finalize_kernel, dim3(static_cast<unsigned>(fgrid)), dim3(256), fsmem, st, x, M,
                        K, ldx, static_cast<const uint32_t*>(mask), static_cast<const uint32_t*>(snap),
                        static_cast<const int32_t*>(snap_cnt), g.rb, o_idx, o_count, xq, ldq, row_amax,
                        xo, o_cap)))
        return e;
    count_launch();
    return cudaGetLastError();
}
size_t row_prologue_scratch_bytes(int64_t M, int64_t K) {
    const int64_t ng = (K + 63) >> 6;
    const size_t two = static_cast<size_t>(((M * ng * 2 + 255) / 256) * 256 + M * 8 + (34 + ng) * 4);
    const size_t one = rp1_scratch_bytes(M, K);
    return one > two ? one : two;
}

cudaError_t launch_row_prologue(const __half* x, int64_t M, int64_t K, int64_t ldx, float alpha,
                                uint32_t* mask, int32_t* o_idx, int32_t* o_count, int8_t* xq,
                                int64_t ldq, float* row_amax, __half* xo, int64_t o_cap,
                                void* scratch, cudaStream_t st, const PerCallFix* fix,
                                int32_t* nonfinite) {
    cudaError_t e;
    uint32_t* zero2 = fix != nullptr ? reinterpret_cast<uint32_t*>(fix->p_count) : nullptr;
    const int64_t zero2_n = fix != nullptr ? fixup_zero_words(fix->N) : 0;
    const bool split = M > 0 && scratch != nullptr && row_prologue_split_ok(K, ldx, ldq, x, xq) &&
                       !rp1_ok(M, K, ldx, ldq, x, xq);
    if (!split) {  // unfused forms: the per-call weight work runs as its own launches
        if (zero2 != nullptr) {
            if ((e = launch_pdl(zero_u32_kernel, dim3(static_cast<unsigned>(imin64((zero2_n + 255) / 256, 64))),
                                dim3(256), 0, st, zero2, zero2_n)))
                return e;
            count_launch();
        }
        if (fix != nullptr && fix->c32 != nullptr && fix->c32_words > 0) {
            if ((e = launch_pdl(zero_u32_kernel, dim3(static_cast<unsigned>(imin64((fix->c32_words + 255) / 256, 1184))),
                                dim3(256), 0, st, reinterpret_cast<uint32_t*>(fix->c32), fix->c32_words)))
                return e;
            count_launch();
        }
        if (nonfinite != nullptr && (e = cudaMemsetAsync(nonfinite, 0, sizeof(int32_t), st))) return e;
        if (M == 0 || scratch == nullptr || !row_prologue_split_ok(K, ldx, ldq, x, xq)) {
            if ((e = launch_outlier_scan(x, M, K, ldx, alpha, mask, nonfinite, st))) return e;
            if ((e = launch_outlier_compact(mask, K, o_idx, o_count, st))) return e;
            e = launch_quantize_rows(x, M, K, ldx, mask, o_idx, o_count, xq, ldq, row_amax, xo, o_cap, st);
        } else {
            e = launch_rp1(x, M, K, ldx, alpha, mask, o_idx, o_count, xq, ldq, row_amax, xo, o_cap, scratch, st);
        }
        if (e || fix == nullptr) return e;
        if ((e = launch_gather_fixup(fix->w, fix->K, fix->N, fix->ldw, mask, o_idx, o_count, o_cap, fix->wo,
                                     fix->ldwo, fix->amax_full, fix->cand_v, fix->cand_r, fix->p_count,
                                     fix->p_idx, fix->p_amax, fix->p_src, st)))
            return e;
        return launch_patch_quantize(fix->w, fix->K, fix->N, fix->ldw, mask, fix->q2, fix->p_count,
                                     fix->p_idx, fix->p_amax, fix->p_src, fix->wq_p, ldq, st);
    }
    const int64_t nwords = (K + 31) >> 5, nvec = K >> 3, ng = (K + 63) >> 6;
    uint16_t* gmax = static_cast<uint16_t*>(scratch);
    double* row_s = reinterpret_cast<double*>(static_cast<char*>(scratch) + ((M * ng * 2 + 255) / 256) * 256);
    int32_t* dgrp = reinterpret_cast<int32_t*>(row_s + M);
    int32_t* done_ctr = dgrp + 33 + ng;  // scan CTAs finished (the last one compacts)
    const int sms = num_sms();
    {
        const int64_t n2 = zero2 != nullptr ? zero2_n : 0;
        uint32_t* z3 = fix != nullptr ? reinterpret_cast<uint32_t*>(fix->c32) : nullptr;
        const int64_t n3 = z3 != nullptr ? fix->c32_words : 0;
        const int64_t work = nwords + n2 + n3 / 4 + 256;
        if ((e = launch_pdl(zero2_u32_kernel, dim3(static_cast<unsigned>(imin64(work / 256 + 1, 1184))),
                            dim3(256), 0, st, mask, nwords, zero2, n2,
                            reinterpret_cast<uint32_t*>(done_ctr), z3, n3,
                            reinterpret_cast<uint32_t*>(nonfinite))))
            return e;
        count_launch();
    }
    const int64_t cb = (nvec + 255) / 256;
    int64_t rpb;
    int rb = grid_rows_chunk(M, cb, static_cast<int64_t>(sms) * 8, &rpb);
    if ((e = launch_pdl(outlier_scan_vec_kernel<true>, dim3(static_cast<unsigned>(cb), rb), dim3(256), 0, st,
                        x, M, K, ldx, alpha_threshold_bits(alpha), rpb, mask,
                        nonfinite, gmax, ng, done_ctr, o_idx, o_count, dgrp)))
        return e;
    count_launch();
    const int64_t rs_grid = imin64((M + 7) / 8, static_cast<int64_t>(sms) * 8);
    const RowScaleArgs ra{x, M, K, ldx, mask, o_idx, o_count, gmax, ng, dgrp, row_amax, row_s, xo, o_cap};
    if (fix == nullptr) {
        if ((e = launch_pdl(row_scale_kernel, dim3(static_cast<unsigned>(rs_grid)), dim3(256), 0, st, ra)))
            return e;
    } else {
        const int vec = (fix->N % 8 == 0) && (fix->ldw % 8 == 0) && (fix->ldwo % 8 == 0) &&
                        (reinterpret_cast<uintptr_t>(fix->w) & 15u) == 0 &&
                        (reinterpret_cast<uintptr_t>(fix->wo) & 15u) == 0;
        const int64_t per = vec ? (fix->N >> 3) : fix->N;
        const int64_t gx = imin64((per + 255) / 256, 16);
        const int64_t blocks = rs_grid + o_cap * gx + (fix->N + 255) / 256;
        if ((e = launch_pdl(row_scale_fix_kernel, dim3(static_cast<unsigned>(blocks)), dim3(256), 0, st, ra,
                            rs_grid, *fix, vec, gx)))
            return e;
    }
    count_launch();
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(quantize_bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             QS_STAGES * QS_STAGE_BYTES);
        configured = true;
    }
    const int64_t ntiles = ((M + QS_ROWS - 1) / QS_ROWS) * ((nvec + QS_VECS - 1) / QS_VECS);
    const unsigned g = static_cast<unsigned>(imin64(ntiles, static_cast<int64_t>(sms) * 2));
    PerCallFix pf{};
    if (fix != nullptr) pf = *fix;
    // tiles in reverse order: the scan just streamed X top to bottom, so the bottom
    // rows are the ones still in L2 (fc1 16384 x 4096: 76 -> 73.6 us per prologue)
    static const int rev = [] {
        const char* v = getenv("I8MM_QS_REVERSE");
        return v ? atoi(v) : 1;
    }();
    if ((e = launch_pdl(quantize_bulk_kernel, dim3(g), dim3(288), QS_STAGES * QS_STAGE_BYTES, st, x, M, K, ldx,
                        static_cast<const uint32_t*>(mask), static_cast<const double*>(row_s), xq, ldq, pf, rev)))
        return e;
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_dequantize_output(const int32_t* c, int64_t M, int64_t N, int64_t ldc,
                                     const double* sx, const double* sw, float* out, int64_t ldo,
                                     cudaStream_t st) {
    if (M * N == 0) return cudaSuccess;
    const int64_t blocks = imin64((M * N + 255) / 256, static_cast<int64_t>(num_sms()) * 16);
    dequantize_output_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(c, M, N, ldc, sx, sw,
                                                                             out, ldo);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_transpose_i8(const int8_t* src, int64_t rows, int64_t cols, int64_t lds,
                                int8_t* dst, int64_t ldd, cudaStream_t st) {
    if (rows * cols == 0) return cudaSuccess;
    dim3 grid(static_cast<unsigned>((cols + 31) / 32), static_cast<unsigned>((rows + 31) / 32));
    transpose_i8_kernel<<<grid, dim3(32, 8), 0, st>>>(src, rows, cols, lds, dst, ldd);
    count_launch();
    return cudaGetLastError();
}

}  // namespace i8mm
