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

#include "kernels.cuh"

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

// ------------------------------------------------------------------ K1 scan
// Vector path: each thread owns 8 consecutive columns (one 16-byte load per
// row) for a chunk of rows; 4 adjacent lanes form one 32-bit mask word.
__global__ void outlier_scan_vec_kernel(const __half* __restrict__ x, int64_t M, int64_t K,
                                        int64_t ldx, float alpha, int64_t rows_per_block,
                                        uint32_t* __restrict__ col_mask,
                                        int32_t* __restrict__ nonfinite) {
    const int64_t v = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;  // vector col
    const int64_t nvec = K >> 3;
    const int64_t r0 = static_cast<int64_t>(blockIdx.y) * rows_per_block;
    const int64_t r1 = min(M, r0 + rows_per_block);
    uint32_t bits = 0, bad = 0;
    if (v < nvec) {
        const __half* p = x + r0 * ldx + (v << 3);
        int64_t r = r0;
        for (; r + 4 <= r1; r += 4) {
            uint4 q[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) q[u] = ld_stream_u4(p + u * ldx);
            p += 4 * ldx;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const __half* h = reinterpret_cast<const __half*>(&q[u]);
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    bits |= (fabsf(__half2float(h[e])) >= alpha ? 1u : 0u) << e;
                    bad |= h_is_nonfinite(h[e]) ? 1u : 0u;
                }
            }
        }
        for (; r < r1; ++r, p += ldx) {
            uint4 q = ld_stream_u4(p);
            const __half* h = reinterpret_cast<const __half*>(&q);
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                bits |= (fabsf(__half2float(h[e])) >= alpha ? 1u : 0u) << e;
                bad |= h_is_nonfinite(h[e]) ? 1u : 0u;
            }
        }
    }
    const uint32_t lane = threadIdx.x & 31u;
    uint32_t word = bits << (8u * (lane & 3u));
    word |= __shfl_xor_sync(0xffffffffu, word, 1);
    word |= __shfl_xor_sync(0xffffffffu, word, 2);
    if ((lane & 3u) == 0 && word != 0 && v < nvec) atomicOr(col_mask + (v >> 2), word);
    if (nonfinite != nullptr && __any_sync(0xffffffffu, bad != 0) && lane == 0)
        atomicExch(nonfinite, 1);
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
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        p[i] = 0u;
}

// ------------------------------------------------------------------ compact
// One block: prefix popcount over the mask words, scatter sorted indices.
__global__ void outlier_compact_kernel(const uint32_t* __restrict__ col_mask, int64_t K,
                                       int32_t* __restrict__ o_idx, int32_t* __restrict__ o_count) {
    __shared__ int32_t warp_sums[32];
    const int64_t nwords = (K + 31) >> 5;
    const int64_t per = (nwords + blockDim.x - 1) / blockDim.x;
    const int64_t w0 = threadIdx.x * per;
    const int64_t w1 = min(nwords, w0 + per);
    int32_t local = 0;
    for (int64_t w = w0; w < w1; ++w) local += __popc(col_mask[w]);
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
        uint32_t m = col_mask[w];
        while (m) {
            const int b = __ffs(m) - 1;
            m &= m - 1;
            o_idx[pos++] = static_cast<int32_t>((w << 5) + b);
        }
    }
    if (threadIdx.x == blockDim.x - 1) *o_count = pos;
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

// One block per row; the row stays in registers (VPT 16-byte vectors/thread).
template <int VPT>
__global__ void __launch_bounds__(512) quantize_rows_vec_kernel(const __half* __restrict__ x, int64_t K, int64_t ldx,
                                         const uint32_t* __restrict__ col_mask,
                                         const int32_t* __restrict__ o_idx,
                                         const int32_t* __restrict__ o_count,
                                         int8_t* __restrict__ xq, int64_t ldq,
                                         float* __restrict__ row_amax, __half* __restrict__ xo,
                                         int64_t o_cap) {
    __shared__ float red[32];
    const int64_t row = blockIdx.x;
    const int64_t nvec = K >> 3;
    const __half* xr = x + row * ldx;
    uint4 q[VPT];
    uint32_t mb[VPT];
    float amax = 0.0f;
#pragma unroll
    for (int j = 0; j < VPT; ++j) {
        const int64_t v = threadIdx.x + static_cast<int64_t>(j) * blockDim.x;
        if (v < nvec) {
            q[j] = ld_stream_u4(xr + (v << 3));
            mb[j] = col_mask ? mask_byte(col_mask, v) : 0u;
            const __half* h = reinterpret_cast<const __half*>(&q[j]);
#pragma unroll
            for (int e = 0; e < 8; ++e)
                if (!((mb[j] >> e) & 1u)) amax = fmaxf(amax, fabsf(__half2float(h[e])));
        }
    }
    amax = block_max(amax, red);
    const double s = scale_of(amax);
    int8_t* qr = xq + row * ldq;
#pragma unroll
    for (int j = 0; j < VPT; ++j) {
        const int64_t v = threadIdx.x + static_cast<int64_t>(j) * blockDim.x;
        if (v < nvec) {
            const __half* h = reinterpret_cast<const __half*>(&q[j]);
            uint32_t lo = 0, hi = 0;
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const int8_t c = ((mb[j] >> e) & 1u) ? int8_t(0) : code_of(__half2float(h[e]), s);
                const uint32_t b = static_cast<uint32_t>(static_cast<uint8_t>(c));
                if (e < 4) lo |= b << (8 * e);
                else hi |= b << (8 * (e - 4));
            }
            *reinterpret_cast<uint2*>(qr + (v << 3)) = make_uint2(lo, hi);
        }
    }
    if (threadIdx.x == 0) row_amax[row] = amax;
    if (xo != nullptr && o_count != nullptr) {
        const int64_t n = min(static_cast<int64_t>(*o_count), o_cap);
        for (int64_t t = threadIdx.x; t < n; t += blockDim.x) xo[row * o_cap + t] = xr[o_idx[t]];
    }
    // zero the K..ldq padding so the codes buffer is fully defined
    for (int64_t k = K + threadIdx.x; k < ldq; k += blockDim.x) qr[k] = 0;
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

// ------------------------------------------------------------------ K3 cols
// Column absmax over keep rows. Threads own 2 adjacent columns (half2), the
// grid splits K into chunks; partial maxima merge with an integer atomicMax
// on the float bit pattern (valid: amax >= 0). col_amax must be zeroed.
__global__ void col_amax_kernel(const __half* __restrict__ w, int64_t K, int64_t N, int64_t ldw,
                                const uint32_t* __restrict__ row_mask, int64_t rows_per_block,
                                float* __restrict__ col_amax) {
    const int64_t j = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 2;
    const int64_t k0 = static_cast<int64_t>(blockIdx.y) * rows_per_block;
    const int64_t k1 = min(K, k0 + rows_per_block);
    if (j >= N) return;
    float m0 = 0.0f, m1 = 0.0f;
    const bool pair = (j + 1 < N) && ((ldw & 1) == 0);
    for (int64_t k = k0; k < k1; ++k) {
        if (row_mask && ((row_mask[k >> 5] >> (k & 31)) & 1u)) continue;  // block-uniform
        if (pair) {
            const float2 f = __half22float2(*reinterpret_cast<const __half2*>(w + k * ldw + j));
            m0 = fmaxf(m0, fabsf(f.x));
            m1 = fmaxf(m1, fabsf(f.y));
        } else {
            m0 = fmaxf(m0, fabsf(__half2float(w[k * ldw + j])));
            if (j + 1 < N) m1 = fmaxf(m1, fabsf(__half2float(w[k * ldw + j + 1])));
        }
    }
    atomicMax(reinterpret_cast<int*>(col_amax + j), __float_as_int(m0));
    if (j + 1 < N) atomicMax(reinterpret_cast<int*>(col_amax + j + 1), __float_as_int(m1));
}

// Quantize a 64(k) x 64(n) tile of W and store it transposed (WqT[n][k]).
__global__ void quantize_cols_t_kernel(const __half* __restrict__ w, int64_t K, int64_t N,
                                       int64_t ldw, const uint32_t* __restrict__ row_mask,
                                       const float* __restrict__ col_amax,
                                       int8_t* __restrict__ wq_t, int64_t ldq) {
    __shared__ double sc[64];
    __shared__ int8_t tile[64][64 + 4];  // [n][k]
    const int64_t n0 = static_cast<int64_t>(blockIdx.x) * 64;
    const int64_t k0 = static_cast<int64_t>(blockIdx.y) * 64;
    const int tid = threadIdx.x;  // 256 threads
    if (tid < 64) sc[tid] = (n0 + tid < N) ? scale_of(col_amax[n0 + tid]) : 1.0;
    __syncthreads();
    // each thread: one k row (tid / 4), 16 columns ((tid % 4) * 16 ..)
    const int kr = tid >> 2;
    const int nc = (tid & 3) * 16;
    const int64_t k = k0 + kr;
    const bool kvalid = k < K;
    const bool out = kvalid && row_mask && ((row_mask[k >> 5] >> (k & 31)) & 1u);
#pragma unroll 4
    for (int e = 0; e < 16; ++e) {
        const int64_t n = n0 + nc + e;
        int8_t c = 0;
        if (kvalid && !out && n < N) c = code_of(__half2float(w[k * ldw + n]), sc[nc + e]);
        tile[nc + e][kr] = c;
    }
    __syncthreads();
    // store: each thread writes 16 bytes (one n row, 16 k) -> 64 rows x 4 chunks
    const int nr = tid >> 2;
    const int kc = (tid & 3) * 16;
    const int64_t n = n0 + nr;
    if (n < N) {
        int8_t* dst = wq_t + n * ldq + k0 + kc;
        const int64_t lim = imin64(16, ldq - (k0 + kc));
        if (lim == 16 && ((reinterpret_cast<uintptr_t>(dst) & 15u) == 0)) {
            uint32_t wv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
                wv[u] = static_cast<uint32_t>(static_cast<uint8_t>(tile[nr][kc + 4 * u])) |
                        static_cast<uint32_t>(static_cast<uint8_t>(tile[nr][kc + 4 * u + 1])) << 8 |
                        static_cast<uint32_t>(static_cast<uint8_t>(tile[nr][kc + 4 * u + 2])) << 16 |
                        static_cast<uint32_t>(static_cast<uint8_t>(tile[nr][kc + 4 * u + 3])) << 24;
            *reinterpret_cast<uint4*>(dst) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
        } else {
            for (int64_t u = 0; u < lim; ++u) dst[u] = tile[nr][kc + u];
        }
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
static inline int grid_rows_chunk(int64_t M, int64_t col_blocks, int64_t target_blocks,
                                  int64_t* rows_per_block) {
    int64_t chunks = (target_blocks + col_blocks - 1) / col_blocks;
    if (chunks < 1) chunks = 1;
    if (chunks > M) chunks = M;
    int64_t rpb = (M + chunks - 1) / chunks;
    if (rpb < 1) rpb = 1;
    *rows_per_block = rpb;
    return static_cast<int>((M + rpb - 1) / rpb);
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
        outlier_scan_vec_kernel<<<dim3(static_cast<unsigned>(cb), rb), 256, 0, st>>>(
            x, M, K, ldx, alpha, rpb, col_mask, nonfinite);
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
    outlier_compact_kernel<<<1, 1024, 0, st>>>(col_mask, K, o_idx, o_count);
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
    const bool vec = (K % 8 == 0) && (K <= 65536) && (ldx % 8 == 0) && (ldq % 8 == 0) &&
                     ((reinterpret_cast<uintptr_t>(x) & 15u) == 0) &&
                     ((reinterpret_cast<uintptr_t>(xq) & 7u) == 0);
    if (!vec) {
        quantize_rows_scalar_kernel<<<static_cast<unsigned>(M), 256, 0, st>>>(
            x, K, ldx, mask, o_idx, o_count, xq, ldq, amax, xo, o_cap);
        count_launch();
        return cudaGetLastError();
    }
    const int64_t nvec = K >> 3;
    int vpt = 1;
    while (vpt < 16 && (nvec + vpt - 1) / vpt > 512) vpt <<= 1;
    int64_t threads = (nvec + vpt - 1) / vpt;
    threads = ((threads + 31) / 32) * 32;
    if (threads < 64) threads = 64;
    if (threads > 1024) return cudaErrorInvalidValue;
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

cudaError_t launch_quantize_cols_t(const __half* w, int64_t K, int64_t N, int64_t ldw,
                                   const uint32_t* row_mask, int8_t* wq_t, int64_t ldq,
                                   float* col_amax, cudaStream_t st) {
    if (N == 0) return cudaSuccess;
    zero_u32_kernel<<<static_cast<unsigned>(imin64((N + 255) / 256, 1024)), 256, 0, st>>>(
        reinterpret_cast<uint32_t*>(col_amax), N);
    count_launch();
    const int64_t cb = ((N + 1) / 2 + 255) / 256;
    int64_t rpb;
    const int rb = grid_rows_chunk(K, cb, static_cast<int64_t>(num_sms()) * 8, &rpb);
    col_amax_kernel<<<dim3(static_cast<unsigned>(cb), rb), 256, 0, st>>>(w, K, N, ldw, row_mask,
                                                                           rpb, col_amax);
    count_launch();
    const int64_t kt = (ldq + 63) / 64;  // cover the padding columns too (written as 0)
    quantize_cols_t_kernel<<<dim3(static_cast<unsigned>((N + 63) / 64), static_cast<unsigned>(kt)),
                             256, 0, st>>>(w, K, N, ldw, row_mask, col_amax, wq_t, ldq);
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
