// W-side kernels of the LLM.int8() path (CUDA cores, HBM-bound).
//
// Per-call column-wise quantization (the reference's exact semantics,
// quantize.py:182-187 applied to w[keep, :], gemm.py:243):
//   col_amax_vec      -- column absmax over keep rows, 8 columns / thread
//   quantize_cols_t   -- codes written transposed (WqT, K-major) for the GEMM
//   gather_rows       -- compact copy of the outlier rows W[O, :] (gemm.py:238)
//
// Weight-stationary form (exact by construction):
//   prepare:  WqT and column amax over ALL rows, plus each column's top-T
//             |w| candidates (value, row);
//   per call: a column's amax over keep rows differs from the cached one only
//             if its cached maximisers are all outlier rows. fixup_kernel walks
//             the candidates against the outlier mask and lists those columns
//             (the "patches", ~|O| N / K of them), patch_quantize re-derives
//             their codes, and the GEMM runs once over the cached codes and
//             once (col-mapped) over the patches, overwriting those columns.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"
#include "quant_common.cuh"
#include "sm100_ptx.cuh"
#include "percall_dev.cuh"

namespace i8mm {


// ------------------------------------------------------------------ amax
// Each thread owns 8 adjacent columns (one 16-byte load per row) over a chunk
// of rows; outlier rows are skipped (block-uniform branch). Partial maxima
// merge with an unsigned atomicMax on the fp16 bit pattern (|w| >= 0, so bit
// order == value order). amax_bits must be zeroed.
__global__ void col_amax_vec_kernel(const __half* __restrict__ w, int64_t K, int64_t N, int64_t ldw,
                                    const uint32_t* __restrict__ row_mask, int64_t rows_per_block,
                                    uint32_t* __restrict__ amax_bits) {
    const int64_t v = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t k0 = static_cast<int64_t>(blockIdx.y) * rows_per_block;
    const int64_t k1 = imin64(K, k0 + rows_per_block);
    if (v >= (N >> 3)) return;
    uint32_t m[4] = {0, 0, 0, 0};
    const __half* p = w + (v << 3);
    auto fold = [&](const uint4& q) {
        m[0] = __vmaxu2(m[0], q.x & 0x7FFF7FFFu);
        m[1] = __vmaxu2(m[1], q.y & 0x7FFF7FFFu);
        m[2] = __vmaxu2(m[2], q.z & 0x7FFF7FFFu);
        m[3] = __vmaxu2(m[3], q.w & 0x7FFF7FFFu);
    };
    // 8 rows per step: the loads are issued unconditionally (an outlier row's is
    // discarded), so they are in flight together instead of each waiting on the
    // row-mask lookup that decides whether to load it
    constexpr int U = 8;
    int64_t k = k0;
    for (; k + U <= k1; k += U) {
        uint4 q[U];
#pragma unroll
        for (int u = 0; u < U; ++u) q[u] = ld_stream_u4(p + (k + u) * ldw);
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (!row_is_out(row_mask, k + u)) fold(q[u]);
    }
    for (; k < k1; ++k)
        if (!row_is_out(row_mask, k)) fold(ld_stream_u4(p + k * ldw));
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        if (m[i] & 0xFFFFu) atomicMax(amax_bits + (v << 3) + 2 * i, m[i] & 0xFFFFu);
        if (m[i] >> 16) atomicMax(amax_bits + (v << 3) + 2 * i + 1, m[i] >> 16);
    }
}

// Scalar fallback (N % 8 != 0 or unaligned W).
__global__ void col_amax_scalar_kernel(const __half* __restrict__ w, int64_t K, int64_t N,
                                       int64_t ldw, const uint32_t* __restrict__ row_mask,
                                       int64_t rows_per_block, uint32_t* __restrict__ amax_bits) {
    const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t k0 = static_cast<int64_t>(blockIdx.y) * rows_per_block;
    const int64_t k1 = imin64(K, k0 + rows_per_block);
    if (j >= N) return;
    uint32_t m = 0;
    for (int64_t k = k0; k < k1; ++k) {
        if (row_is_out(row_mask, k)) continue;
        m = max(m, static_cast<uint32_t>(__half_as_ushort(w[k * ldw + j])) & 0x7FFFu);
    }
    if (m) atomicMax(amax_bits + j, m);
}

// fp16 amax bits -> float amax (in place: the buffer is reused as float[N])
__global__ void amax_bits_to_float_kernel(uint32_t* a, int64_t n) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const float f = half_bits_to_float(a[i]);
        a[i] = __float_as_uint(f);
    }
}

__global__ void zero_words_kernel(uint32_t* p, int64_t n) {
    pdl_wait();
    pdl_trigger();
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        p[i] = 0u;
}

// ------------------------------------------------------------------ codes
// 64(k) x 64(n) tile: coalesced 16-byte loads of W rows, fast exact
// quantization with the column scale, transpose through smem, 16-byte stores
// of WqT rows. Outlier rows and the K..ldq padding are written as 0.
__global__ void __launch_bounds__(256) quantize_cols_t_kernel(
    const __half* __restrict__ w, int64_t K, int64_t N, int64_t ldw,
    const uint32_t* __restrict__ row_mask, const float* __restrict__ col_amax,
    int8_t* __restrict__ wq_t, int64_t ldq, int vec) {
    __shared__ double sc[64];
    __shared__ float sc32[64];
    __shared__ uint32_t tile[64][64 / 4 + 1];  // [n][k/4] packed bytes (+1 pad)
    const int64_t n0 = static_cast<int64_t>(blockIdx.x) * 64;
    const int64_t k0 = static_cast<int64_t>(blockIdx.y) * 64;
    const int tid = threadIdx.x;
    if (tid < 64) {
        const double s = (n0 + tid < N) ? scale_of(col_amax[n0 + tid]) : 1.0;
        sc[tid] = s;
        sc32[tid] = static_cast<float>(s);
    }
    __syncthreads();
    // thread -> (4 consecutive k rows, 8 consecutive n columns): 16 x 8 threads
    const int kq = tid >> 3;         // 0..31 -> k rows 2*kq, 2*kq+1 ... use 2 rows
    const int nv = (tid & 7) * 8;    // column group
    uint32_t packed[8][1];
#pragma unroll
    for (int e = 0; e < 8; ++e) packed[e][0] = 0;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const int kr = kq * 2 + r;
        const int64_t k = k0 + kr;
        int c8[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        if (k < K && !row_is_out(row_mask, k)) {
            const __half* src = w + k * ldw + n0 + nv;
            if (vec && n0 + nv + 8 <= N) {
                const uint4 q = *reinterpret_cast<const uint4*>(src);
                const __half* h = reinterpret_cast<const __half*>(&q);
#pragma unroll
                for (int e = 0; e < 8; ++e) c8[e] = code_fast(__half2float(h[e]), sc32[nv + e], sc[nv + e]);
            } else {
                for (int e = 0; e < 8; ++e)
                    if (n0 + nv + e < N) c8[e] = code_fast(__half2float(src[e]), sc32[nv + e], sc[nv + e]);
            }
            // |x| above the column amax only occurs for the q2 codes (top-1 row
            // under the second candidate's scale): clip like quantize.py:117
#pragma unroll
            for (int e = 0; e < 8; ++e) c8[e] = max(-127, min(127, c8[e]));
        }
#pragma unroll
        for (int e = 0; e < 8; ++e)
            packed[e][0] |= (static_cast<uint32_t>(c8[e]) & 0xFFu) << (8 * (kr & 3));
    }
    // rows kq*2, kq*2+1 live in byte lanes (kr & 3) of word (kr >> 2); two
    // threads (kq even/odd) share a word: combine with a shuffle.
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const uint32_t other = __shfl_xor_sync(0xffffffffu, packed[e][0], 8);
        packed[e][0] |= other;
    }
    if ((kq & 1) == 0) {
#pragma unroll
        for (int e = 0; e < 8; ++e) tile[nv + e][kq >> 1] = packed[e][0];
    }
    __syncthreads();
    // store: 64 n rows x 64 k bytes = 64 x 4 chunks of 16 B -> one per thread
    const int nr = tid >> 2;
    const int kc = (tid & 3) * 16;
    const int64_t n = n0 + nr;
    if (n < N) {
        int8_t* dst = wq_t + n * ldq + k0 + kc;
        const int64_t lim = imin64(16, ldq - (k0 + kc));
        const uint4 val = make_uint4(tile[nr][kc / 4], tile[nr][kc / 4 + 1], tile[nr][kc / 4 + 2],
                                     tile[nr][kc / 4 + 3]);
        if (lim == 16 && ((reinterpret_cast<uintptr_t>(dst) & 15u) == 0)) {
            *reinterpret_cast<uint4*>(dst) = val;
        } else if (lim > 0) {
            const int8_t* b = reinterpret_cast<const int8_t*>(&val);
            for (int64_t u = 0; u < lim; ++u) dst[u] = b[u];
        }
    }
}

// ------------------------------------------------------------------ gather
// out[t, :] = w[idx[t], :] for t < min(*count, cap) (compact outlier rows).

__global__ void gather_rows_kernel(const __half* __restrict__ w, int64_t ldw, int64_t N,
                                   const int32_t* __restrict__ idx, const int32_t* __restrict__ count,
                                   int64_t cap, __half* __restrict__ out, int64_t ldo, int vec) {
    pdl_wait();
    pdl_trigger();
    gather_rows_block(w, ldw, N, idx, count, cap, out, ldo, vec, blockIdx.y, blockIdx.x, gridDim.x);
}

// ------------------------------------------------------------------ top-T

struct TopT {
    uint32_t v[TOPT];  // |w| fp16 bits, descending
    int32_t r[TOPT];   // row, -1 = empty
    __device__ __forceinline__ void init() {
#pragma unroll
        for (int i = 0; i < TOPT; ++i) {
            v[i] = 0;
            r[i] = -1;
        }
    }
    // keep the T largest; on equal values the earlier-inserted entry stays first
    __device__ __forceinline__ void insert(uint32_t val, int32_t row) {
        int pos = TOPT;
#pragma unroll
        for (int i = TOPT - 1; i >= 0; --i)
            if (r[i] < 0 || val > v[i]) pos = i;
        if (pos == TOPT) return;
#pragma unroll
        for (int i = TOPT - 1; i > 0; --i)
            if (i > pos) {
                v[i] = v[i - 1];
                r[i] = r[i - 1];
            }
#pragma unroll
        for (int i = 0; i < TOPT; ++i)
            if (i == pos) {
                v[i] = val;
                r[i] = row;
            }
    }
};

// partial top-T over a chunk of rows, 2 columns per thread (half2 loads)
__global__ void topt_partial_kernel(const __half* __restrict__ w, int64_t K, int64_t N,
                                    int64_t ldw, int64_t rows_per_block,
                                    uint32_t* __restrict__ pv, int32_t* __restrict__ pr) {
    const int64_t j = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 2;
    const int64_t chunk = blockIdx.y;
    const int64_t k0 = chunk * rows_per_block;
    const int64_t k1 = imin64(K, k0 + rows_per_block);
    if (j >= N) return;
    TopT a, b;
    a.init();
    b.init();
    const bool pair = (j + 1 < N) && ((ldw & 1) == 0);
    for (int64_t k = k0; k < k1; ++k) {
        if (pair) {
            const uint32_t q = *reinterpret_cast<const uint32_t*>(w + k * ldw + j);
            a.insert(q & 0x7FFFu, static_cast<int32_t>(k));
            b.insert((q >> 16) & 0x7FFFu, static_cast<int32_t>(k));
        } else {
            a.insert(__half_as_ushort(w[k * ldw + j]) & 0x7FFFu, static_cast<int32_t>(k));
            if (j + 1 < N) b.insert(__half_as_ushort(w[k * ldw + j + 1]) & 0x7FFFu, static_cast<int32_t>(k));
        }
    }
#pragma unroll
    for (int i = 0; i < TOPT; ++i) {
        pv[(chunk * TOPT + i) * N + j] = a.v[i];
        pr[(chunk * TOPT + i) * N + j] = a.r[i];
        if (j + 1 < N) {
            pv[(chunk * TOPT + i) * N + j + 1] = b.v[i];
            pr[(chunk * TOPT + i) * N + j + 1] = b.r[i];
        }
    }
}

// merge the per-chunk candidates (ascending chunk = ascending row order, so
// equal values keep the lower row first) into the final top-T per column
__global__ void topt_merge_kernel(int64_t N, int64_t chunks, const uint32_t* __restrict__ pv,
                                  const int32_t* __restrict__ pr, uint16_t* __restrict__ cand_v,
                                  int32_t* __restrict__ cand_r) {
    const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= N) return;
    TopT a;
    a.init();
    for (int64_t c = 0; c < chunks; ++c)
#pragma unroll
        for (int i = 0; i < TOPT; ++i) {
            const int32_t r = pr[(c * TOPT + i) * N + j];
            if (r >= 0) a.insert(pv[(c * TOPT + i) * N + j], r);
        }
#pragma unroll
    for (int i = 0; i < TOPT; ++i) {
        cand_v[i * N + j] = static_cast<uint16_t>(a.v[i]);
        cand_r[i * N + j] = a.r[i];
    }
}

// ------------------------------------------------------------------ fixup
// One thread per column: the column's amax over keep rows from the cached
// candidates (full rescan only if every candidate row is an outlier row).
// Columns whose amax changes are appended to the patch list.

// One launch for the two independent consumers of the outlier set: blocks
// [0, cap * gx) gather W[O, :] (row t = b / gx), the rest run the column fixup.
__global__ void gather_fixup_kernel(const __half* __restrict__ w, int64_t K, int64_t N, int64_t ldw,
                                    const uint32_t* __restrict__ mask, const int32_t* __restrict__ o_idx,
                                    const int32_t* __restrict__ o_count, int64_t o_cap,
                                    __half* __restrict__ wo, int64_t ldwo, int vec, int64_t gx,
                                    const float* __restrict__ amax_full,
                                    const uint16_t* __restrict__ cand_v,
                                    const int32_t* __restrict__ cand_r, int32_t* __restrict__ p_count,
                                    int32_t* __restrict__ p_idx, float* __restrict__ p_amax,
                                    int32_t* __restrict__ p_src) {
    pdl_wait();
    pdl_trigger();
    const int64_t b = blockIdx.x, ng = o_cap * gx;
    if (b < ng) {
        gather_rows_block(w, ldw, N, o_idx, o_count, o_cap, wo, ldwo, vec, b / gx, b % gx, gx);
        return;
    }
    fixup_column(w, K, N, ldw, mask, amax_full, cand_v, cand_r, p_count, p_idx, p_amax, p_src,
                 (b - ng) * blockDim.x + threadIdx.x);
}

// codes of the patched columns (K-major rows of WqP), outlier rows = 0.
// grid.x covers ldq in chunks of 2048 (8 consecutive k per thread: 8
// independent strided loads in flight), grid.y strides over the patches.
__global__ void __launch_bounds__(256) patch_quantize_kernel(
    const __half* __restrict__ w, int64_t K, int64_t ldw, const uint32_t* __restrict__ mask,
    const int32_t* __restrict__ p_count, const int32_t* __restrict__ p_idx,
    const float* __restrict__ p_amax, const int32_t* __restrict__ p_src,
    const int8_t* __restrict__ q2, int8_t* __restrict__ wq_p, int64_t ldq) {
    pdl_wait();
    pdl_trigger();
    const int32_t np = *p_count;
    const int64_t k0 = static_cast<int64_t>(blockIdx.x) * 2048 + threadIdx.x * 8;
    if (k0 >= ldq) return;
    for (int32_t p = blockIdx.y; p < np; p += gridDim.y)
        patch_chunk(w, K, ldw, mask, p_idx, p_amax, p_src, q2, wq_p, ldq, p, k0);
}

// amax over all rows but the top-1 (candidate 1; 0 when K < 2): the scale of
// the q2 codes a column needs when its top-1 row is an outlier
__global__ void second_amax_kernel(int64_t N, const uint16_t* __restrict__ cand_v,
                                   const int32_t* __restrict__ cand_r, float* __restrict__ out) {
    const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= N) return;
    out[j] = cand_r[N + j] >= 0 ? half_bits_to_float(cand_v[N + j]) : 0.0f;
}

// ------------------------------------------------------------------ launchers
static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

cudaError_t launch_col_amax(const __half* w, int64_t K, int64_t N, int64_t ldw,
                            const uint32_t* row_mask, float* col_amax, cudaStream_t st) {
    uint32_t* bits = reinterpret_cast<uint32_t*>(col_amax);
    zero_words_kernel<<<static_cast<unsigned>(imin64((N + 255) / 256, 1024)), 256, 0, st>>>(bits, N);
    count_launch();
    int64_t rpb;
    const bool vec = (N % 8 == 0) && (ldw % 8 == 0) && aligned16(w);
    if (vec) {
        const int64_t cb = ((N >> 3) + 127) / 128;
        // ~2 blocks per SM, each thread over many rows: 16x fewer row chunks than the
        // 16-per-SM split (each chunk costs one atomicMax per column; at 4096 x 4096
        // they serialised in the L2: 62 us for 32 MB)
        const int rb = grid_rows_chunk(K, cb, static_cast<int64_t>(num_sms()) * 2, &rpb);
        col_amax_vec_kernel<<<dim3(static_cast<unsigned>(cb), rb), 128, 0, st>>>(w, K, N, ldw, row_mask,
                                                                                   rpb, bits);
    } else {
        const int64_t cb = (N + 255) / 256;
        const int rb = grid_rows_chunk(K, cb, static_cast<int64_t>(num_sms()) * 16, &rpb);
        col_amax_scalar_kernel<<<dim3(static_cast<unsigned>(cb), rb), 256, 0, st>>>(w, K, N, ldw,
                                                                                      row_mask, rpb, bits);
    }
    count_launch();
    amax_bits_to_float_kernel<<<static_cast<unsigned>(imin64((N + 255) / 256, 1024)), 256, 0, st>>>(bits, N);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_quantize_cols_t(const __half* w, int64_t K, int64_t N, int64_t ldw,
                                   const uint32_t* row_mask, int8_t* wq_t, int64_t ldq,
                                   float* col_amax, cudaStream_t st) {
    if (N == 0) return cudaSuccess;
    cudaError_t e = launch_col_amax(w, K, N, ldw, row_mask, col_amax, st);
    if (e != cudaSuccess) return e;
    const int vec = (ldw % 8 == 0) && aligned16(w);
    const int64_t kt = (ldq + 63) / 64;  // cover the padding columns too (written as 0)
    quantize_cols_t_kernel<<<dim3(static_cast<unsigned>((N + 63) / 64), static_cast<unsigned>(kt)),
                             256, 0, st>>>(w, K, N, ldw, row_mask, col_amax, wq_t, ldq, vec);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_gather_rows(const __half* w, int64_t ldw, int64_t N, const int32_t* idx,
                               const int32_t* count, int64_t cap, __half* out, int64_t ldo,
                               cudaStream_t st) {
    if (cap <= 0 || N == 0) return cudaSuccess;
    const int vec = (N % 8 == 0) && (ldw % 8 == 0) && (ldo % 8 == 0) && aligned16(w) && aligned16(out);
    const int64_t per = vec ? (N >> 3) : N;
    const unsigned gx = static_cast<unsigned>(imin64((per + 255) / 256, 64));
    cudaError_t e = launch_pdl(gather_rows_kernel, dim3(gx, static_cast<unsigned>(cap)), dim3(256), 0, st,
                               w, ldw, N, idx, count, cap, out, ldo, vec);
    count_launch();
    return e != cudaSuccess ? e : cudaGetLastError();
}

int64_t fixup_zero_words(int64_t N) { return 4 + (N + 31) / 32; }

cudaError_t launch_gather_fixup(const __half* w, int64_t K, int64_t N, int64_t ldw,
                                const uint32_t* mask, const int32_t* o_idx, const int32_t* o_count,
                                int64_t o_cap, __half* wo, int64_t ldwo, const float* amax_full,
                                const uint16_t* cand_v, const int32_t* cand_r, int32_t* p_count,
                                int32_t* p_idx, float* p_amax, int32_t* p_src, cudaStream_t st) {
    if (N == 0) return cudaSuccess;
    const int vec = (N % 8 == 0) && (ldw % 8 == 0) && (ldwo % 8 == 0) && aligned16(w) && aligned16(wo);
    const int64_t per = vec ? (N >> 3) : N;
    const int64_t gx = imin64((per + 255) / 256, 16);
    const int64_t blocks = o_cap * gx + (N + 255) / 256;
    cudaError_t e = launch_pdl(gather_fixup_kernel, dim3(static_cast<unsigned>(blocks)), dim3(256), 0, st,
                               w, K, N, ldw, mask, o_idx, o_count, o_cap, wo, ldwo, vec, gx, amax_full,
                               cand_v, cand_r, p_count, p_idx, p_amax, p_src);
    count_launch();
    return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_patch_quantize(const __half* w, int64_t K, int64_t N, int64_t ldw,
                                  const uint32_t* mask, const int8_t* q2, const int32_t* p_count,
                                  const int32_t* p_idx, const float* p_amax, const int32_t* p_src,
                                  int8_t* wq_p, int64_t ldq, cudaStream_t st) {
    const dim3 pgrid(static_cast<unsigned>((ldq + 2047) / 2048), static_cast<unsigned>(imin64(N, 256)));
    cudaError_t e = launch_pdl(patch_quantize_kernel, pgrid, dim3(256), 0, st, w, K, ldw, mask, p_count,
                               p_idx, p_amax, p_src, q2, wq_p, ldq);
    count_launch();
    return e != cudaSuccess ? e : cudaGetLastError();
}

int64_t topt_chunk_rows(int64_t K) { return K < 512 ? (K > 0 ? K : 1) : 512; }

cudaError_t launch_weight_prepare(const __half* w, int64_t K, int64_t N, int64_t ldw, int8_t* wq_t,
                                  int8_t* q2, int64_t ldq, float* col_amax, uint16_t* cand_v,
                                  int32_t* cand_r, uint32_t* scratch_v, int32_t* scratch_r,
                                  cudaStream_t st) {
    cudaError_t e = launch_quantize_cols_t(w, K, N, ldw, nullptr, wq_t, ldq, col_amax, st);
    if (e != cudaSuccess) return e;
    const int64_t rpb = topt_chunk_rows(K);
    const int64_t chunks = (K + rpb - 1) / rpb;
    const int64_t cb = ((N + 1) / 2 + 127) / 128;
    topt_partial_kernel<<<dim3(static_cast<unsigned>(cb), static_cast<unsigned>(chunks)), 128, 0, st>>>(
        w, K, N, ldw, rpb, scratch_v, scratch_r);
    count_launch();
    topt_merge_kernel<<<static_cast<unsigned>((N + 127) / 128), 128, 0, st>>>(N, chunks, scratch_v,
                                                                              scratch_r, cand_v, cand_r);
    count_launch();
    // q2: codes under the second candidate's amax (scratch_v reused as float[N])
    float* amax2 = reinterpret_cast<float*>(scratch_v);
    second_amax_kernel<<<static_cast<unsigned>((N + 255) / 256), 256, 0, st>>>(N, cand_v, cand_r, amax2);
    count_launch();
    const int vec = (ldw % 8 == 0) && aligned16(w);
    const int64_t kt = (ldq + 63) / 64;
    quantize_cols_t_kernel<<<dim3(static_cast<unsigned>((N + 63) / 64), static_cast<unsigned>(kt)),
                             256, 0, st>>>(w, K, N, ldw, nullptr, amax2, q2, ldq, vec);
    count_launch();
    return cudaGetLastError();
}


}  // namespace i8mm
