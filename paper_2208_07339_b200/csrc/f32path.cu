// float32-operand path of the reference API (SURVEY.md 8a a1-a13 at the
// reference's own container type).
//
// The reference's DenseMatrix stores float32 (pkg/src/int8mm/tensors.py:31-49):
// any finite f32 value, not only fp16-representable ones. The production
// kernels (prologue.cu, weights.cu, gemm_sm100.cu) consume fp16 operands; for
// f32 operands the operators first run f32_scan (outlier mask, non-finite and
// fp16-exactness flags, optional fp16 copy). When every value is exactly an
// fp16 value the fp16 kernels run on the copy (bit-identical results). When
// not, this file's kernels reproduce the reference on the f32 values:
//
//   f32_scan         gemm.py:208-210 (|x| >= f32(alpha), float32 compare) and
//                    tensors.py:47-48 (NaN/Inf flag)
//   f32_rowq         quantize.py:168-179 on x[:, keep] (gemm.py:242)
//   f32_colq_t       quantize.py:168-171, 182-187 on w[keep, :] (gemm.py:243),
//                    written K-major for the tcgen05 GEMM
//   f32_combine      gemm.py:130-147 (row x col dequant), 110-117 (ordered f64
//                    outlier term over the sorted O), 239-247 (sum, f32 cast)
//   ordered_mm       gemm.py:110-117 ordered_matmul_f64
//   rha              quantize.py:26-29 round_half_away
//   dequant_codes    quantize.py:214-227 dequantize
//   check_codes      tensors.py:95-98 (code -128 rejected)
//
// Every float64 operation is one explicit IEEE round-to-nearest op
// (__dmul_rn / __dadd_rn / __ddiv_rn), so nvcc cannot contract into FMA.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "../../include/llmint8.h"
#include "kernels.cuh"
#include "quant_common.cuh"

namespace i8mm {
namespace f32p {

constexpr int32_t FLAG_NONFINITE = 1;
constexpr int32_t FLAG_NOT_F16 = 2;
constexpr int32_t FLAG_CODE_128 = 4;

__device__ __forceinline__ bool masked(const uint32_t* mask, int64_t k) {
    return mask != nullptr && ((mask[k >> 5] >> (k & 31)) & 1u);
}

// One row per block iteration; lanes of a warp cover 32 consecutive columns so
// a ballot is one whole mask word.
__global__ void __launch_bounds__(256) f32_scan_kernel(const float* __restrict__ x, int64_t rows,
                                                       int64_t cols, int64_t ld, float alpha,
                                                       uint32_t* __restrict__ mask,
                                                       int32_t* __restrict__ flags,
                                                       __half* __restrict__ y16, int64_t ldy) {
    const int lane = threadIdx.x & 31;
    int32_t f = 0;
    const int64_t cols_pad = (cols + 31) / 32 * 32;
    for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
        for (int64_t c = threadIdx.x; c < cols_pad; c += blockDim.x) {
            const bool in = c < cols;
            const float v = in ? x[r * ld + c] : 0.0f;
            const float a = fabsf(v);
            if (in) {
                if (!(a <= 3.402823466e38f)) f |= FLAG_NONFINITE;  // NaN or Inf
                const __half h = __float2half_rn(v);
                if (__half2float(h) != v) f |= FLAG_NOT_F16;
                if (y16 != nullptr) y16[r * ldy + c] = h;
            }
            if (mask != nullptr) {
                const uint32_t bits = __ballot_sync(0xffffffffu, in && a >= alpha);
                if (lane == 0 && bits) atomicOr(mask + (c >> 5), bits);
            }
        }
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) f |= __shfl_xor_sync(0xffffffffu, f, d);
    if (lane == 0 && f) atomicOr(flags, f);
}

__device__ __forceinline__ float block_max(float v, float* red) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, d));
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    float m = 0.0f;
    for (int i = 0; i < static_cast<int>(blockDim.x >> 5); ++i) m = fmaxf(m, red[i]);
    return m;
}

// quantize.py:168-179 per row over the keep columns; codes at outlier columns
// and in the ldq padding are 0 (the GEMM runs over the full K).
__global__ void __launch_bounds__(256) f32_rowq_kernel(const float* __restrict__ x, int64_t M,
                                                       int64_t K, int64_t ldx,
                                                       const uint32_t* __restrict__ mask,
                                                       int8_t* __restrict__ xq, int64_t ldq,
                                                       float* __restrict__ amax_out) {
    __shared__ float red[8];
    for (int64_t r = blockIdx.x; r < M; r += gridDim.x) {
        const float* row = x + r * ldx;
        float m = 0.0f;
        for (int64_t c = threadIdx.x; c < K; c += blockDim.x)
            if (!masked(mask, c)) m = fmaxf(m, fabsf(row[c]));
        const float amax = block_max(m, red);
        const double s = scale_of(amax);
        const float s32 = static_cast<float>(s);
        for (int64_t c = threadIdx.x; c < ldq; c += blockDim.x) {
            int code = 0;
            if (c < K && !masked(mask, c)) code = code_fast(row[c], s32, s);
            xq[r * ldq + c] = static_cast<int8_t>(code);
        }
        if (threadIdx.x == 0) amax_out[r] = amax;
    }
}

// quantize.py:182-187 per column over the keep rows, stored transposed
// (N x ldq, K-major) through a 32 x 32 shared-memory tile.
__global__ void __launch_bounds__(256) f32_colq_t_kernel(const float* __restrict__ w, int64_t K,
                                                         int64_t N, int64_t ldw,
                                                         const uint32_t* __restrict__ mask,
                                                         int8_t* __restrict__ wq_t, int64_t ldq,
                                                         float* __restrict__ amax_out) {
    __shared__ float part[8][32];
    __shared__ float s_amax[32];
    __shared__ int8_t tile[32][33];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int64_t c0 = static_cast<int64_t>(blockIdx.x) * 32;
    const int64_t c = c0 + tx;
    float m = 0.0f;
    if (c < N)
        for (int64_t k = ty; k < K; k += 8)
            if (!masked(mask, k)) m = fmaxf(m, fabsf(w[k * ldw + c]));
    part[ty][tx] = m;
    __syncthreads();
    if (ty == 0) {
        float a = part[0][tx];
        for (int i = 1; i < 8; ++i) a = fmaxf(a, part[i][tx]);
        s_amax[tx] = a;
        if (c < N) amax_out[c] = a;
    }
    __syncthreads();
    const double s = scale_of(s_amax[tx]);
    const float s32 = static_cast<float>(s);
    for (int64_t k0 = 0; k0 < ldq; k0 += 32) {
        for (int i = ty; i < 32; i += 8) {
            const int64_t k = k0 + i;
            int code = 0;
            if (c < N && k < K && !masked(mask, k)) code = code_fast(w[k * ldw + c], s32, s);
            tile[i][tx] = static_cast<int8_t>(code);
        }
        __syncthreads();
        for (int i = ty; i < 32; i += 8) {
            const int64_t orow = c0 + i, ocol = k0 + tx;
            if (orow < N && ocol < ldq) wq_t[orow * ldq + ocol] = tile[tx][i];
        }
        __syncthreads();
    }
}

// gemm.py:239-247: out = f32(f64(lo) + hi) with lo = f32(f64(C) / (sx * sw))
// (gemm.py:141) and hi = sum over the ascending O of f64(x) * f64(w)
// (gemm.py:110-117); no keep columns -> out = f32(hi); O empty -> out = lo.
__global__ void __launch_bounds__(256) f32_combine_kernel(
    const int32_t* __restrict__ c, int64_t ldc, const float* __restrict__ ramax,
    const float* __restrict__ camax, const float* __restrict__ x, int64_t ldx,
    const float* __restrict__ w, int64_t ldw, const int32_t* __restrict__ o_idx,
    const int32_t* __restrict__ o_count, int64_t K, int64_t M, int64_t N, float* __restrict__ y,
    int64_t ldy) {
    const int n_out = *o_count;
    const bool keep_any = n_out < K;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < M * N;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = i / N, col = i % N;
        double lo = 0.0;
        if (keep_any) {
            const double d = __dmul_rn(scale_of(ramax[r]), scale_of(camax[col]));
            lo = static_cast<double>(
                __double2float_rn(__ddiv_rn(static_cast<double>(c[r * ldc + col]), d)));
        }
        if (n_out == 0) {
            y[r * ldy + col] = static_cast<float>(lo);
            continue;
        }
        double hi = 0.0;
        for (int o = 0; o < n_out; ++o) {
            const int64_t k = o_idx[o];
            hi = __dadd_rn(hi, __dmul_rn(static_cast<double>(x[r * ldx + k]),
                                         static_cast<double>(w[k * ldw + col])));
        }
        y[r * ldy + col] = __double2float_rn(keep_any ? __dadd_rn(lo, hi) : hi);
    }
}

template <typename T>
__global__ void __launch_bounds__(256) ordered_mm_kernel(const T* __restrict__ x, int64_t ldx,
                                                         const T* __restrict__ w, int64_t ldw,
                                                         int64_t M, int64_t K, int64_t N,
                                                         double* __restrict__ out, int64_t ldo) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < M * N;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = i / N, col = i % N;
        double acc = 0.0;  // np.zeros, then acc += outer(x[:, k], w[k, :]) for k ascending
        for (int64_t k = 0; k < K; ++k)
            acc = __dadd_rn(acc, __dmul_rn(static_cast<double>(x[r * ldx + k]),
                                           static_cast<double>(w[k * ldw + col])));
        out[r * ldo + col] = acc;
    }
}

template <typename T>
__global__ void rha_kernel(const T* __restrict__ src, int64_t n, double* __restrict__ dst) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double v = static_cast<double>(src[i]);
        dst[i] = copysign(floor(__dadd_rn(fabs(v), 0.5)), v);
    }
}

// quantize.py:214-227
__global__ void dequant_codes_kernel(const int8_t* __restrict__ q, int64_t rows, int64_t cols,
                                     int64_t ldq, int mode, const double* __restrict__ s_row,
                                     const double* __restrict__ s_col, double scale, int32_t zp,
                                     double nd, double offset, float* __restrict__ out,
                                     int64_t ldo) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < rows * cols;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = i / cols, c = i % cols;
        const double v = static_cast<double>(q[r * ldq + c]);
        double o;
        switch (mode) {
            case I8MM_DEQ_ABSMAX: o = __ddiv_rn(v, scale); break;
            case I8MM_DEQ_ZEROPOINT:
                o = __dadd_rn(__ddiv_rn(__dadd_rn(v, static_cast<double>(zp)), nd), offset);
                break;
            case I8MM_DEQ_ROWWISE: o = __ddiv_rn(v, s_row[r]); break;
            default: o = __ddiv_rn(v, s_col[c]); break;
        }
        out[r * ldo + c] = __double2float_rn(o);
    }
}

__global__ void check_codes_kernel(const int8_t* __restrict__ q, int64_t rows, int64_t cols,
                                   int64_t ldq, int32_t* __restrict__ flags) {
    int32_t f = 0;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < rows * cols;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = i / cols, c = i % cols;
        if (q[r * ldq + c] == -128) f = FLAG_CODE_128;
    }
    f = __reduce_or_sync(0xffffffffu, static_cast<unsigned>(f));
    if ((threadIdx.x & 31) == 0 && f) atomicOr(flags, f);
}

static unsigned grid_for(int64_t n, int64_t per = 256) {
    int64_t b = (n + per - 1) / per;
    const int64_t cap = static_cast<int64_t>(num_sms()) * 16;
    if (b > cap) b = cap;
    if (b < 1) b = 1;
    return static_cast<unsigned>(b);
}
static unsigned grid_rows(int64_t rows) {
    const int64_t cap = static_cast<int64_t>(num_sms()) * 8;
    return static_cast<unsigned>(rows < 1 ? 1 : (rows < cap ? rows : cap));
}

}  // namespace f32p
}  // namespace i8mm

using namespace i8mm;
using namespace i8mm::f32p;

static int st_ok(cudaError_t e) { return e == cudaSuccess ? I8MM_OK : I8MM_ERR_CUDA; }

extern "C" {

int i8mm_f32_scan(const float* x, int64_t rows, int64_t cols, int64_t ld, float alpha,
                  uint32_t* col_mask, int32_t* flags, void* y16, int64_t ldy, void* stream) {
    if (int s = check_device()) return s;
    if (rows < 0 || cols < 0 || ld < cols || !flags || (rows > 0 && !x)) return I8MM_ERR_ARGUMENT;
    if (col_mask && (!(alpha > 0.0f) || !std::isfinite(alpha))) return I8MM_ERR_ALPHA;
    if (y16 && ldy < cols) return I8MM_ERR_ARGUMENT;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (col_mask && cudaMemsetAsync(col_mask, 0, sizeof(uint32_t) * ((cols + 31) / 32), st) != cudaSuccess)
        return I8MM_ERR_CUDA;
    if (rows == 0 || cols == 0) return I8MM_OK;
    f32_scan_kernel<<<grid_rows(rows), 256, 0, st>>>(x, rows, cols, ld, alpha, col_mask, flags,
                                                     static_cast<__half*>(y16), ldy);
    count_launch();
    return st_ok(cudaGetLastError());
}

int i8mm_f32_quantize_rows(const float* x, int64_t M, int64_t K, int64_t ldx, const uint32_t* col_mask,
                           int8_t* xq, int64_t ldq, float* row_amax, void* stream) {
    if (int s = check_device()) return s;
    if (M < 0 || K < 0 || ldx < K || ldq < K || (M > 0 && (!x || !xq || !row_amax))) return I8MM_ERR_ARGUMENT;
    if (M == 0) return I8MM_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    f32_rowq_kernel<<<grid_rows(M), 256, 0, st>>>(x, M, K, ldx, col_mask, xq, ldq, row_amax);
    count_launch();
    return st_ok(cudaGetLastError());
}

int i8mm_f32_quantize_cols_t(const float* w, int64_t K, int64_t N, int64_t ldw, const uint32_t* row_mask,
                             int8_t* wq_t, int64_t ldq, float* col_amax, void* stream) {
    if (int s = check_device()) return s;
    if (K < 0 || N < 0 || ldw < N || ldq < K || (N > 0 && (!w || !wq_t || !col_amax))) return I8MM_ERR_ARGUMENT;
    if (N == 0) return I8MM_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    f32_colq_t_kernel<<<static_cast<unsigned>((N + 31) / 32), 256, 0, st>>>(w, K, N, ldw, row_mask, wq_t, ldq,
                                                                           col_amax);
    count_launch();
    return st_ok(cudaGetLastError());
}

int i8mm_f32_llm_int8_combine(const int32_t* c, int64_t ldc, int64_t M, int64_t N, int64_t K,
                              const float* row_amax, const float* col_amax, const float* x, int64_t ldx,
                              const float* w, int64_t ldw, const int32_t* o_idx, const int32_t* o_count,
                              float* y, int64_t ldy, void* stream) {
    if (int s = check_device()) return s;
    if (M < 0 || N < 0 || ldc < N || ldy < N || ldx < K || ldw < N || !o_count || !o_idx)
        return I8MM_ERR_ARGUMENT;
    if (M == 0 || N == 0) return I8MM_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    f32_combine_kernel<<<grid_for(M * N), 256, 0, st>>>(c, ldc, row_amax, col_amax, x, ldx, w, ldw, o_idx,
                                                        o_count, K, M, N, y, ldy);
    count_launch();
    return st_ok(cudaGetLastError());
}

size_t i8mm_f32_workspace_size(int64_t M, int64_t K, int64_t N) {
    auto r = [](int64_t b) { return static_cast<size_t>((b + 255) / 256 * 256); };
    const int64_t ldq = (K + 15) / 16 * 16;
    return 256 + r(4 * ((K + 31) / 32)) + r(16) + r(4 * K) + r(M * ldq) + r(4 * M) + r(N * ldq) +
           r(4 * N) + r(4 * M * N);
}

int i8mm_llm_int8_matmul_f32(const float* x, int64_t ldx, const float* w, int64_t ldw, int64_t M,
                             int64_t K, int64_t N, float alpha, float* y, int64_t ldy, void* workspace,
                             size_t workspace_bytes, int32_t* status_out, void* stream) {
    if (int s = check_device()) return s;
    if (K > I8MM_MAX_INNER_DIM) return I8MM_ERR_OVERFLOW;
    if (!(alpha > 0.0f) || !std::isfinite(alpha)) return I8MM_ERR_ALPHA;
    if (M <= 0 || K <= 0 || N <= 0 || ldx < K || ldw < N || ldy < N || !x || !w || !y || !workspace ||
        !status_out)
        return I8MM_ERR_ARGUMENT;
    if (workspace_bytes < i8mm_f32_workspace_size(M, K, N)) return I8MM_ERR_ARGUMENT;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    uintptr_t p = (reinterpret_cast<uintptr_t>(workspace) + 255) & ~uintptr_t(255);
    auto take = [&](int64_t b) {
        uintptr_t r = p;
        p += static_cast<uintptr_t>((b + 255) / 256 * 256);
        return r;
    };
    const int64_t ldq = (K + 15) / 16 * 16;
    uint32_t* mask = reinterpret_cast<uint32_t*>(take(4 * ((K + 31) / 32)));
    int32_t* cnt = reinterpret_cast<int32_t*>(take(16));  // [o_count, flags]
    int32_t* o_idx = reinterpret_cast<int32_t*>(take(4 * K));
    int8_t* xq = reinterpret_cast<int8_t*>(take(M * ldq));
    float* ramax = reinterpret_cast<float*>(take(4 * M));
    int8_t* wq_t = reinterpret_cast<int8_t*>(take(N * ldq));
    float* camax = reinterpret_cast<float*>(take(4 * N));
    int32_t* c = reinterpret_cast<int32_t*>(take(4 * M * N));
    // status_out[0] receives |O|, status_out[1] the non-finite flag (device words)
    if (cudaMemsetAsync(status_out, 0, 8, st) != cudaSuccess) return I8MM_ERR_CUDA;
    if (int s = i8mm_f32_scan(x, M, K, ldx, alpha, mask, status_out + 1, nullptr, 0, stream)) return s;
    if (int s = i8mm_f32_scan(w, K, N, ldw, 0.0f, nullptr, status_out + 1, nullptr, 0, stream)) return s;
    if (cudaGetLastError() != cudaSuccess) return I8MM_ERR_CUDA;
    if (st_ok(launch_outlier_compact(mask, K, o_idx, cnt, st))) return I8MM_ERR_CUDA;
    if (int s = i8mm_f32_quantize_rows(x, M, K, ldx, mask, xq, ldq, ramax, stream)) return s;
    if (int s = i8mm_f32_quantize_cols_t(w, K, N, ldw, mask, wq_t, ldq, camax, stream)) return s;
    if (int s = i8mm_gemm_i32(xq, ldq, wq_t, ldq, c, N, M, N, K, stream)) return s;
    if (int s = i8mm_f32_llm_int8_combine(c, N, M, N, K, ramax, camax, x, ldx, w, ldw, o_idx, cnt, y, ldy,
                                          stream))
        return s;
    if (cudaMemcpyAsync(status_out, cnt, 4, cudaMemcpyDeviceToDevice, st) != cudaSuccess) return I8MM_ERR_CUDA;
    return I8MM_OK;
}

int i8mm_ordered_matmul_f64(const void* x, int64_t ldx, const void* w, int64_t ldw, int64_t M, int64_t K,
                            int64_t N, int elt_bytes, double* out, int64_t ldo, void* stream) {
    if (int s = check_device()) return s;
    if (M < 0 || K < 0 || N < 0 || ldx < K || ldw < N || ldo < N || (elt_bytes != 4 && elt_bytes != 8))
        return I8MM_ERR_ARGUMENT;
    if (M == 0 || N == 0) return I8MM_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (elt_bytes == 4)
        ordered_mm_kernel<float><<<grid_for(M * N), 256, 0, st>>>(static_cast<const float*>(x), ldx,
                                                                  static_cast<const float*>(w), ldw, M, K, N,
                                                                  out, ldo);
    else
        ordered_mm_kernel<double><<<grid_for(M * N), 256, 0, st>>>(static_cast<const double*>(x), ldx,
                                                                   static_cast<const double*>(w), ldw, M, K, N,
                                                                   out, ldo);
    count_launch();
    return st_ok(cudaGetLastError());
}

int i8mm_round_half_away(const void* src, int64_t n, int elt_bytes, double* dst, void* stream) {
    if (int s = check_device()) return s;
    if (n < 0 || (elt_bytes != 4 && elt_bytes != 8) || (n > 0 && (!src || !dst))) return I8MM_ERR_ARGUMENT;
    if (n == 0) return I8MM_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (elt_bytes == 4)
        rha_kernel<float><<<grid_for(n), 256, 0, st>>>(static_cast<const float*>(src), n, dst);
    else
        rha_kernel<double><<<grid_for(n), 256, 0, st>>>(static_cast<const double*>(src), n, dst);
    count_launch();
    return st_ok(cudaGetLastError());
}

int i8mm_dequantize_codes(const int8_t* q, int64_t rows, int64_t cols, int64_t ldq, int mode,
                          const double* s_row, const double* s_col, double scale, int32_t zp, double nd,
                          double offset, float* out, int64_t ldo, void* stream) {
    if (int s = check_device()) return s;
    if (rows < 0 || cols < 0 || ldq < cols || ldo < cols || !q || !out) return I8MM_ERR_ARGUMENT;
    if ((mode == I8MM_DEQ_ROWWISE && !s_row) || (mode == I8MM_DEQ_COLWISE && !s_col) || mode < 0 || mode > 3)
        return I8MM_ERR_ARGUMENT;
    if (rows == 0 || cols == 0) return I8MM_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    dequant_codes_kernel<<<grid_for(rows * cols), 256, 0, st>>>(q, rows, cols, ldq, mode, s_row, s_col, scale,
                                                                zp, nd, offset, out, ldo);
    count_launch();
    return st_ok(cudaGetLastError());
}

int i8mm_check_codes(const int8_t* q, int64_t rows, int64_t cols, int64_t ldq, int32_t* flags, void* stream) {
    if (int s = check_device()) return s;
    if (rows < 0 || cols < 0 || ldq < cols || !flags || (rows * cols > 0 && !q)) return I8MM_ERR_ARGUMENT;
    if (rows == 0 || cols == 0) return I8MM_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    check_codes_kernel<<<grid_for(rows * cols), 256, 0, st>>>(q, rows, cols, ldq, flags);
    count_launch();
    return st_ok(cudaGetLastError());
}

}  // extern "C"

namespace i8mm {
namespace f32p {
__global__ void f16_check_kernel(const __half* __restrict__ x, int64_t rows, int64_t cols, int64_t ld,
                                 int32_t* __restrict__ flags) {
    unsigned f = 0;
    for (int64_t r = blockIdx.x; r < rows; r += gridDim.x)
        for (int64_t c = threadIdx.x; c < cols; c += blockDim.x)
            if ((__half_as_ushort(x[r * ld + c]) & 0x7C00u) == 0x7C00u) f = FLAG_NONFINITE;
    f = __reduce_or_sync(0xffffffffu, f);
    if ((threadIdx.x & 31) == 0 && f) atomicOr(flags, static_cast<int32_t>(f));
}
__global__ void f16_to_f32_kernel(const __half* __restrict__ x, int64_t rows, int64_t cols, int64_t ld,
                                  float* __restrict__ y, int64_t ldy) {
    for (int64_t r = blockIdx.x; r < rows; r += gridDim.x)
        for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) y[r * ldy + c] = __half2float(x[r * ld + c]);
}
}  // namespace f32p
}  // namespace i8mm

extern "C" {
int i8mm_f16_check(const void* x, int64_t rows, int64_t cols, int64_t ld, int32_t* flags, void* stream) {
    if (int s = check_device()) return s;
    if (rows < 0 || cols < 0 || ld < cols || !flags || (rows * cols > 0 && !x)) return I8MM_ERR_ARGUMENT;
    if (rows == 0 || cols == 0) return I8MM_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    f16_check_kernel<<<grid_rows(rows), 256, 0, st>>>(static_cast<const __half*>(x), rows, cols, ld, flags);
    count_launch();
    return st_ok(cudaGetLastError());
}
int i8mm_f16_to_f32(const void* x, int64_t rows, int64_t cols, int64_t ld, float* y, int64_t ldy, void* stream) {
    if (int s = check_device()) return s;
    if (rows < 0 || cols < 0 || ld < cols || ldy < cols || (rows * cols > 0 && (!x || !y))) return I8MM_ERR_ARGUMENT;
    if (rows == 0 || cols == 0) return I8MM_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    f16_to_f32_kernel<<<grid_rows(rows), 256, 0, st>>>(static_cast<const __half*>(x), rows, cols, ld, y, ldy);
    count_launch();
    return st_ok(cudaGetLastError());
}
int i8mm_zero(void* p, size_t bytes, void* stream) {
    if (bytes == 0) return I8MM_OK;
    if (!p) return I8MM_ERR_ARGUMENT;
    return st_ok(cudaMemsetAsync(p, 0, bytes, static_cast<cudaStream_t>(stream)));
}
}  // extern "C"
