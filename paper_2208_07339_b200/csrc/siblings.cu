// Sibling quantization pipelines of the reference's backend plugin point
// (SURVEY.md 8f rank 4): tensor-wise absmax and zeropoint quantization and
// their matmuls (pkg/src/int8mm/quantize.py:120-165, gemm.py:85-104, 150-187).
// The int8 x int8 product runs on the same tcgen05 GEMM as the LLM.int8() path
// (EPI_I32); these kernels are the HBM-bound quantizers, reductions and the
// exact float64 epilogues around it.
//
// Bit-exactness with the reference:
//   absmax   codes = clip(rha(fl64(127/amax * x)), +-127); an all-zero tensor
//            has scale 1 and zero codes (quantize.py:137-151)
//   zeropoint stored = clip(rha(fl64(nd * x)) - zp, +-127) with nd, zp computed
//            on the host exactly as numpy does (quantize.py:153-171)
//   matmul   C = A@B exact int32 on the tensor cores; the zeropoint shift is
//            the unrolled integer identity (gemm.py:98-104) in int64, range-
//            checked like gemm.py:71-75; f32(f64(acc) / (s_x * s_w)) epilogues
//            (gemm.py:133, 135, 175-187) with every f64 op a single IEEE op.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>

#include "kernels.cuh"
#include "quant_common.cuh"

namespace i8mm {

// ------------------------------------------------------------------ reductions
// stats[0] = max |x| (fp16 bits), stats[1] = ordered-int min, stats[2] = ordered-int max
__device__ __forceinline__ int f32_ordered(float f) {
    const int i = __float_as_int(f);
    return i >= 0 ? i : i ^ 0x7FFFFFFF;
}
__device__ __forceinline__ float ordered_f32(int o) { return __int_as_float(o >= 0 ? o : o ^ 0x7FFFFFFF); }

__global__ void stats_init_kernel(int32_t* stats) {
    stats[0] = 0;
    stats[1] = INT_MAX;
    stats[2] = INT_MIN;
}

// Element access for fp16 and float32 operands (the reference's DenseMatrix
// is float32, tensors.py:31-49): value as float, |x| as order-preserving bits.
template <typename T> struct Elt;
template <> struct Elt<__half> {
    static __device__ __forceinline__ float f(__half h) { return __half2float(h); }
    static __device__ __forceinline__ uint32_t abits(__half h) { return __half_as_ushort(h) & 0x7FFFu; }
    static __device__ __forceinline__ float from_abits(uint32_t b) {
        return __half2float(__ushort_as_half(static_cast<unsigned short>(b)));
    }
};
template <> struct Elt<float> {
    static __device__ __forceinline__ float f(float v) { return v; }
    static __device__ __forceinline__ uint32_t abits(float v) { return __float_as_uint(v) & 0x7FFFFFFFu; }
    static __device__ __forceinline__ float from_abits(uint32_t b) { return __uint_as_float(b); }
};

template <typename T>
__global__ void __launch_bounds__(256) tensor_stats_kernel(const T* __restrict__ x, int64_t rows,
                                                           int64_t cols, int64_t ld,
                                                           int32_t* __restrict__ stats) {
    uint32_t amax = 0;
    int mn = INT_MAX, mx = INT_MIN;
    const int64_t n = rows * cols;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = i / cols, c = i % cols;
        const T h = x[r * ld + c];
        amax = max(amax, Elt<T>::abits(h));
        const int o = f32_ordered(Elt<T>::f(h));
        mn = min(mn, o);
        mx = max(mx, o);
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        amax = max(amax, __shfl_xor_sync(0xffffffffu, amax, d));
        mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, d));
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, d));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(reinterpret_cast<uint32_t*>(stats), amax);
        atomicMin(stats + 1, mn);
        atomicMax(stats + 2, mx);
    }
}

// stats -> floats: out[0] = amax, out[1] = min, out[2] = max
template <typename T>
__global__ void stats_finish_kernel(const int32_t* stats, float* out) {
    out[0] = Elt<T>::from_abits(static_cast<uint32_t>(stats[0]));
    out[1] = ordered_f32(stats[1]);
    out[2] = ordered_f32(stats[2]);
    out[3] = 0.0f;  // the host reads the 4-float record whole
}

// ------------------------------------------------------------------ quantizers
// 32 x 32 tiles through shared memory; TRANSPOSE writes the K-major layout the
// tensor-core GEMM reads for B (out[c][r]); the ld_out padding is written 0.
enum ScalarMode : int { MODE_ABSMAX = 0, MODE_ZEROPOINT = 1 };

template <int MODE>
__device__ __forceinline__ int scalar_code(float x, const float* amax_dev, double nd, int32_t zp) {
    if constexpr (MODE == MODE_ABSMAX) {
        const float amax = *amax_dev;
        if (amax == 0.0f) return 0;  // quantize.py:144-147: scale 1, all-zero codes
        const double s = 127.0 / static_cast<double>(amax);
        return code_fast(x, static_cast<float>(s), s);
    } else {
        // quantize.py:167: clip(rha(nd * data) - zp, -127, 127)
        const double p = __dmul_rn(nd, static_cast<double>(x));
        const double r = copysign(floor(__dadd_rn(fabs(p), 0.5)), p);
        double v = __dadd_rn(r, -static_cast<double>(zp));
        v = fmin(fmax(v, -127.0), 127.0);
        return static_cast<int>(v);
    }
}

template <typename T, int MODE, bool TRANSPOSE>
__global__ void __launch_bounds__(256) quantize_scalar_kernel(
    const T* __restrict__ x, int64_t rows, int64_t cols, int64_t ld, const float* amax_dev,
    double nd, int32_t zp, int8_t* __restrict__ out, int64_t ld_out, int64_t out_rows,
    int64_t out_cols) {
    __shared__ int8_t tile[32][33];
    const int64_t r0 = static_cast<int64_t>(blockIdx.y) * 32, c0 = static_cast<int64_t>(blockIdx.x) * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
    if constexpr (!TRANSPOSE) {
        for (int i = ty; i < 32; i += 8) {
            const int64_t r = r0 + i, c = c0 + tx;
            if (r < out_rows && c < out_cols)
                out[r * ld_out + c] = (r < rows && c < cols)
                                          ? static_cast<int8_t>(scalar_code<MODE>(Elt<T>::f(x[r * ld + c]), amax_dev, nd, zp))
                                          : int8_t(0);
        }
    } else {
        // input tile rows r0.. (K), cols c0.. (N); output row = input col
        for (int i = ty; i < 32; i += 8) {
            const int64_t r = r0 + i, c = c0 + tx;
            tile[i][tx] = (r < rows && c < cols)
                              ? static_cast<int8_t>(scalar_code<MODE>(Elt<T>::f(x[r * ld + c]), amax_dev, nd, zp))
                              : int8_t(0);
        }
        __syncthreads();
        for (int i = ty; i < 32; i += 8) {
            const int64_t orow = c0 + i, ocol = r0 + tx;
            if (orow < out_rows && ocol < out_cols) out[orow * ld_out + ocol] = tile[tx][i];
        }
    }
}

// sum of each int8 row (warp per row)
__global__ void rowsum_i8_kernel(const int8_t* __restrict__ q, int64_t rows, int64_t cols, int64_t ld,
                                 int32_t* __restrict__ out) {
    const int64_t row = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= rows) return;
    int32_t s = 0;
    for (int64_t c = lane; c < cols; c += 32) s += q[row * ld + c];
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) s += __shfl_xor_sync(0xffffffffu, s, d);
    if (lane == 0) out[row] = s;
}

// ------------------------------------------------------------------ epilogues
// absmax: f32(f64(c) / (s_x * s_w)) with s = 127/amax (amax 0 -> 1) (gemm.py:133)
__global__ void dequant_absmax_kernel(const int32_t* __restrict__ c, int64_t M, int64_t N, int64_t ldc,
                                      const float* amax_x, const float* amax_w, float* __restrict__ out,
                                      int64_t ldo) {
    const float ax = *amax_x, aw = *amax_w;
    const double sx = ax == 0.0f ? 1.0 : 127.0 / static_cast<double>(ax);
    const double sw = aw == 0.0f ? 1.0 : 127.0 / static_cast<double>(aw);
    const double d = __dmul_rn(sx, sw);
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < M * N;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = i / N, col = i % N;
        out[r * ldo + col] = __double2float_rn(__ddiv_rn(static_cast<double>(c[r * ldc + col]), d));
    }
}

// zeropoint (gemm.py:98-104 unrolled, 71-75 range check, 175-187 dequant + offsets)
__global__ void zeropoint_combine_kernel(const int32_t* __restrict__ c, int64_t M, int64_t N,
                                         int64_t ldc, const int32_t* __restrict__ rowsum_a,
                                         const int32_t* __restrict__ colsum_b, int64_t K, int32_t zp_a,
                                         int32_t zp_b, double nd_a, double nd_b, double off_a,
                                         double off_b, float* __restrict__ out, int64_t ldo,
                                         int32_t* __restrict__ acc_out, int32_t* overflow) {
    const double nd = __dmul_rn(nd_a, nd_b);
    const bool offs = off_a != 0.0 || off_b != 0.0;
    const double fa = offs ? __ddiv_rn(off_b, nd_a) : 0.0;  // (pw.offset / px.nd)
    const double fb = offs ? __ddiv_rn(off_a, nd_b) : 0.0;  // (px.offset / pw.nd)
    const double fc = offs ? __dmul_rn(__dmul_rn(off_a, off_b), static_cast<double>(K)) : 0.0;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < M * N;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = i / N, col = i % N;
        const int64_t acc = static_cast<int64_t>(c[r * ldc + col]) +
                            static_cast<int64_t>(zp_b) * rowsum_a[r] +
                            static_cast<int64_t>(zp_a) * colsum_b[col] +
                            K * static_cast<int64_t>(zp_a) * static_cast<int64_t>(zp_b);
        if (acc < INT_MIN || acc > INT_MAX) {
            atomicOr(overflow, 1);
            continue;
        }
        if (acc_out != nullptr) acc_out[r * N + col] = static_cast<int32_t>(acc);
        if (out == nullptr) continue;
        double v = __ddiv_rn(static_cast<double>(acc), nd);
        if (offs) {
            const int64_t ta = static_cast<int64_t>(rowsum_a[r]) + K * zp_a;
            const int64_t tb = static_cast<int64_t>(colsum_b[col]) + K * zp_b;
            v = __dadd_rn(v, __dmul_rn(fa, static_cast<double>(ta)));
            v = __dadd_rn(v, __dmul_rn(fb, static_cast<double>(tb)));
            v = __dadd_rn(v, fc);
        }
        out[r * ldo + col] = __double2float_rn(v);
    }
}

// ------------------------------------------------------------------ launchers
static unsigned blocks_for(int64_t n, int64_t per = 256, int64_t cap = 4096) {
    int64_t b = (n + per - 1) / per;
    if (b < 1) b = 1;
    if (b > cap) b = cap;
    return static_cast<unsigned>(b);
}

template <typename T>
static cudaError_t tensor_stats_t(const T* x, int64_t rows, int64_t cols, int64_t ld,
                                  int32_t* stats_scratch, float* out3, cudaStream_t st) {
    stats_init_kernel<<<1, 1, 0, st>>>(stats_scratch);
    count_launch();
    tensor_stats_kernel<T><<<blocks_for(rows * cols, 256, num_sms() * 8), 256, 0, st>>>(x, rows, cols, ld,
                                                                                    stats_scratch);
    count_launch();
    stats_finish_kernel<T><<<1, 1, 0, st>>>(stats_scratch, out3);
    count_launch();
    return cudaGetLastError();
}
cudaError_t launch_tensor_stats(const __half* x, int64_t rows, int64_t cols, int64_t ld,
                                int32_t* stats_scratch, float* out3, cudaStream_t st) {
    return tensor_stats_t(x, rows, cols, ld, stats_scratch, out3, st);
}
cudaError_t launch_tensor_stats(const float* x, int64_t rows, int64_t cols, int64_t ld,
                                int32_t* stats_scratch, float* out3, cudaStream_t st) {
    return tensor_stats_t(x, rows, cols, ld, stats_scratch, out3, st);
}

template <typename T>
static cudaError_t quantize_scalar_t(const T* x, int64_t rows, int64_t cols, int64_t ld, int mode,
                                     const float* amax_dev, double nd, int32_t zp, int8_t* out,
                                     int64_t ld_out, int transpose, cudaStream_t st) {
    // output covers [out_rows x ld_out] including the K..ld_out padding
    const int64_t out_rows = transpose ? cols : rows;
    const int64_t out_cols = ld_out;
    const int64_t in_r = transpose ? ld_out : rows;   // tile grid over the input (rows padded for T)
    const int64_t in_c = transpose ? cols : ld_out;
    const dim3 grid(static_cast<unsigned>((in_c + 31) / 32), static_cast<unsigned>((in_r + 31) / 32));
    if (mode == MODE_ABSMAX) {
        if (transpose)
            quantize_scalar_kernel<T, MODE_ABSMAX, true><<<grid, 256, 0, st>>>(x, rows, cols, ld, amax_dev, nd, zp,
                                                                             out, ld_out, out_rows, out_cols);
        else
            quantize_scalar_kernel<T, MODE_ABSMAX, false><<<grid, 256, 0, st>>>(x, rows, cols, ld, amax_dev, nd, zp,
                                                                              out, ld_out, out_rows, out_cols);
    } else {
        if (transpose)
            quantize_scalar_kernel<T, MODE_ZEROPOINT, true><<<grid, 256, 0, st>>>(x, rows, cols, ld, amax_dev, nd,
                                                                                zp, out, ld_out, out_rows,
                                                                                out_cols);
        else
            quantize_scalar_kernel<T, MODE_ZEROPOINT, false><<<grid, 256, 0, st>>>(x, rows, cols, ld, amax_dev, nd,
                                                                                 zp, out, ld_out, out_rows,
                                                                                 out_cols);
    }
    count_launch();
    return cudaGetLastError();
}
cudaError_t launch_quantize_scalar(const __half* x, int64_t rows, int64_t cols, int64_t ld, int mode,
                                   const float* amax_dev, double nd, int32_t zp, int8_t* out,
                                   int64_t ld_out, int transpose, cudaStream_t st) {
    return quantize_scalar_t(x, rows, cols, ld, mode, amax_dev, nd, zp, out, ld_out, transpose, st);
}
cudaError_t launch_quantize_scalar(const float* x, int64_t rows, int64_t cols, int64_t ld, int mode,
                                   const float* amax_dev, double nd, int32_t zp, int8_t* out,
                                   int64_t ld_out, int transpose, cudaStream_t st) {
    return quantize_scalar_t(x, rows, cols, ld, mode, amax_dev, nd, zp, out, ld_out, transpose, st);
}

cudaError_t launch_rowsum_i8(const int8_t* q, int64_t rows, int64_t cols, int64_t ld, int32_t* out,
                             cudaStream_t st) {
    if (rows <= 0) return cudaSuccess;
    rowsum_i8_kernel<<<static_cast<unsigned>((rows + 7) / 8), 256, 0, st>>>(q, rows, cols, ld, out);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_dequant_absmax(const int32_t* c, int64_t M, int64_t N, int64_t ldc, const float* amax_x,
                                  const float* amax_w, float* out, int64_t ldo, cudaStream_t st) {
    dequant_absmax_kernel<<<blocks_for(M * N), 256, 0, st>>>(c, M, N, ldc, amax_x, amax_w, out, ldo);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_zeropoint_combine(const int32_t* c, int64_t M, int64_t N, int64_t ldc,
                                     const int32_t* rowsum_a, const int32_t* colsum_b, int64_t K,
                                     int32_t zp_a, int32_t zp_b, double nd_a, double nd_b, double off_a,
                                     double off_b, float* out, int64_t ldo, int32_t* acc_out,
                                     int32_t* overflow, cudaStream_t st) {
    zeropoint_combine_kernel<<<blocks_for(M * N), 256, 0, st>>>(c, M, N, ldc, rowsum_a, colsum_b, K, zp_a, zp_b,
                                                              nd_a, nd_b, off_a, off_b, out, ldo, acc_out,
                                                              overflow);
    count_launch();
    return cudaGetLastError();
}

}  // namespace i8mm
