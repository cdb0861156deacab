/*
 * Plain-C restatement of the reference LLM.int8() matmul path.
 * TEST INFRASTRUCTURE ONLY: the checker for the CUDA path and the CPU
 * baseline timed by bench.py. The product never links or loads this file.
 *
 * Every function cites the reference line it restates (paths relative to
 * pkg/src/int8mm/ in the reference tree). Build: oracle/Makefile, compiled
 * with -ffp-contract=off so each double op is one IEEE round-to-nearest op,
 * exactly like numpy's per-ufunc float64 arithmetic.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

static void set_threads(int threads) {
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#else
    (void)threads;
#endif
}

/* quantize.py:26-29  round_half_away = copysign(floor(|x| + 0.5), x) */
static inline double round_half_away(double x) {
    volatile double t = fabs(x) + 0.5; /* one RN add, never fused */
    return copysign(floor(t), x);
}

/* quantize.py:115-117  clip(round_half_away(scaled), -127, 127) */
static inline int8_t to_code(double scaled) {
    double r = round_half_away(scaled);
    if (r > 127.0) r = 127.0;
    if (r < -127.0) r = -127.0;
    return (int8_t)r;
}

/* gemm.py:208-210  mask[k] = any_i |x_ik| >= f32(alpha); returns |O|. */
int64_t oracle_outlier_mask(const float* x, int64_t M, int64_t K, float alpha, uint8_t* mask) {
    memset(mask, 0, (size_t)K);
    for (int64_t i = 0; i < M; ++i) {
        const float* row = x + i * K;
        for (int64_t k = 0; k < K; ++k)
            if (fabsf(row[k]) >= alpha) mask[k] = 1;
    }
    int64_t n = 0;
    for (int64_t k = 0; k < K; ++k) n += mask[k];
    return n;
}

/* quantize.py:168-179 rowwise_quantize applied to x[:, keep] (gemm.py:242).
 * codes are written full-width (zeros at outlier columns); scales[i] =
 * 127/amax_i in f64, amax 0 -> scale 1. keep_mask NULL = keep everything. */
void oracle_rowwise_quantize(const float* x, int64_t M, int64_t K, const uint8_t* out_mask,
                             int8_t* codes, double* scales) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < M; ++i) {
        const float* row = x + i * K;
        float amax = 0.0f;
        for (int64_t k = 0; k < K; ++k)
            if (!out_mask || !out_mask[k]) {
                float a = fabsf(row[k]);
                if (a > amax) amax = a;
            }
        double s = 127.0 / (amax == 0.0f ? 127.0 : (double)amax);
        scales[i] = s;
        int8_t* q = codes + i * K;
        for (int64_t k = 0; k < K; ++k) {
            if (out_mask && out_mask[k]) { q[k] = 0; continue; }
            volatile double p = (double)row[k] * s;
            q[k] = to_code(p);
        }
    }
}

/* quantize.py:168-171,182-187 colwise_quantize applied to w[keep, :]
 * (gemm.py:243); codes full-height, zeros at outlier rows. */
void oracle_colwise_quantize(const float* w, int64_t K, int64_t N, const uint8_t* out_mask,
                             int8_t* codes, double* scales) {
    float* amax = (float*)calloc((size_t)N, sizeof(float));
    for (int64_t k = 0; k < K; ++k) {
        if (out_mask && out_mask[k]) continue;
        const float* row = w + k * N;
        for (int64_t j = 0; j < N; ++j) {
            float a = fabsf(row[j]);
            if (a > amax[j]) amax[j] = a;
        }
    }
    for (int64_t j = 0; j < N; ++j) scales[j] = 127.0 / (amax[j] == 0.0f ? 127.0 : (double)amax[j]);
    free(amax);
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < K; ++k) {
        int8_t* q = codes + k * N;
        if (out_mask && out_mask[k]) { memset(q, 0, (size_t)N); continue; }
        const float* row = w + k * N;
        for (int64_t j = 0; j < N; ++j) {
            volatile double p = (double)row[j] * scales[j];
            q[j] = to_code(p);
        }
    }
}

/* gemm.py:78-82 exact int8 x int8 -> int32 (|sum| <= 127^2 * 2^17 < 2^31).
 * a: MxK row-major, b: KxN row-major, c: MxN. Cache-blocked i-k-j order:
 * a block of RB rows of C (CB columns wide) stays in L1/L2 while each B row
 * segment is reused RB times; OpenMP over (row block, column block) tiles.
 * Integer addition is associative, so the blocking is exact. */
#define ORACLE_RB 16
#define ORACLE_CB 2048
__attribute__((target_clones("arch=x86-64-v4", "arch=x86-64-v3", "default")))
void oracle_gemm_i32(const int8_t* a, const int8_t* b, int32_t* c, int64_t M, int64_t N,
                     int64_t K, int threads) {
    set_threads(threads);
    const int64_t nrb = (M + ORACLE_RB - 1) / ORACLE_RB;
    const int64_t ncb = (N + ORACLE_CB - 1) / ORACLE_CB;
#pragma omp parallel for schedule(dynamic, 1) collapse(2)
    for (int64_t rb = 0; rb < nrb; ++rb) {
        for (int64_t cb = 0; cb < ncb; ++cb) {
            const int64_t i0 = rb * ORACLE_RB, i1 = i0 + ORACLE_RB < M ? i0 + ORACLE_RB : M;
            const int64_t j0 = cb * ORACLE_CB, j1 = j0 + ORACLE_CB < N ? j0 + ORACLE_CB : N;
            const int64_t w = j1 - j0;
            for (int64_t i = i0; i < i1; ++i) memset(c + i * N + j0, 0, (size_t)w * sizeof(int32_t));
            for (int64_t k = 0; k < K; ++k) {
                const int8_t* brow = b + k * N + j0;
                for (int64_t i = i0; i < i1; ++i) {
                    const int32_t av = a[i * K + k];
                    if (!av) continue;
                    int32_t* crow = c + i * N + j0;
                    for (int64_t j = 0; j < w; ++j) crow[j] += av * (int32_t)brow[j];
                }
            }
        }
    }
}

/* gemm.py:130,141,147  out = f32( f64(C) / (sx[i] * sw[j]) ) */
void oracle_dequantize_output(const int32_t* c, const double* sx, const double* sw, float* out,
                              int64_t M, int64_t N) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < M; ++i)
        for (int64_t j = 0; j < N; ++j) {
            volatile double d = sx[i] * sw[j];
            out[i * N + j] = (float)((double)c[i * N + j] / d);
        }
}

/* gemm.py:214-247 llm_int8_matmul. Returns |O| (decomposed_cols).
 * mask_out[K], sx[M], sw[N], out[MxN] required; xq (MxK), wq (KxN), c (MxN)
 * optional intermediate outputs (NULL = internal scratch). */
int64_t oracle_llm_int8_matmul(const float* x, const float* w, int64_t M, int64_t K, int64_t N,
                               float alpha, float* out, uint8_t* mask, double* sx, double* sw,
                               int8_t* xq, int8_t* wq, int32_t* c, int threads) {
    set_threads(threads);
    int64_t n_out = oracle_outlier_mask(x, M, K, alpha, mask); /* gemm.py:225 */
    int own_xq = !xq, own_wq = !wq, own_c = !c;
    if (own_xq) xq = (int8_t*)malloc((size_t)(M * K));
    if (own_wq) wq = (int8_t*)malloc((size_t)(K * N));
    if (own_c) c = (int32_t*)malloc((size_t)(M * N) * sizeof(int32_t));
    int64_t n_keep = K - n_out;
    if (n_keep > 0) {
        oracle_rowwise_quantize(x, M, K, mask, xq, sx);  /* gemm.py:242, 190-191 */
        oracle_colwise_quantize(w, K, N, mask, wq, sw);  /* gemm.py:243, 192 */
        oracle_gemm_i32(xq, wq, c, M, N, K, threads);     /* gemm.py:193 */
        oracle_dequantize_output(c, sx, sw, out, M, N);   /* gemm.py:194 */
    } else {
        memset(xq, 0, (size_t)(M * K));
        memset(wq, 0, (size_t)(K * N));
        memset(c, 0, (size_t)(M * N) * sizeof(int32_t));
        for (int64_t i = 0; i < M; ++i) sx[i] = 1.0;
        for (int64_t j = 0; j < N; ++j) sw[j] = 1.0;
    }
    if (n_out > 0) {
        int64_t* idx = (int64_t*)malloc((size_t)n_out * sizeof(int64_t));
        int64_t t = 0;
        for (int64_t k = 0; k < K; ++k)
            if (mask[k]) idx[t++] = k;
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < M; ++i) {
            for (int64_t j = 0; j < N; ++j) {
                /* gemm.py:110-117 ordered f64 accumulation, ascending k */
                double acc = 0.0;
                for (int64_t o = 0; o < n_out; ++o) {
                    volatile double p = (double)x[i * K + idx[o]] * (double)w[idx[o] * N + j];
                    acc = acc + p;
                }
                /* gemm.py:239-240 (no keep columns) / gemm.py:244 combine */
                if (n_keep > 0) out[i * N + j] = (float)((double)out[i * N + j] + acc);
                else out[i * N + j] = (float)acc;
            }
        }
        free(idx);
    }
    if (own_xq) free(xq);
    if (own_wq) free(wq);
    if (own_c) free(c);
    return n_out;
}

/* gemm.py:242-247 for a block of rows once O (mask) and the column side
 * (gemm.py:243: wq full-height codes with zeros at outlier rows, sw) are known:
 * rows are independent (rowwise scales, int8 GEMM, dequant, ordered f64
 * outlier term). bench.py's reference arm times this together with the scan
 * and the column quantization of the matching share of the workload. */
void oracle_llm_int8_rows(const float* x, int64_t M, int64_t K, int64_t N, const uint8_t* mask,
                          const int8_t* wq, const double* sw, const float* w, float* out,
                          int threads) {
    set_threads(threads);
    int64_t n_out = 0;
    for (int64_t k = 0; k < K; ++k) n_out += mask[k] ? 1 : 0;
    int64_t n_keep = K - n_out;
    int8_t* xq = (int8_t*)malloc((size_t)(M * K));
    int32_t* c = (int32_t*)malloc((size_t)(M * N) * sizeof(int32_t));
    double* sx = (double*)malloc((size_t)M * sizeof(double));
    if (n_keep > 0) {
        oracle_rowwise_quantize(x, M, K, mask, xq, sx);
        oracle_gemm_i32(xq, wq, c, M, N, K, threads);
        oracle_dequantize_output(c, sx, sw, out, M, N);
    }
    if (n_out > 0) {
        int64_t* idx = (int64_t*)malloc((size_t)n_out * sizeof(int64_t));
        int64_t t = 0;
        for (int64_t k = 0; k < K; ++k)
            if (mask[k]) idx[t++] = k;
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < M; ++i) {
            for (int64_t j = 0; j < N; ++j) {
                double acc = 0.0;
                for (int64_t o = 0; o < n_out; ++o) {
                    volatile double p = (double)x[i * K + idx[o]] * (double)w[idx[o] * N + j];
                    acc = acc + p;
                }
                if (n_keep > 0) out[i * N + j] = (float)((double)out[i * N + j] + acc);
                else out[i * N + j] = (float)acc;
            }
        }
        free(idx);
    }
    free(xq);
    free(c);
    free(sx);
}
