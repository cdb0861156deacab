/*
 * llmint8.h -- C ABI of the B200 (sm_100a) LLM.int8() linear-layer path.
 *
 * Drop-in boundary for the reference package `int8mm`'s operator API
 * (reference tree: pkg/src/int8mm/). Plain pointers and sizes only; every
 * pointer argument is DEVICE memory unless stated otherwise, every function is
 * stream-ordered on `stream` (a cudaStream_t, NULL = legacy default stream)
 * and never synchronizes the host. The caller owns every buffer; nothing is
 * allocated or freed inside the library.
 *
 * Layouts (row-major, leading dimensions in elements):
 *   X     fp16  M x K   (activations; the reference's DenseMatrix x, f16-valued)
 *   W     fp16  K x N   (weights in the reference orientation, x @ w)
 *   Xq    int8  M x ldq (row-quantized X, 0 at outlier columns, ldq % 16 == 0)
 *   WqT   int8  N x ldq (column-quantized W stored K-major, 0 at outlier rows)
 *   Y     fp16 or fp32, M x N
 * Scales are carried as the exact absmax values (float32, exact for fp16
 * inputs): the reference's f64 scale is 127.0 / (amax == 0 ? 127 : amax).
 *
 * Return value: I8MM_OK (0) or one of the I8MM_ERR_* codes below; the Python
 * shim maps them onto the reference's exception classes.
 */
#ifndef LLMINT8_H
#define LLMINT8_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    I8MM_OK = 0,
    I8MM_ERR_SHAPE = 1,      /* ShapeMismatchError   (tensors.py:21, gemm.py:64-65) */
    I8MM_ERR_OVERFLOW = 2,   /* GemmOverflowError    (gemm.py:41, 66-69)            */
    I8MM_ERR_ALPHA = 3,      /* ValueError on alpha  (gemm.py:208-209)              */
    I8MM_ERR_PARAMS = 4,     /* ParamsMismatchError  (gemm.py:45, 136-146)          */
    I8MM_ERR_ARGUMENT = 5,   /* bad pointer / alignment / workspace too small        */
    I8MM_ERR_CUDA = 6,       /* CUDA launch or driver error                           */
    I8MM_ERR_UNSUPPORTED = 7, /* device is not sm_100                                 */
    I8MM_ERR_ZEROPOINT = 8   /* ValueError: zeropoint outside int16 (quantize.py:162-166) */
};

enum { I8MM_OUT_F16 = 0, I8MM_OUT_F32 = 1, I8MM_OUT_F32_EXACT = 2 };

#define I8MM_MAX_INNER_DIM (1 << 17) /* gemm.py:35 MAX_INNER_DIM */

/* Library identification / diagnostics. */
int i8mm_version(void);
const char* i8mm_status_string(int status);
/* Number of kernels this library launched since load (for bench accounting). */
uint64_t i8mm_launch_count(void);
/* Pin a GEMM kernel variant (A/B measurements, tests): cg_override 1 = the
 * 1-CTA kernel; mc_override 2 = 4-CTA clusters multicasting WqT between two
 * CTA pairs (M >= 2048); 0 = defaults (CTA pairs, no multicast). */
void i8mm_debug_set_gemm_variant(int cg_override, int mc_override);

/* K1. Outlier-column scan.  Replaces extract_outlier_columns' mask
 * (gemm.py:208-210): col_mask bit k is set iff some |X[i,k]| >= (float)alpha.
 * col_mask (ceil(K/32) words) is zeroed by the call. nonfinite (1 int32,
 * nullable) is set to 1 if X holds NaN/Inf (DenseMatrix rejects those,
 * tensors.py:47-48). */
int i8mm_outlier_scan(const void* x, int64_t M, int64_t K, int64_t ldx, float alpha,
                      uint32_t* col_mask, int32_t* nonfinite, void* stream);

/* Outlier index list: sorted ascending indices of set bits (gemm.py:211,
 * outliers.py:27-44) into o_idx[K], their count into *o_count (device). */
int i8mm_outlier_compact(const uint32_t* col_mask, int64_t K, int32_t* o_idx, int32_t* o_count,
                         void* stream);

/* K2. Row-wise quantization over the keep columns (quantize.py:168-179 applied
 * to x[:, keep], gemm.py:242) plus the outlier gather x[:, O] (gemm.py:238).
 * col_mask NULL = no outliers (plain rowwise_quantize). xo (M x o_cap fp16,
 * nullable) receives X[i, o_idx[t]] for t < min(*o_count, o_cap). */
int i8mm_quantize_rows(const void* x, int64_t M, int64_t K, int64_t ldx, const uint32_t* col_mask,
                       const int32_t* o_idx, const int32_t* o_count, int8_t* xq, int64_t ldq,
                       float* row_amax, void* xo, int64_t o_cap, void* stream);

/* K3. Column-wise quantization of W over the keep rows (quantize.py:168-171,
 * 182-187 applied to w[keep, :], gemm.py:243), written transposed (WqT, N x
 * ldq, K-major) for the tensor-core GEMM. row_mask NULL = no outliers. */
int i8mm_quantize_cols_t(const void* w, int64_t K, int64_t N, int64_t ldw, const uint32_t* row_mask,
                         int8_t* wq_t, int64_t ldq, float* col_amax, void* stream);

/* K4a. Exact int8 GEMM, C = A @ B with int32 accumulation (gemm.py:78-82).
 * a: M x K (lda), b_t: N x K (ldb) i.e. B stored K-major, c: M x N int32. */
int i8mm_gemm_i32(const int8_t* a, int64_t lda, const int8_t* b_t, int64_t ldb, int32_t* c,
                  int64_t ldc, int64_t M, int64_t N, int64_t K, void* stream);

/* K4b. Fused GEMM + dequantization + outlier term (gemm.py:120-147 row x col
 * branch, gemm.py:238 + 244-247):
 *   Y[i,j] = C[i,j] * (ax_i/127) * (aw_j/127) + sum_{t<|O|} X[i,O_t] * W[O_t, j]
 * xq/wq_t as produced by K2/K3; w (K x N fp16) supplies the outlier rows;
 * xo/o_cap as produced by K2 (x is used for outliers beyond o_cap).
 * out_kind: I8MM_OUT_F16 | I8MM_OUT_F32 (fp32 epilogue math) |
 * I8MM_OUT_F32_EXACT (f64 epilogue replicating the reference bit-for-bit). */
int i8mm_gemm_dequant(const int8_t* xq, const int8_t* wq_t, int64_t ldq, int64_t M, int64_t N,
                      int64_t K, const float* row_amax, const float* col_amax, const void* x,
                      int64_t ldx, const void* w, int64_t ldw, const void* xo, int64_t o_cap,
                      const void* wo, int64_t ldwo, const int32_t* o_idx, const int32_t* o_count,
                      void* y, int64_t ldy, int out_kind, void* stream);

/* Compact copy of the outlier rows W[O, :] (gemm.py:238 w.data[idx_out, :]):
 * wo[t * ldwo + j] = W[o_idx[t], j] for t < min(*o_count, cap). Feeds the
 * epilogue's outlier term with contiguous 16-byte loads (wo/ldwo above). */
int i8mm_gather_outlier_rows(const void* w, int64_t ldw, int64_t N, const int32_t* o_idx,
                             const int32_t* o_count, int64_t cap, void* wo, int64_t ldwo,
                             void* stream);

/* Exact dequantization of an int32 accumulator (gemm.py:130,141,147):
 * out[i,j] = (float)((double)c[i,j] / (sx[i] * sw[j])), f64 scales. */
int i8mm_dequantize_output(const int32_t* c, int64_t M, int64_t N, int64_t ldc, const double* sx,
                           const double* sw, float* out, int64_t ldo, void* stream);

/* int8 transpose helper (K x N -> N x ldq) for callers holding B row-major. */
int i8mm_transpose_i8(const int8_t* src, int64_t rows, int64_t cols, int64_t lds, int8_t* dst,
                      int64_t ldd, void* stream);

/* Whole-pipeline entry: llm_int8_matmul(x, w, alpha) (gemm.py:214-247) with
 * per-call W quantization, exactly the reference semantics. workspace must
 * hold i8mm_llm_int8_workspace_size(M, K, N) bytes (256-byte aligned).
 * *o_count_dev (device int32) receives |O| (decomposed_cols). */
size_t i8mm_llm_int8_workspace_size(int64_t M, int64_t K, int64_t N);
int i8mm_llm_int8_matmul(const void* x, int64_t ldx, const void* w, int64_t ldw, int64_t M,
                         int64_t K, int64_t N, float alpha, void* y, int64_t ldy, int out_kind,
                         void* workspace, size_t workspace_bytes, int32_t* o_count_dev,
                         void* stream);
/* Same, plus the reference's NaN/Inf rejection of X and W (tensors.py:47-48):
 * *nonfinite_dev (device int32, nullable) ends non-zero when either holds NaN/Inf. */
int i8mm_llm_int8_matmul_checked(const void* x, int64_t ldx, const void* w, int64_t ldw, int64_t M,
                                 int64_t K, int64_t N, float alpha, void* y, int64_t ldy, int out_kind,
                                 void* workspace, size_t workspace_bytes, int32_t* o_count_dev,
                                 int32_t* nonfinite_dev, void* stream);

/* ---------------------------------------------------------------------------
 * Int8 linear module (weight-stationary). Replaces the reference's module
 * boundary LinearBackend("llm_int8") + _linear (transformer.py:45-66,
 * 257-267), which re-quantizes W on every call (transformer.py:260, 267).
 * prepare() caches WqT with full-column scales, the codes q2 under each
 * column's second-largest |w| (what a patched column needs when only its
 * top-1 row is an outlier: one contiguous row instead of a strided column of
 * W; 1 byte per parameter), plus each column's top-4 |w|
 * candidates; forward() reproduces the per-call column scales over the keep
 * rows EXACTLY (quantize.py:182-187 on w[keep, :], gemm.py:243) by patching
 * only the columns whose cached maximisers are all outlier rows. Outputs are
 * identical to i8mm_llm_int8_matmul. W (fp16, K x N) must stay resident: the
 * outlier rows are multiplied in fp16 (gemm.py:238).
 */
size_t i8mm_linear_weight_bytes(int64_t K, int64_t N);
size_t i8mm_linear_prepare_scratch_bytes(int64_t K, int64_t N);
int i8mm_linear_prepare(const void* w, int64_t ldw, int64_t K, int64_t N, void* wbuf,
                        size_t wbuf_bytes, void* scratch, size_t scratch_bytes, void* stream);
size_t i8mm_linear_workspace_size(int64_t M, int64_t K, int64_t N);
/* scan + compact + quantize rows + gather outlier rows + column fixup */
int i8mm_linear_prologue(const void* x, int64_t ldx, int64_t M, const void* w, int64_t ldw,
                         const void* wbuf, int64_t K, int64_t N, float alpha, void* workspace,
                         size_t workspace_bytes, void* stream);
/* main tcgen05 GEMM over the cached codes + col-mapped GEMM over the patches */
int i8mm_linear_gemm(const void* x, int64_t ldx, int64_t M, const void* w, int64_t ldw,
                     const void* wbuf, int64_t K, int64_t N, void* y, int64_t ldy, int out_kind,
                     void* workspace, size_t workspace_bytes, void* stream);
/* GEMM + epilogue over rows [row0, row0 + rows) only, after one
 * i8mm_linear_prologue over all M rows (same workspace; y is the full output,
 * rows outside the range are untouched). Rows are independent once O and the
 * row scales are known (gemm.py:210, 242), so a caller can pipeline output
 * transfers (all-gather, device-to-host) behind later row ranges. Prefill
 * routing only (decode calls are a single launch: row0 = 0, rows = M). */
int i8mm_linear_gemm_rows(const void* x, int64_t ldx, int64_t M, const void* w, int64_t ldw,
                          const void* wbuf, int64_t K, int64_t N, void* y, int64_t ldy, int out_kind,
                          void* workspace, size_t workspace_bytes, int64_t row0, int64_t rows,
                          void* stream);
/* prologue + gemm; *o_count_dev (nullable) receives |O| */
int i8mm_linear_forward(const void* x, int64_t ldx, int64_t M, const void* w, int64_t ldw,
                        const void* wbuf, int64_t K, int64_t N, float alpha, void* y, int64_t ldy,
                        int out_kind, void* workspace, size_t workspace_bytes,
                        int32_t* o_count_dev, void* stream);
/* Decode routing. Calls with M <= max_m (default 16, env I8MM_DECODE_MAX_M,
 * at most 16) run ONE launch of 8-CTA thread-block clusters (decode_sm100.cu):
 * each cluster derives the outlier set, row scales and codes in distributed
 * shared memory, the weight stream starts before the dependency wait, and a
 * swap-AB stream-K tcgen05 GEMM streams WqT once over all SMs; patched columns
 * are decided and dotted per tile. i8mm_linear_forward issues exactly that
 * launch; with the split entries, i8mm_linear_prologue only records alpha and
 * i8mm_linear_gemm runs the kernel. Outputs are bit-identical to the prefill
 * kernels. The workspace layout depends on the routing, so set max_m before
 * sizing a workspace. A decode-routed workspace carries split-tile partial
 * slots that must be empty (and per-tile counters zero) when it is first used:
 * call i8mm_linear_workspace_init once after allocating it (every decode call
 * leaves them so; one workspace per stream and per (M, K, N): the slots' offset
 * depends on the shape, so re-initialise a buffer before using it for another). */
int i8mm_linear_workspace_init(void* workspace, size_t workspace_bytes, int64_t M, int64_t K, int64_t N,
                               void* stream);
/* Patched-column list of the last decode-routed call on this workspace
 * (p_count / p_idx / p_amax views): the decode kernel decides patched columns
 * per tile without publishing them; this recomputes the list the prefill
 * prologue writes (introspection only, not needed for the outputs). No-op for
 * prefill-routed workspaces. */
int i8mm_linear_patch_stats(const void* w, int64_t ldw, const void* wbuf, int64_t M, int64_t K, int64_t N,
                            void* workspace, size_t workspace_bytes, void* stream);
void i8mm_debug_set_decode_max_m(int max_m);
/* Test / A-B hook: route weight-stationary prefill calls with 17 <= M <= 128 through
 * the swap-AB stream-K GEMM (1, default; env I8MM_SWAPAB=0 disables) or the row-tile
 * GEMM (0). Workspaces sized under one setting must be used under the same one. */
void i8mm_debug_set_swapab(int on);
/* Dev tool: per-CTA %globaltimer stamps of the swap-AB GEMM (16 u64 per CTA, dev
 * build only; NULL disables). */
void i8mm_debug_swapab_timeline(void* stamps);
/* Programmatic dependent launch on the prefill path: 1 on (default), 0 off
   (same as I8MM_PDL=0); for A/B measurements. */
void i8mm_debug_set_pdl(int on);
int i8mm_linear_uses_decode(int64_t M, int64_t K, int64_t N);
/* Dev tool: per-CTA %globaltimer stamps of the decode kernel (64 u64 per CTA,
 * device buffer sized for one CTA per SM; NULL disables). */
void i8mm_debug_decode_timeline(void* stamps);
/* Fused output all-gather for N-sharded layers (fp16 out): like
 * i8mm_linear_forward, and every output element Y[i, j] is also stored, from the
 * GEMM epilogue, to y_peers[q][i * ldy_peer + col_off + j] for q < n_peers
 * (n_peers <= 8). y_peers are device pointers this device can store to: the
 * other ranks' full-width Y buffers in NVLink peer memory (symmetric memory),
 * this rank's own included. The caller orders the peers' reads after the
 * writes (a cross-rank barrier). Decode-routed calls (M <= 16) store the block
 * with copy-engine peer copies instead. */
int i8mm_linear_forward_peers(const void* x, int64_t ldx, int64_t M, const void* w, int64_t ldw,
                              const void* wbuf, int64_t K, int64_t N, float alpha, void* y, int64_t ldy,
                              void* workspace, size_t workspace_bytes, void* const* y_peers, int n_peers,
                              int64_t ldy_peer, int64_t col_off, void* stream);
/* introspection (tests): device pointers into the workspace / weight buffer.
 * workspace views: [o_count, o_idx, xq, row_amax, p_count, p_idx, p_amax, wq_p]
 * weight views:    [wq_t, col_amax, cand_v, cand_r(, q2)] */
int i8mm_linear_workspace_views(void* workspace, int64_t M, int64_t K, int64_t N, void** views,
                                int n_views);
int i8mm_linear_weight_views(void* wbuf, int64_t K, int64_t N, void** views, int n_views);

/* ---------------------------------------------------------------------------
 * Sibling schemes of the backend plugin point (LinearBackend kinds "absmax"
 * and "zeropoint", transformer.py:42-62): tensor-wise quantization and its
 * matmuls on the same tcgen05 int8 GEMM.
 */
/* One pass over X: out3 = [max|x|, min x, max x] (float, device); scratch =
 * 3 int32 of device memory. (quantize.py:141, 157-158) */
int i8mm_tensor_stats(const void* x, int64_t rows, int64_t cols, int64_t ld, int32_t* scratch,
                      float* out3, void* stream);
/* absmax_quantize codes (quantize.py:137-151): clip(rha(127/amax * x)), amax
 * read from device memory (0 -> all-zero codes). transpose = 1 writes the
 * K-major layout (cols x ldq) the GEMM uses for B; padding written 0. */
int i8mm_absmax_quantize(const void* x, int64_t rows, int64_t cols, int64_t ld, const float* amax,
                         int8_t* q, int64_t ldq, int transpose, void* stream);
/* Host-side zeropoint parameters from the tensor's min/max, exactly as
 * quantize.py:153-166: constant tensor -> (nd 1, zp 0, offset lo); else
 * nd = 254/(hi-lo), zp = rha(nd*lo) + 127, I8MM_ERR_ZEROPOINT outside int16. */
int i8mm_zeropoint_params(float lo, float hi, double* nd, int32_t* zp, double* offset);
/* zeropoint_quantize codes (quantize.py:167-171): clip(rha(nd*x) - zp). */
int i8mm_zeropoint_quantize(const void* x, int64_t rows, int64_t cols, int64_t ld, double nd, int32_t zp,
                            int8_t* q, int64_t ldq, int transpose, void* stream);
/* out[r] = sum of the int8 row r (rowsum(A); colsum(B) of a K-major B). */
int i8mm_rowsum_i8(const int8_t* q, int64_t rows, int64_t cols, int64_t ld, int32_t* out, void* stream);
/* absmax dequantization (gemm.py:133): f32(f64(c) / (s_x * s_w)), s = 127/amax. */
int i8mm_dequantize_absmax(const int32_t* c, int64_t M, int64_t N, int64_t ldc, const float* amax_x,
                           const float* amax_w, float* out, int64_t ldo, void* stream);
/* zeropoint_gemm_i32 (gemm.py:85-104, unrolled form, exact int64) with the
 * int32 range check (gemm.py:71-75 -> *overflow = 1) and, when out != NULL,
 * the dequantization + constant-offset terms of zeropoint_matmul
 * (gemm.py:175-187); acc_out (nullable) receives the int32 accumulator. */
int i8mm_zeropoint_combine(const int32_t* c, int64_t M, int64_t N, int64_t ldc, const int32_t* rowsum_a,
                           const int32_t* colsum_b, int64_t K, int32_t zp_a, int32_t zp_b, double nd_a,
                           double nd_b, double off_a, double off_b, float* out, int64_t ldo,
                           int32_t* acc_out, int32_t* overflow, void* stream);
/* Whole pipelines, fp16 X (M x K) and W (K x N), float32 Y. */
size_t i8mm_scalar_workspace_size(int64_t M, int64_t K, int64_t N);
/* absmax_matmul (gemm.py:150-156); never synchronizes the host. */
int i8mm_absmax_matmul(const void* x, int64_t ldx, const void* w, int64_t ldw, int64_t M, int64_t K,
                       int64_t N, float* y, int64_t ldy, void* workspace, size_t workspace_bytes,
                       void* stream);
/* zeropoint_matmul (gemm.py:159-187; unrolled and direct forms are identical).
 * Synchronizes the stream: the zeropoints are validated on the host. */
int i8mm_zeropoint_matmul(const void* x, int64_t ldx, const void* w, int64_t ldw, int64_t M, int64_t K,
                          int64_t N, float* y, int64_t ldy, void* workspace, size_t workspace_bytes,
                          void* stream);

/* ---------------------------------------------------------------------------
 * float32 operands: the reference's DenseMatrix holds float32
 * (tensors.py:31-49). Values that are all exactly fp16 run the fp16 kernels
 * above (bit-identical); otherwise these reproduce the reference on the f32
 * values themselves. Flags words: bit 0 = a NaN/Inf entry (the reference's
 * DenseMatrix raises ValueError, tensors.py:47-48), bit 1 = an entry that is
 * not exactly an fp16 value, bit 2 = an int8 code of -128 (tensors.py:95-98).
 */
#define I8MM_FLAG_NONFINITE 1
#define I8MM_FLAG_NOT_F16 2
#define I8MM_FLAG_CODE_128 4
/* One pass over f32 X: outlier column mask (|x| >= f32(alpha), gemm.py:208-210;
 * zeroed here; NULL = no mask), flags |= (atomic OR; caller zeroes), and an
 * fp16 copy when y16 != NULL. */
int i8mm_f32_scan(const float* x, int64_t rows, int64_t cols, int64_t ld, float alpha, uint32_t* col_mask,
                  int32_t* flags, void* y16, int64_t ldy, void* stream);
/* quantize.py:168-179 / 182-187 on f32 operands (mask NULL = no outliers). */
int i8mm_f32_quantize_rows(const float* x, int64_t M, int64_t K, int64_t ldx, const uint32_t* col_mask,
                           int8_t* xq, int64_t ldq, float* row_amax, void* stream);
int i8mm_f32_quantize_cols_t(const float* w, int64_t K, int64_t N, int64_t ldw, const uint32_t* row_mask,
                             int8_t* wq_t, int64_t ldq, float* col_amax, void* stream);
/* gemm.py:239-247 from the int32 accumulator: row x col dequantization, the
 * ordered f64 outlier term over the sorted o_idx[0..*o_count), the sum. */
int i8mm_f32_llm_int8_combine(const int32_t* c, int64_t ldc, int64_t M, int64_t N, int64_t K,
                              const float* row_amax, const float* col_amax, const float* x, int64_t ldx,
                              const float* w, int64_t ldw, const int32_t* o_idx, const int32_t* o_count,
                              float* y, int64_t ldy, void* stream);
/* The whole of gemm.py:214-247 on f32 X (M x K) and W (K x N), float32 Y,
 * bit-identical to the reference for every finite input. status_out (2 device
 * int32): [|O|, flags]; never synchronizes the host. */
size_t i8mm_f32_workspace_size(int64_t M, int64_t K, int64_t N);
int i8mm_llm_int8_matmul_f32(const float* x, int64_t ldx, const float* w, int64_t ldw, int64_t M,
                             int64_t K, int64_t N, float alpha, float* y, int64_t ldy, void* workspace,
                             size_t workspace_bytes, int32_t* status_out, void* stream);
/* gemm.py:110-117 ordered_matmul_f64: f64 accumulation in ascending inner
 * index, each product and sum one IEEE op; x, w f32 (elt_bytes 4) or f64 (8). */
int i8mm_ordered_matmul_f64(const void* x, int64_t ldx, const void* w, int64_t ldw, int64_t M, int64_t K,
                            int64_t N, int elt_bytes, double* out, int64_t ldo, void* stream);
/* quantize.py:26-29 round_half_away on n f32 (4) / f64 (8) values -> f64. */
int i8mm_round_half_away(const void* src, int64_t n, int elt_bytes, double* dst, void* stream);
/* quantize.py:214-227 dequantize: codes -> float32 per params kind. */
#define I8MM_DEQ_ABSMAX 0
#define I8MM_DEQ_ZEROPOINT 1
#define I8MM_DEQ_ROWWISE 2
#define I8MM_DEQ_COLWISE 3
int i8mm_dequantize_codes(const int8_t* q, int64_t rows, int64_t cols, int64_t ldq, int mode,
                          const double* s_row, const double* s_col, double scale, int32_t zp, double nd,
                          double offset, float* out, int64_t ldo, void* stream);
/* flags |= I8MM_FLAG_CODE_128 when any code is -128 (tensors.py:95-98). */
int i8mm_check_codes(const int8_t* q, int64_t rows, int64_t cols, int64_t ldq, int32_t* flags, void* stream);
/* flags |= I8MM_FLAG_NONFINITE when an fp16 entry is NaN/Inf (tensors.py:47-48). */
int i8mm_f16_check(const void* x, int64_t rows, int64_t cols, int64_t ld, int32_t* flags, void* stream);
/* exact fp16 -> f32 widening (mixed f16 / f32 operand pairs). */
int i8mm_f16_to_f32(const void* x, int64_t rows, int64_t cols, int64_t ld, float* y, int64_t ldy, void* stream);
/* stream-ordered memset 0 of device bytes (flag words, counters). */
int i8mm_zero(void* p, size_t bytes, void* stream);
/* tensor-wise statistics / quantizers of the sibling schemes on f32 operands. */
int i8mm_tensor_stats_f32(const float* x, int64_t rows, int64_t cols, int64_t ld, int32_t* scratch,
                          float* out3, void* stream);
int i8mm_absmax_quantize_f32(const float* x, int64_t rows, int64_t cols, int64_t ld, const float* amax,
                             int8_t* q, int64_t ldq, int transpose, void* stream);
int i8mm_zeropoint_quantize_f32(const float* x, int64_t rows, int64_t cols, int64_t ld, double nd, int32_t zp,
                                int8_t* q, int64_t ldq, int transpose, void* stream);

/* ---------------------------------------------------------------------------
 * Measurement (not on the reference path): the box's own dense
 * INT8 tensor-core ceiling, the roofline denominator of bench.py. Launches a
 * kernel that only issues tcgen05.mma.kind::i8 from shared memory (random
 * operands), one CTA (cg = 1, M = 128) or CTA pair (cg = 2, M = 256) per SM,
 * N = 256, `iters` x 8 MMAs each. i8mm_peak_mma_ops = int8 ops of one launch. */
int i8mm_peak_mma_launch(int cg, int iters, void* stream);
double i8mm_peak_mma_ops(int cg, int iters);

#ifdef __cplusplus
}
#endif
#endif /* LLMINT8_H */
