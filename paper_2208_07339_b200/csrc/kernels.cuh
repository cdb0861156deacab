// Internal declarations shared by the LLM.int8() CUDA translation units.
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdint>

namespace i8mm {

// launch accounting + device properties (capi.cu)
void count_launch();
int num_sms();
int check_device();  // I8MM_OK on sm_100, else I8MM_ERR_UNSUPPORTED
bool pdl_enabled();  // I8MM_PDL (default 1)

// Launch with programmatic dependent launch allowed (see pdl_wait in
// sm100_ptx.cuh); the kernel must call pdl_wait() before touching memory.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

cudaError_t launch_outlier_scan(const __half* x, int64_t M, int64_t K, int64_t ldx, float alpha,
                                uint32_t* col_mask, int32_t* nonfinite, cudaStream_t st);
cudaError_t launch_outlier_compact(const uint32_t* col_mask, int64_t K, int32_t* o_idx,
                                   int32_t* o_count, cudaStream_t st);
cudaError_t launch_quantize_rows(const __half* x, int64_t M, int64_t K, int64_t ldx,
                                 const uint32_t* mask, const int32_t* o_idx,
                                 const int32_t* o_count, int8_t* xq, int64_t ldq, float* amax,
                                 __half* xo, int64_t o_cap, cudaStream_t st);
// Row side of the prologue in one call: scan (+ per-row 64-column group maxima),
// compact, row scales (+ x[:, O]), streaming codes. `scratch` holds
// row_prologue_scratch_bytes(M, K); nullptr (or unaligned X) = scan, compact, quantize_rows.
size_t row_prologue_scratch_bytes(int64_t M, int64_t K);
// Weight-stationary per-call state that rides along with the row prologue
// (W[O, :] gather, column fixup, patched codes; see percall_dev.cuh).
struct PerCallFix {
    int32_t* c32;       // split-K scratch zeroed with the mask (or nullptr)
    int64_t c32_words;  // partial sums + counters
    const __half* w;
    int64_t K, N, ldw;
    __half* wo;
    int64_t ldwo;
    const float* amax_full;
    const uint16_t* cand_v;
    const int32_t* cand_r;
    const int8_t* q2;
    int32_t* p_count;  // [count, pad x3, patched-column bits]
    int32_t* p_idx;
    float* p_amax;
    int32_t* p_src;
    int8_t* wq_p;
};

// fix != nullptr: the weight-stationary per-call work is done too (its
// counters zeroed with the mask, gather + fixup fused into the row-scale
// grid, patched codes written by the code-pass CTAs).
cudaError_t launch_row_prologue(const __half* x, int64_t M, int64_t K, int64_t ldx, float alpha,
                                uint32_t* mask, int32_t* o_idx, int32_t* o_count, int8_t* xq,
                                int64_t ldq, float* row_amax, __half* xo, int64_t o_cap,
                                void* scratch, cudaStream_t st, const PerCallFix* fix = nullptr,
                                int32_t* nonfinite = nullptr);
cudaError_t launch_quantize_cols_t(const __half* w, int64_t K, int64_t N, int64_t ldw,
                                   const uint32_t* row_mask, int8_t* wq_t, int64_t ldq,
                                   float* col_amax, cudaStream_t st);
cudaError_t launch_dequantize_output(const int32_t* c, int64_t M, int64_t N, int64_t ldc,
                                     const double* sx, const double* sw, float* out, int64_t ldo,
                                     cudaStream_t st);
cudaError_t launch_gather_rows(const __half* w, int64_t ldw, int64_t N, const int32_t* idx,
                               const int32_t* count, int64_t cap, __half* out, int64_t ldo,
                               cudaStream_t st);
cudaError_t launch_col_amax(const __half* w, int64_t K, int64_t N, int64_t ldw,
                            const uint32_t* row_mask, float* col_amax, cudaStream_t st);
int64_t topt_chunk_rows(int64_t K);
constexpr int kTopT = 4;  // cached |w| candidates per column (weight-stationary fixup)
cudaError_t launch_weight_prepare(const __half* w, int64_t K, int64_t N, int64_t ldw, int8_t* wq_t,
                                  int8_t* q2, int64_t ldq, float* col_amax, uint16_t* cand_v,
                                  int32_t* cand_r, uint32_t* scratch_v, int32_t* scratch_r,
                                  cudaStream_t st);
// Weight-stationary per-call work after an unfused row prologue, in two
// launches: W[O, :] gather + column fixup (one grid; the p_count region
// already zeroed), then the patched columns' codes.
// p_count points at [count, pad x3, patched-column bit mask (ceil(N/32) words)];
// q2: cached codes under each column's second-largest |w| (K-major, ldq);
// p_src[p] = 1 when patch p's codes are q2's row (its top-1 row is the only
// outlier among the candidates), else they are re-derived from W.
cudaError_t launch_gather_fixup(const __half* w, int64_t K, int64_t N, int64_t ldw,
                                const uint32_t* mask, const int32_t* o_idx, const int32_t* o_count,
                                int64_t o_cap, __half* wo, int64_t ldwo, const float* amax_full,
                                const uint16_t* cand_v, const int32_t* cand_r, int32_t* p_count,
                                int32_t* p_idx, float* p_amax, int32_t* p_src, cudaStream_t st);
cudaError_t launch_patch_quantize(const __half* w, int64_t K, int64_t N, int64_t ldw,
                                  const uint32_t* mask, const int8_t* q2, const int32_t* p_count,
                                  const int32_t* p_idx, const float* p_amax, const int32_t* p_src,
                                  int8_t* wq_p, int64_t ldq, cudaStream_t st);
int64_t fixup_zero_words(int64_t N);  // size of the p_count region
cudaError_t launch_transpose_i8(const int8_t* src, int64_t rows, int64_t cols, int64_t lds,
                                int8_t* dst, int64_t ldd, cudaStream_t st);

// Sibling schemes (siblings.cu): tensor-wise absmax / zeropoint.
// stats_scratch: 3 int32 (device); out3: [amax, min, max] floats (device)
cudaError_t launch_tensor_stats(const __half* x, int64_t rows, int64_t cols, int64_t ld,
                                int32_t* stats_scratch, float* out3, cudaStream_t st);
// mode 0 = absmax (amax_dev), 1 = zeropoint (nd, zp); transpose writes K-major (cols x ld_out)
cudaError_t launch_quantize_scalar(const __half* x, int64_t rows, int64_t cols, int64_t ld, int mode,
                                   const float* amax_dev, double nd, int32_t zp, int8_t* out,
                                   int64_t ld_out, int transpose, cudaStream_t st);
cudaError_t launch_tensor_stats(const float* x, int64_t rows, int64_t cols, int64_t ld,
                                int32_t* stats_scratch, float* out3, cudaStream_t st);
cudaError_t launch_quantize_scalar(const float* x, int64_t rows, int64_t cols, int64_t ld, int mode,
                                   const float* amax_dev, double nd, int32_t zp, int8_t* out,
                                   int64_t ld_out, int transpose, cudaStream_t st);
cudaError_t launch_rowsum_i8(const int8_t* q, int64_t rows, int64_t cols, int64_t ld, int32_t* out,
                             cudaStream_t st);
cudaError_t launch_dequant_absmax(const int32_t* c, int64_t M, int64_t N, int64_t ldc, const float* amax_x,
                                  const float* amax_w, float* out, int64_t ldo, cudaStream_t st);
cudaError_t launch_zeropoint_combine(const int32_t* c, int64_t M, int64_t N, int64_t ldc,
                                     const int32_t* rowsum_a, const int32_t* colsum_b, int64_t K,
                                     int32_t zp_a, int32_t zp_b, double nd_a, double nd_b, double off_a,
                                     double off_b, float* out, int64_t ldo, int32_t* acc_out,
                                     int32_t* overflow, cudaStream_t st);

// Output kinds of the tcgen05 GEMM epilogue.
enum EpiKind : int { EPI_I32 = 0, EPI_F16 = 1, EPI_F32 = 2, EPI_F32_EXACT = 3 };

struct GemmArgs {
    const int8_t* a;  // M x lda int8 (K-major)
    int64_t lda;
    const int8_t* b;  // N x ldb int8 (K-major)
    int64_t ldb;
    int64_t M, N, K;
    void* y;
    int64_t ldy;
    // dequant + outlier epilogue (unused for EPI_I32)
    const float* row_amax;
    const float* col_amax;
    const __half* x;
    int64_t ldx;
    const __half* w;
    int64_t ldw;
    const __half* xo;
    int64_t o_cap;
    const int32_t* o_idx;
    const int32_t* o_count;
    // compact outlier rows of W: wo[t * ldwo + j] = W[o_idx[t], j] (nullable)
    const __half* wo;
    int64_t ldwo;
    int64_t wo_cap;
    // weight-stationary patches (nullable): b_patch holds the re-derived codes
    // (K-major, ldb) of *patch_count columns, patched column j is Y column
    // patch_idx[j] with amax patch_amax[j]; run as extra tiles of the same launch
    const int8_t* b_patch;
    const int32_t* patch_count;
    const int32_t* patch_idx;
    const float* patch_amax;
    const uint32_t* patch_mask;  // bit j set: column j is patched (main tiles skip it)
    // split-K for one m-tile (M <= 128) when few N-tiles would leave SMs idle
    // (nullable): zeroed int32 partial sums, column-major [cols x c32_rows]
    // (cols = gemm_split_cols: main and patch tiles), and per-tile arrival
    // counters [c32_tiles]
    int32_t* c32;
    int64_t c32_rows;
    int32_t* c32_cnt;
    int64_t c32_tiles;
    // fused output all-gather (fp16 out only): also store every output to
    // n_peer buffers y_peer[q] + row * peer_ldy + peer_col + column
    void* y_peer[8];
    int n_peer;
    int64_t peer_ldy, peer_col;
};
constexpr int kMaxPeers = 8;

// split-K scratch of the single-m-tile GEMM: c32 [cols x M] + counters
int64_t gemm_split_cols(int64_t N, bool patches);
int gemm_split_factor(int64_t M, int64_t N, int64_t K);  // 1 = no split
int64_t gemm_split_tiles(int64_t N, bool patches);
// swap-AB stream-K GEMM for M = 17..128 (swapab_sm100.cu)
bool swapab_route(int64_t M, int64_t K, int64_t N);
void set_swapab(int on);
void set_swapab_timeline(unsigned long long* stamps);
int64_t swapab_c32_words(int64_t M);
int64_t swapab_cnt_words(int64_t N);
cudaError_t launch_swapab(const GemmArgs& a, int32_t* c32, int32_t* tile_cnt, int epi, cudaStream_t st);

cudaError_t launch_gemm_sm100(const GemmArgs& args, int epi, cudaStream_t st);

// smallest fp16 bit pattern h (as |x| bits) with float(h) >= alpha (prologue.cu)
uint32_t alpha_threshold_bits(float alpha);

// Decode path (decode_sm100.cu): weight-stationary linear layer for M <= 256.
struct DecodeArgs {
    const __half* x;
    int64_t ldx;
    int64_t M, K, N;
    int x_vec;  // X rows 16-byte aligned (ldx % 8 == 0, base aligned)
    uint32_t thr_bits;
    const uint32_t* thr_bits_dev;  // nullable: threshold bits stored by i8mm_linear_prologue
    int32_t* nonfinite;   // [1] X holds NaN/Inf (the reference's DenseMatrix(x) rejects it)
    uint32_t* mask;       // [ceil(K/32)] outlier columns (published by cluster 0)
    int32_t* o_idx;       // [K]
    int32_t* o_count;     // [1]
    uint32_t* ramax_bits; // [M] row amax as fp16 bits
    float* row_amax;      // [M]
    int8_t* xq;           // [M x ldq] codes (published by cluster 0)
    int64_t ldq;
    const __half* w;      // K x N fp16 (resident)
    int64_t ldw;
    int w_vec;            // W rows 16-byte aligned (ldw % 8 == 0, base aligned)
    const int8_t* wq_t;   // N x ldq cached codes
    const float* amax_full;
    const uint16_t* cand_v;
    const int32_t* cand_r;
    const int8_t* q2;     // N x ldq second-candidate codes (weight buffer)
    int32_t* c32;         // [grid] x [16 x 128] split-tile partial slots: empty (0x80 bytes) on
                          // first use, emptied again by the finishers
    void* y;
    int64_t ldy;
};
constexpr int kDecodeMaxM = 16;  // decode_sm100.cu: the MMA N is 16 token rows
int decode_stages(int64_t M);
int decode_grid(int64_t K, int64_t N);
bool decode_fits(int64_t M, int64_t K, int64_t N);
// one launch of 8-CTA clusters: token side in distributed shared memory, then the
// swap-AB stream-K weight-stream GEMM + epilogue
cudaError_t launch_decode(const DecodeArgs& a, int epi, cudaStream_t st);
cudaError_t launch_set_word(uint32_t* dst, uint32_t value, cudaStream_t st);
void set_decode_timeline(unsigned long long* stamps);
unsigned long long* debug_timeline();  // the same buffer, also stamped by the GEMM (16 per CTA)
void set_gemm_variant(int cg_override, int mc_override);

}  // namespace i8mm
