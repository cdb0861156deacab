// extern "C" boundary of the B200 LLM.int8() library (declared in
// include/llmint8.h). Host-side validation mirrors the reference's error
// contract (gemm.py:63-69, 208-209; tensors.py:21) so the Python shim can
// raise the same exception classes; compute is stream-ordered and never
// synchronizes the host.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstring>
#include <cstdint>
#include <cstdlib>
#include <mutex>

#include "../../include/llmint8.h"
#include "kernels.cuh"

namespace i8mm {

static std::atomic<uint64_t> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

static int g_pdl = -1;
bool pdl_enabled() {
    if (g_pdl < 0) {
        const char* e = getenv("I8MM_PDL");
        g_pdl = (e && e[0] == '0') ? 0 : 1;
    }
    return g_pdl == 1;
}

int num_sms() {
    static int sms = 0;
    static std::once_flag once;
    std::call_once(once, [] {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    });
    return sms;
}

int check_device() {
    static int ok = -1;
    static std::once_flag once;
    std::call_once(once, [] {
        int dev = 0, major = 0, minor = 0;
        if (cudaGetDevice(&dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess) {
            ok = 0;
            return;
        }
        ok = (major == 10 && minor == 0) ? 1 : 0;
    });
    return ok ? I8MM_OK : I8MM_ERR_UNSUPPORTED;
}

static int cuda_status(cudaError_t e) { return e == cudaSuccess ? I8MM_OK : I8MM_ERR_CUDA; }

static inline int64_t round_up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }

// gemm.py:63-69 _check_inner (shape part is checked by the callers)
static int check_inner(int64_t K) {
    if (K > I8MM_MAX_INNER_DIM) return I8MM_ERR_OVERFLOW;
    return I8MM_OK;
}

}  // namespace i8mm

using namespace i8mm;

extern "C" {

int i8mm_version(void) { return 1; }

const char* i8mm_status_string(int s) {
    switch (s) {
        case I8MM_OK: return "ok";
        case I8MM_ERR_SHAPE: return "shape mismatch";
        case I8MM_ERR_OVERFLOW: return "inner dimension exceeds the int32 overflow guard";
        case I8MM_ERR_ALPHA: return "alpha must be positive and finite";
        case I8MM_ERR_PARAMS: return "quantization params mismatch";
        case I8MM_ERR_ARGUMENT: return "invalid argument";
        case I8MM_ERR_CUDA: return "CUDA error";
        case I8MM_ERR_UNSUPPORTED: return "device is not sm_100 (B200)";
        case I8MM_ERR_ZEROPOINT: return "input offset too extreme for a 16-bit zeropoint";
        default: return "unknown status";
    }
}

uint64_t i8mm_launch_count(void) { return g_launches.load(); }

void i8mm_debug_set_gemm_variant(int cg_override, int mc_override) {
    set_gemm_variant(cg_override, mc_override);
}

int i8mm_outlier_scan(const void* x, int64_t M, int64_t K, int64_t ldx, float alpha,
                      uint32_t* col_mask, int32_t* nonfinite, void* stream) {
    if (int s = check_device()) return s;
    if (!(alpha > 0.0f) || !std::isfinite(alpha)) return I8MM_ERR_ALPHA;
    if (M < 0 || K <= 0 || ldx < K || !col_mask || (M > 0 && !x)) return I8MM_ERR_ARGUMENT;
    return cuda_status(launch_outlier_scan(static_cast<const __half*>(x), M, K, ldx, alpha,
                                           col_mask, nonfinite, static_cast<cudaStream_t>(stream)));
}

int i8mm_outlier_compact(const uint32_t* col_mask, int64_t K, int32_t* o_idx, int32_t* o_count,
                         void* stream) {
    if (int s = check_device()) return s;
    if (K <= 0 || !col_mask || !o_idx || !o_count) return I8MM_ERR_ARGUMENT;
    return cuda_status(
        launch_outlier_compact(col_mask, K, o_idx, o_count, static_cast<cudaStream_t>(stream)));
}

int i8mm_quantize_rows(const void* x, int64_t M, int64_t K, int64_t ldx, const uint32_t* col_mask,
                       const int32_t* o_idx, const int32_t* o_count, int8_t* xq, int64_t ldq,
                       float* row_amax, void* xo, int64_t o_cap, void* stream) {
    if (int s = check_device()) return s;
    if (M < 0 || K <= 0 || ldx < K || ldq < K || !xq || !row_amax || (M > 0 && !x))
        return I8MM_ERR_ARGUMENT;
    if (xo && (!o_idx || !o_count || o_cap <= 0)) return I8MM_ERR_ARGUMENT;
    return cuda_status(launch_quantize_rows(static_cast<const __half*>(x), M, K, ldx, col_mask,
                                            o_idx, o_count, xq, ldq, row_amax,
                                            static_cast<__half*>(xo), o_cap,
                                            static_cast<cudaStream_t>(stream)));
}

int i8mm_quantize_cols_t(const void* w, int64_t K, int64_t N, int64_t ldw, const uint32_t* row_mask,
                         int8_t* wq_t, int64_t ldq, float* col_amax, void* stream) {
    if (int s = check_device()) return s;
    if (K <= 0 || N < 0 || ldw < N || ldq < K || !wq_t || !col_amax || (N > 0 && !w))
        return I8MM_ERR_ARGUMENT;
    return cuda_status(launch_quantize_cols_t(static_cast<const __half*>(w), K, N, ldw, row_mask,
                                              wq_t, ldq, col_amax,
                                              static_cast<cudaStream_t>(stream)));
}

int i8mm_gemm_i32(const int8_t* a, int64_t lda, const int8_t* b_t, int64_t ldb, int32_t* c,
                  int64_t ldc, int64_t M, int64_t N, int64_t K, void* stream) {
    if (int s = check_device()) return s;
    if (int s = check_inner(K)) return s;
    if (M < 0 || N < 0 || K < 0 || lda < K || ldb < K || ldc < N || !a || !b_t || !c)
        return I8MM_ERR_ARGUMENT;
    if ((lda % 16) || (ldb % 16)) return I8MM_ERR_ARGUMENT;
    GemmArgs g{};
    g.a = a;
    g.lda = lda;
    g.b = b_t;
    g.ldb = ldb;
    g.M = M;
    g.N = N;
    g.K = K;
    g.y = c;
    g.ldy = ldc;
    return cuda_status(launch_gemm_sm100(g, EPI_I32, static_cast<cudaStream_t>(stream)));
}

int i8mm_gemm_dequant(const int8_t* xq, const int8_t* wq_t, int64_t ldq, int64_t M, int64_t N,
                      int64_t K, const float* row_amax, const float* col_amax, const void* x,
                      int64_t ldx, const void* w, int64_t ldw, const void* xo, int64_t o_cap,
                      const void* wo, int64_t ldwo, const int32_t* o_idx, const int32_t* o_count,
                      void* y, int64_t ldy, int out_kind, void* stream) {
    if (int s = check_device()) return s;
    if (int s = check_inner(K)) return s;
    if (M < 0 || N < 0 || K <= 0 || ldq < K || (ldq % 16) || ldy < N || !xq || !wq_t ||
        !row_amax || !col_amax || !y)
        return I8MM_ERR_ARGUMENT;
    if (o_count && (!o_idx || !x || !w || ldx < K || ldw < N)) return I8MM_ERR_ARGUMENT;
    int epi;
    switch (out_kind) {
        case I8MM_OUT_F16: epi = EPI_F16; break;
        case I8MM_OUT_F32: epi = EPI_F32; break;
        case I8MM_OUT_F32_EXACT: epi = EPI_F32_EXACT; break;
        default: return I8MM_ERR_ARGUMENT;
    }
    GemmArgs g{};
    g.a = xq;
    g.lda = ldq;
    g.b = wq_t;
    g.ldb = ldq;
    g.M = M;
    g.N = N;
    g.K = K;
    g.y = y;
    g.ldy = ldy;
    g.row_amax = row_amax;
    g.col_amax = col_amax;
    g.x = static_cast<const __half*>(x);
    g.ldx = ldx;
    g.w = static_cast<const __half*>(w);
    g.ldw = ldw;
    g.xo = static_cast<const __half*>(xo);
    g.o_cap = xo ? o_cap : 0;
    g.o_idx = o_idx;
    g.o_count = o_count;
    g.wo = static_cast<const __half*>(wo);
    g.ldwo = ldwo;
    g.wo_cap = wo ? o_cap : 0;
    return cuda_status(launch_gemm_sm100(g, epi, static_cast<cudaStream_t>(stream)));
}

int i8mm_gather_outlier_rows(const void* w, int64_t ldw, int64_t N, const int32_t* o_idx,
                             const int32_t* o_count, int64_t cap, void* wo, int64_t ldwo,
                             void* stream) {
    if (int s = check_device()) return s;
    if (N <= 0 || ldw < N || ldwo < N || cap < 0 || !w || !o_idx || !o_count || !wo)
        return I8MM_ERR_ARGUMENT;
    return cuda_status(launch_gather_rows(static_cast<const __half*>(w), ldw, N, o_idx, o_count, cap,
                                          static_cast<__half*>(wo), ldwo,
                                          static_cast<cudaStream_t>(stream)));
}

int i8mm_dequantize_output(const int32_t* c, int64_t M, int64_t N, int64_t ldc, const double* sx,
                           const double* sw, float* out, int64_t ldo, void* stream) {
    if (int s = check_device()) return s;
    if (M < 0 || N < 0 || ldc < N || ldo < N || !c || !sx || !sw || !out) return I8MM_ERR_ARGUMENT;
    return cuda_status(
        launch_dequantize_output(c, M, N, ldc, sx, sw, out, ldo, static_cast<cudaStream_t>(stream)));
}

int i8mm_transpose_i8(const int8_t* src, int64_t rows, int64_t cols, int64_t lds, int8_t* dst,
                      int64_t ldd, void* stream) {
    if (int s = check_device()) return s;
    if (rows < 0 || cols < 0 || lds < cols || ldd < rows || !src || !dst) return I8MM_ERR_ARGUMENT;
    return cuda_status(
        launch_transpose_i8(src, rows, cols, lds, dst, ldd, static_cast<cudaStream_t>(stream)));
}

// ---------------------------------------------------------------- pipeline
namespace {
struct Workspace {
    uint32_t* mask;
    int32_t* o_idx;
    int32_t* o_count;
    int32_t* nonfinite;
    float* row_amax;
    float* col_amax;
    int8_t* xq;
    int8_t* wq_t;
    __half* xo;
    __half* wo;
    int32_t* p_count;
    int32_t* p_idx;
    float* p_amax;
    int32_t* p_src;
    int8_t* wq_p;
    // decode path (M <= decode_max_m(), weight-stationary only)
    bool decode;
    uint32_t* ramax_bits;
    int32_t* patch_pos;
    int32_t* c32;
    int64_t c32_words;
    int32_t* tile_cnt;
    int64_t n_tiles;
    uint32_t* thr_word;  // alpha threshold bits, written by the prologue entry
    void* rp_scratch;    // prefill: per-row group maxima + f64 row scales (launch_row_prologue)
    int32_t* sk_c32;     // prefill M <= 128 (linear): split-K partial sums, then tile counters
    int64_t sk_ld, sk_words;
    int32_t* sab_c32;    // prefill M = 17..128 (linear): swap-AB partial slots, then tile counters
    int32_t* sab_cnt;
    int64_t sab_cnt_words;
    int64_t ldq, o_cap;
    size_t bytes;
};
constexpr int64_t kOCap = 64;

// Largest M routed to the decode kernels (decode_sm100.cu). Default from
// I8MM_DECODE_MAX_M (0 disables), else 16 (measured crossover, profiles/r1); capped at kDecodeMaxM.
int g_decode_max_m = -1;
int decode_max_m() {
    if (g_decode_max_m < 0) {
        const char* e = getenv("I8MM_DECODE_MAX_M");
        g_decode_max_m = (e && e[0]) ? atoi(e) : 16;
        if (g_decode_max_m > kDecodeMaxM) g_decode_max_m = kDecodeMaxM;
        if (g_decode_max_m < 0) g_decode_max_m = 0;
    }
    return g_decode_max_m;
}

bool uses_decode(int64_t M, int64_t K, int64_t N) {
    // small weight matrices at 12 <= M <= 16 run faster through the swap-AB GEMM
    return M > 0 && M <= decode_max_m() && decode_fits(M, K, N) && !swapab_route(M, K, N);
}  // compacted outlier slice width (wider |O| reads X directly)

// Per-call workspace. `linear` = weight-stationary layout: no WqT (it lives in
// the prepared weight buffer) but room for the patched columns (worst case N).
Workspace carve(void* base, int64_t M, int64_t K, int64_t N, bool linear = false) {
    Workspace w{};
    w.ldq = round_up(K, 16);
    w.o_cap = kOCap;
    uintptr_t p = reinterpret_cast<uintptr_t>(base);
    const uintptr_t p0 = p;
    auto take = [&](size_t bytes) {
        uintptr_t r = p;
        p += static_cast<uintptr_t>(round_up(static_cast<int64_t>(bytes), 256));
        return r;
    };
    w.mask = reinterpret_cast<uint32_t*>(take(sizeof(uint32_t) * ((K + 31) / 32)));
    w.o_idx = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * K));
    w.o_count = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * 2));
    w.nonfinite = w.o_count + 1;
    w.row_amax = reinterpret_cast<float*>(take(sizeof(float) * (M > 0 ? M : 1)));
    w.col_amax = reinterpret_cast<float*>(take(sizeof(float) * (N > 0 ? N : 1)));
    w.xq = reinterpret_cast<int8_t*>(take(static_cast<size_t>(M * w.ldq)));
    w.wq_t = linear ? nullptr : reinterpret_cast<int8_t*>(take(static_cast<size_t>(N * w.ldq)));
    w.xo = reinterpret_cast<__half*>(take(sizeof(__half) * static_cast<size_t>(M * kOCap)));
    w.wo = reinterpret_cast<__half*>(take(sizeof(__half) * static_cast<size_t>(kOCap * round_up(N, 8))));
    if (linear) {
        w.p_count = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * (4 + (N + 31) / 32)));
        w.p_idx = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * N));
        w.p_amax = reinterpret_cast<float*>(take(sizeof(float) * N));
        w.p_src = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * N));
        w.decode = uses_decode(M, K, N);
        if (w.decode) {
            // patched columns are dotted in the prologue: no patch codes, but
            // split-K accumulators, partial mask words and per-column state
            const int64_t grid = decode_grid(K, N);
            w.ramax_bits = reinterpret_cast<uint32_t*>(take(sizeof(uint32_t) * M));
            w.patch_pos = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * N));
            // split-tile partials: one [16 x 128] int32 slot per CTA
            w.c32_words = grid * 16 * 128;
            w.c32 = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * static_cast<size_t>(w.c32_words)));
            w.n_tiles = (N + 127) / 128;
            // split-tile partial slots (above) start empty and per-tile counters
            // zero (i8mm_linear_workspace_init); every decode call leaves them so
            w.tile_cnt = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * (w.n_tiles + 2)));
            w.thr_word = reinterpret_cast<uint32_t*>(w.tile_cnt + w.n_tiles + 1);
            w.wq_p = reinterpret_cast<int8_t*>(take(static_cast<size_t>(128 * w.ldq)));  // patch tile rows
        } else {
            w.wq_p = reinterpret_cast<int8_t*>(take(static_cast<size_t>(N * w.ldq)));
        }
    }
    if (!w.decode) w.rp_scratch = reinterpret_cast<void*>(take(row_prologue_scratch_bytes(M > 0 ? M : 1, K)));
    if (linear && !w.decode && swapab_route(M, K, N)) {
        w.sab_c32 = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * static_cast<size_t>(swapab_c32_words(M))));
        w.sab_cnt_words = swapab_cnt_words(N);
        w.sab_cnt = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * static_cast<size_t>(w.sab_cnt_words)));
    } else if (linear && !w.decode && gemm_split_factor(M, N, K) > 1) {
        w.sk_ld = gemm_split_cols(N, true);  // column-major partials: sk_ld columns x M rows
        w.sk_words = M * w.sk_ld + gemm_split_tiles(N, true);
        w.sk_c32 = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * static_cast<size_t>(w.sk_words)));
    }
    w.bytes = p - p0;
    return w;
}

// Prepared weight buffer of the weight-stationary linear layer.
struct WeightBuf {
    int8_t* wq_t;     // N x ldq codes with the full-column scale
    int8_t* q2;       // N x ldq codes with the second-candidate scale (patched columns)
    float* col_amax;  // N, amax over all K rows
    uint16_t* cand_v; // kTopT x N, |w| fp16 bits, descending
    int32_t* cand_r;  // kTopT x N, rows
    int64_t ldq;
    size_t bytes;
};

WeightBuf carve_weight(void* base, int64_t K, int64_t N) {
    WeightBuf b{};
    b.ldq = round_up(K, 16);
    uintptr_t p = reinterpret_cast<uintptr_t>(base);
    const uintptr_t p0 = p;
    auto take = [&](size_t bytes) {
        uintptr_t r = p;
        p += static_cast<uintptr_t>(round_up(static_cast<int64_t>(bytes), 256));
        return r;
    };
    b.wq_t = reinterpret_cast<int8_t*>(take(static_cast<size_t>(N * b.ldq)));
    b.q2 = reinterpret_cast<int8_t*>(take(static_cast<size_t>(N * b.ldq)));
    b.col_amax = reinterpret_cast<float*>(take(sizeof(float) * N));
    b.cand_v = reinterpret_cast<uint16_t*>(take(sizeof(uint16_t) * kTopT * N));
    b.cand_r = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * kTopT * N));
    b.bytes = p - p0;
    return b;
}
}  // namespace

size_t i8mm_llm_int8_workspace_size(int64_t M, int64_t K, int64_t N) {
    if (M < 0 || K <= 0 || N < 0) return 0;
    return carve(nullptr, M, K, N).bytes + 256;
}

int i8mm_llm_int8_matmul(const void* x, int64_t ldx, const void* w, int64_t ldw, int64_t M,
                         int64_t K, int64_t N, float alpha, void* y, int64_t ldy, int out_kind,
                         void* workspace, size_t workspace_bytes, int32_t* o_count_dev,
                         void* stream) {
    if (int s = check_device()) return s;
    if (int s = check_inner(K)) return s;
    if (!(alpha > 0.0f) || !std::isfinite(alpha)) return I8MM_ERR_ALPHA;
    if (M <= 0 || K <= 0 || N <= 0 || ldx < K || ldw < N || ldy < N || !x || !w || !y ||
        !workspace)
        return I8MM_ERR_ARGUMENT;
    void* base = reinterpret_cast<void*>(round_up(reinterpret_cast<intptr_t>(workspace), 256));
    Workspace ws = carve(base, M, K, N);
    if (ws.bytes + (static_cast<char*>(base) - static_cast<char*>(workspace)) > workspace_bytes)
        return I8MM_ERR_ARGUMENT;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const __half* xh = static_cast<const __half*>(x);
    const __half* wh = static_cast<const __half*>(w);
    cudaError_t e;
    // gemm.py:225 extract_outlier_columns
    // + gemm.py:242 rowwise over keep columns + gather of x[:, O] (gemm.py:238)
    if ((e = launch_row_prologue(xh, M, K, ldx, alpha, ws.mask, ws.o_idx, ws.o_count, ws.xq, ws.ldq,
                                 ws.row_amax, ws.xo, ws.o_cap, ws.rp_scratch, st, nullptr, ws.nonfinite)))
        return I8MM_ERR_CUDA;
    // gemm.py:243 colwise over keep rows, stored K-major
    if ((e = launch_quantize_cols_t(wh, K, N, ldw, ws.mask, ws.wq_t, ws.ldq, ws.col_amax, st)))
        return I8MM_ERR_CUDA;
    // compact copy of the outlier rows W[O, :] for the epilogue (gemm.py:238)
    if ((e = launch_gather_rows(wh, ldw, N, ws.o_idx, ws.o_count, ws.o_cap, ws.wo, round_up(N, 8), st)))
        return I8MM_ERR_CUDA;
    // gemm.py:193-194, 238, 244-247: int8 GEMM + dequant + outlier term
    int s = i8mm_gemm_dequant(ws.xq, ws.wq_t, ws.ldq, M, N, K, ws.row_amax, ws.col_amax, x, ldx, w,
                              ldw, ws.xo, ws.o_cap, ws.wo, round_up(N, 8), ws.o_idx, ws.o_count, y,
                              ldy, out_kind, stream);
    if (s) return s;
    if (o_count_dev) {
        if (cudaMemcpyAsync(o_count_dev, ws.o_count, sizeof(int32_t), cudaMemcpyDeviceToDevice,
                            st) != cudaSuccess)
            return I8MM_ERR_CUDA;
    }
    return I8MM_OK;
}

// The whole call plus the reference's NaN/Inf rejection of both operands
// (tensors.py:47-48) as one device word: X's flag from the scan, W's from one
// check pass (OR). One entry instead of a host round trip per stage.
int i8mm_llm_int8_matmul_checked(const void* x, int64_t ldx, const void* w, int64_t ldw, int64_t M,
                                 int64_t K, int64_t N, float alpha, void* y, int64_t ldy, int out_kind,
                                 void* workspace, size_t workspace_bytes, int32_t* o_count_dev,
                                 int32_t* nonfinite_dev, void* stream) {
    int s = i8mm_llm_int8_matmul(x, ldx, w, ldw, M, K, N, alpha, y, ldy, out_kind, workspace, workspace_bytes,
                                 o_count_dev, stream);
    if (s || nonfinite_dev == nullptr) return s;
    void* base = reinterpret_cast<void*>(round_up(reinterpret_cast<intptr_t>(workspace), 256));
    const Workspace ws = carve(base, M, K, N);
    if (cudaMemcpyAsync(nonfinite_dev, ws.nonfinite, sizeof(int32_t), cudaMemcpyDeviceToDevice,
                        static_cast<cudaStream_t>(stream)) != cudaSuccess)
        return I8MM_ERR_CUDA;
    return i8mm_f16_check(w, K, N, ldw, nonfinite_dev, stream);
}

// ---------------------------------------------------------------- linear layer
void i8mm_debug_set_pdl(int on) { g_pdl = on ? 1 : 0; }

void i8mm_debug_set_swapab(int on) { set_swapab(on); }

void i8mm_debug_swapab_timeline(void* stamps) {
    set_swapab_timeline(static_cast<unsigned long long*>(stamps));
}

void i8mm_debug_set_decode_max_m(int max_m) {
    g_decode_max_m = max_m < 0 ? 0 : (max_m > kDecodeMaxM ? kDecodeMaxM : max_m);
}

void i8mm_debug_decode_timeline(void* stamps) {
    set_decode_timeline(static_cast<unsigned long long*>(stamps));
}

int i8mm_linear_uses_decode(int64_t M, int64_t K, int64_t N) { return uses_decode(M, K, N) ? 1 : 0; }

size_t i8mm_linear_weight_bytes(int64_t K, int64_t N) {
    if (K <= 0 || N <= 0) return 0;
    return carve_weight(nullptr, K, N).bytes + 256;
}

size_t i8mm_linear_prepare_scratch_bytes(int64_t K, int64_t N) {
    if (K <= 0 || N <= 0) return 0;
    const int64_t rpb = topt_chunk_rows(K);
    const int64_t chunks = (K + rpb - 1) / rpb;
    return static_cast<size_t>(2 * chunks * kTopT * N) * sizeof(uint32_t) + 512;
}

int i8mm_linear_prepare(const void* w, int64_t ldw, int64_t K, int64_t N, void* wbuf,
                        size_t wbuf_bytes, void* scratch, size_t scratch_bytes, void* stream) {
    if (int s = check_device()) return s;
    if (int s = check_inner(K)) return s;
    if (K <= 0 || N <= 0 || ldw < N || !w || !wbuf || !scratch) return I8MM_ERR_ARGUMENT;
    void* base = reinterpret_cast<void*>(round_up(reinterpret_cast<intptr_t>(wbuf), 256));
    WeightBuf b = carve_weight(base, K, N);
    if (b.bytes + (static_cast<char*>(base) - static_cast<char*>(wbuf)) > wbuf_bytes)
        return I8MM_ERR_ARGUMENT;
    if (scratch_bytes < i8mm_linear_prepare_scratch_bytes(K, N)) return I8MM_ERR_ARGUMENT;
    const int64_t rpb = topt_chunk_rows(K);
    const int64_t chunks = (K + rpb - 1) / rpb;
    uint32_t* sv = reinterpret_cast<uint32_t*>(round_up(reinterpret_cast<intptr_t>(scratch), 256));
    int32_t* sr = reinterpret_cast<int32_t*>(sv + chunks * kTopT * N);
    return cuda_status(launch_weight_prepare(static_cast<const __half*>(w), K, N, ldw, b.wq_t, b.q2, b.ldq,
                                             b.col_amax, b.cand_v, b.cand_r, sv, sr,
                                             static_cast<cudaStream_t>(stream)));
}

size_t i8mm_linear_workspace_size(int64_t M, int64_t K, int64_t N) {
    if (M < 0 || K <= 0 || N <= 0) return 0;
    return carve(nullptr, M, K, N, true).bytes + 256;
}

static int linear_ws(void* workspace, size_t bytes, int64_t M, int64_t K, int64_t N, Workspace* ws) {
    void* base = reinterpret_cast<void*>(round_up(reinterpret_cast<intptr_t>(workspace), 256));
    *ws = carve(base, M, K, N, true);
    if (ws->bytes + (static_cast<char*>(base) - static_cast<char*>(workspace)) > bytes)
        return I8MM_ERR_ARGUMENT;
    return I8MM_OK;
}

static DecodeArgs decode_args(const Workspace& ws, const WeightBuf& b, const __half* x, int64_t ldx,
                              int64_t M, int64_t K, const __half* w, int64_t ldw, int64_t N,
                              float alpha, void* y, int64_t ldy) {
    DecodeArgs d{};
    d.x = x;
    d.ldx = ldx;
    d.M = M;
    d.K = K;
    d.N = N;
    d.x_vec = (ldx % 8 == 0) && ((reinterpret_cast<uintptr_t>(x) & 15u) == 0);
    d.thr_bits = alpha_threshold_bits(alpha);
    d.nonfinite = ws.nonfinite;
    d.mask = ws.mask;
    d.o_idx = ws.o_idx;
    d.o_count = ws.o_count;
    d.ramax_bits = ws.ramax_bits;
    d.row_amax = ws.row_amax;
    d.xq = ws.xq;
    d.ldq = ws.ldq;
    d.w = w;
    d.ldw = ldw;
    d.w_vec = (ldw % 8 == 0) && ((reinterpret_cast<uintptr_t>(w) & 15u) == 0);
    d.wq_t = b.wq_t;
    d.amax_full = b.col_amax;
    d.cand_v = b.cand_v;
    d.cand_r = b.cand_r;
    d.q2 = b.q2;
    d.c32 = ws.c32;
    d.y = y;
    d.ldy = ldy;
    return d;
}

int i8mm_linear_prologue(const void* x, int64_t ldx, int64_t M, const void* w, int64_t ldw,
                         const void* wbuf, int64_t K, int64_t N, float alpha, void* workspace,
                         size_t workspace_bytes, void* stream) {
    if (int s = check_device()) return s;
    if (int s = check_inner(K)) return s;
    if (!(alpha > 0.0f) || !std::isfinite(alpha)) return I8MM_ERR_ALPHA;
    if (M <= 0 || K <= 0 || N <= 0 || ldx < K || ldw < N || !x || !w || !wbuf || !workspace)
        return I8MM_ERR_ARGUMENT;
    Workspace ws;
    if (int s = linear_ws(workspace, workspace_bytes, M, K, N, &ws)) return s;
    const WeightBuf b = carve_weight(
        reinterpret_cast<void*>(round_up(reinterpret_cast<intptr_t>(wbuf), 256)), K, N);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const __half* xh = static_cast<const __half*>(x);
    const __half* wh = static_cast<const __half*>(w);
    // decode routing: the whole layer is one launch in i8mm_linear_gemm; the
    // prologue entry only records the threshold for it (i8mm_linear_forward
    // passes it directly and skips this launch)
    if (ws.decode) return cuda_status(launch_set_word(ws.thr_word, alpha_threshold_bits(alpha), st));
    // row side (+ the fixup counters zeroed in the same first launch), then
    // W[O, :] gather + column fixup in one launch, then the patched codes
    // zeroed with the mask: the split-K scratch, or the swap-AB GEMM's tile counters
    const PerCallFix fix{ws.sab_cnt != nullptr ? ws.sab_cnt : ws.sk_c32,
                         ws.sab_cnt != nullptr ? ws.sab_cnt_words : (ws.sk_c32 != nullptr ? ws.sk_words : 0), wh, K,
                         N, ldw, ws.wo, round_up(N, 8),
                         b.col_amax, b.cand_v, b.cand_r, b.q2, ws.p_count, ws.p_idx, ws.p_amax, ws.p_src,
                         ws.wq_p};
    if (launch_row_prologue(xh, M, K, ldx, alpha, ws.mask, ws.o_idx, ws.o_count, ws.xq, ws.ldq,
                            ws.row_amax, ws.xo, ws.o_cap, ws.rp_scratch, st, &fix, ws.nonfinite))
        return I8MM_ERR_CUDA;
    return I8MM_OK;
}

// GEMM + epilogue over rows [row0, row0 + rows) of a prologue's workspace
// (rows are independent once O and the row scales are known, gemm.py:210, 242)
struct PeerOut {  // fused output all-gather destinations (i8mm_linear_forward_peers)
    void* const* y;
    int n;
    int64_t ldy, col;
};

static int linear_gemm_rows_impl(const void* x, int64_t ldx, int64_t M, const void* w, int64_t ldw,
                                 const void* wbuf, int64_t K, int64_t N, void* y, int64_t ldy,
                                 int out_kind, void* workspace, size_t workspace_bytes, int64_t row0,
                                 int64_t rows, void* stream, const PeerOut* peers = nullptr) {
    if (int s = check_device()) return s;
    if (M <= 0 || K <= 0 || N <= 0 || ldy < N || !y || !wbuf || !workspace) return I8MM_ERR_ARGUMENT;
    if (row0 < 0 || rows < 0 || row0 + rows > M) return I8MM_ERR_ARGUMENT;
    Workspace ws;
    if (int s = linear_ws(workspace, workspace_bytes, M, K, N, &ws)) return s;
    const WeightBuf b = carve_weight(
        reinterpret_cast<void*>(round_up(reinterpret_cast<intptr_t>(wbuf), 256)), K, N);
    int epi, elt;
    switch (out_kind) {
        case I8MM_OUT_F16: epi = EPI_F16; elt = 2; break;
        case I8MM_OUT_F32: epi = EPI_F32; elt = 4; break;
        case I8MM_OUT_F32_EXACT: epi = EPI_F32_EXACT; elt = 4; break;
        default: return I8MM_ERR_ARGUMENT;
    }
    if (ws.decode) {
        if (row0 != 0 || rows != M) return I8MM_ERR_ARGUMENT;  // one launch for the whole call
        DecodeArgs d = decode_args(ws, b, static_cast<const __half*>(x), ldx, M, K,
                                   static_cast<const __half*>(w), ldw, N, 6.0f, y, ldy);
        d.thr_bits_dev = ws.thr_word;
        return cuda_status(launch_decode(d, epi, static_cast<cudaStream_t>(stream)));
    }
    if (rows == 0) return I8MM_OK;
    GemmArgs g{};
    g.a = ws.xq + row0 * ws.ldq;
    g.lda = ws.ldq;
    g.b = b.wq_t;
    g.ldb = b.ldq;
    g.M = rows;
    g.N = N;
    g.K = K;
    g.y = static_cast<char*>(y) + row0 * ldy * elt;
    g.ldy = ldy;
    g.row_amax = ws.row_amax + row0;
    g.col_amax = b.col_amax;
    g.x = static_cast<const __half*>(x) + row0 * ldx;
    g.ldx = ldx;
    g.w = static_cast<const __half*>(w);
    g.ldw = ldw;
    g.xo = ws.xo + row0 * ws.o_cap;
    g.o_cap = ws.o_cap;
    g.o_idx = ws.o_idx;
    g.o_count = ws.o_count;
    g.wo = ws.wo;
    g.ldwo = round_up(N, 8);
    g.wo_cap = ws.o_cap;
    // patched columns (their amax over keep rows differs from the cached one)
    // run as extra tiles of the same launch
    g.b_patch = ws.wq_p;
    g.patch_count = ws.p_count;
    g.patch_idx = ws.p_idx;
    g.patch_amax = ws.p_amax;
    g.patch_mask = reinterpret_cast<const uint32_t*>(ws.p_count) + 4;
    if (peers != nullptr && peers->n > 0) {
        if (peers->n > kMaxPeers || epi != EPI_F16) return I8MM_ERR_ARGUMENT;
        g.n_peer = peers->n;
        for (int q = 0; q < peers->n; ++q)
            g.y_peer[q] = static_cast<char*>(peers->y[q]) + row0 * peers->ldy * 2;
        g.peer_ldy = peers->ldy;
        g.peer_col = peers->col;
    }
    // mid-size M, whole call: the swap-AB stream-K GEMM (swapab_sm100.cu)
    if (ws.sab_cnt != nullptr && row0 == 0 && rows == M && g.n_peer == 0 && (epi == EPI_F16 || epi == EPI_F32))
        return cuda_status(launch_swapab(g, ws.sab_c32, ws.sab_cnt, epi, static_cast<cudaStream_t>(stream)));
    if (ws.sk_c32 != nullptr && row0 == 0 && rows == M) {  // split-K scratch (zeroed by the prologue)
        g.c32 = ws.sk_c32;
        g.c32_rows = M;
        g.c32_cnt = ws.sk_c32 + M * ws.sk_ld;
        g.c32_tiles = gemm_split_tiles(N, true);
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (launch_gemm_sm100(g, epi, st) != cudaSuccess) return I8MM_ERR_CUDA;
    return I8MM_OK;
}

int i8mm_linear_forward_peers(const void* x, int64_t ldx, int64_t M, const void* w, int64_t ldw,
                              const void* wbuf, int64_t K, int64_t N, float alpha, void* y, int64_t ldy,
                              void* workspace, size_t workspace_bytes, void* const* y_peers, int n_peers,
                              int64_t ldy_peer, int64_t col_off, void* stream) {
    if (n_peers < 0 || n_peers > kMaxPeers || (n_peers > 0 && y_peers == nullptr) || col_off < 0 ||
        ldy_peer < col_off + N)
        return I8MM_ERR_ARGUMENT;
    for (int q = 0; q < n_peers; ++q)
        if (y_peers[q] == nullptr) return I8MM_ERR_ARGUMENT;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (uses_decode(M, K, N)) {  // one decode launch, then copy-engine stores of the block to the peers
        int s = i8mm_linear_forward(x, ldx, M, w, ldw, wbuf, K, N, alpha, y, ldy, I8MM_OUT_F16, workspace,
                                    workspace_bytes, nullptr, stream);
        if (s) return s;
        for (int q = 0; q < n_peers; ++q)
            if (cudaMemcpy2DAsync(static_cast<char*>(y_peers[q]) + col_off * 2, ldy_peer * 2, y, ldy * 2, N * 2, M,
                                  cudaMemcpyDeviceToDevice, st) != cudaSuccess)
                return I8MM_ERR_CUDA;
        return I8MM_OK;
    }
    int s = i8mm_linear_prologue(x, ldx, M, w, ldw, wbuf, K, N, alpha, workspace, workspace_bytes, stream);
    if (s) return s;
    const PeerOut peers{y_peers, n_peers, ldy_peer, col_off};
    return linear_gemm_rows_impl(x, ldx, M, w, ldw, wbuf, K, N, y, ldy, I8MM_OUT_F16, workspace,
                                 workspace_bytes, 0, M, stream, &peers);
}

int i8mm_linear_gemm(const void* x, int64_t ldx, int64_t M, const void* w, int64_t ldw,
                     const void* wbuf, int64_t K, int64_t N, void* y, int64_t ldy, int out_kind,
                     void* workspace, size_t workspace_bytes, void* stream) {
    return linear_gemm_rows_impl(x, ldx, M, w, ldw, wbuf, K, N, y, ldy, out_kind, workspace,
                                 workspace_bytes, 0, M, stream);
}

int i8mm_linear_gemm_rows(const void* x, int64_t ldx, int64_t M, const void* w, int64_t ldw,
                          const void* wbuf, int64_t K, int64_t N, void* y, int64_t ldy, int out_kind,
                          void* workspace, size_t workspace_bytes, int64_t row0, int64_t rows,
                          void* stream) {
    return linear_gemm_rows_impl(x, ldx, M, w, ldw, wbuf, K, N, y, ldy, out_kind, workspace,
                                 workspace_bytes, row0, rows, stream);
}

int i8mm_linear_forward(const void* x, int64_t ldx, int64_t M, const void* w, int64_t ldw,
                        const void* wbuf, int64_t K, int64_t N, float alpha, void* y, int64_t ldy,
                        int out_kind, void* workspace, size_t workspace_bytes,
                        int32_t* o_count_dev, void* stream) {
    if (uses_decode(M, K, N)) {  // decode routing: one launch
        if (int s = check_device()) return s;
        if (int s = check_inner(K)) return s;
        if (!(alpha > 0.0f) || !std::isfinite(alpha)) return I8MM_ERR_ALPHA;
        if (K <= 0 || N <= 0 || ldx < K || ldw < N || ldy < N || !x || !w || !y || !wbuf ||
            !workspace)
            return I8MM_ERR_ARGUMENT;
        int epi;
        switch (out_kind) {
            case I8MM_OUT_F16: epi = EPI_F16; break;
            case I8MM_OUT_F32: epi = EPI_F32; break;
            case I8MM_OUT_F32_EXACT: epi = EPI_F32_EXACT; break;
            default: return I8MM_ERR_ARGUMENT;
        }
        Workspace ws;
        if (int s = linear_ws(workspace, workspace_bytes, M, K, N, &ws)) return s;
        const WeightBuf b = carve_weight(
            reinterpret_cast<void*>(round_up(reinterpret_cast<intptr_t>(wbuf), 256)), K, N);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const DecodeArgs d = decode_args(ws, b, static_cast<const __half*>(x), ldx, M, K,
                                         static_cast<const __half*>(w), ldw, N, alpha, y, ldy);
        if (launch_decode(d, epi, st) != cudaSuccess) return I8MM_ERR_CUDA;
        if (o_count_dev && cudaMemcpyAsync(o_count_dev, ws.o_count, sizeof(int32_t),
                                           cudaMemcpyDeviceToDevice, st) != cudaSuccess)
            return I8MM_ERR_CUDA;
        return I8MM_OK;
    }
    int s = i8mm_linear_prologue(x, ldx, M, w, ldw, wbuf, K, N, alpha, workspace, workspace_bytes,
                                 stream);
    if (s) return s;
    s = i8mm_linear_gemm(x, ldx, M, w, ldw, wbuf, K, N, y, ldy, out_kind, workspace,
                         workspace_bytes, stream);
    if (s) return s;
    if (o_count_dev) {
        Workspace ws;
        linear_ws(workspace, workspace_bytes, M, K, N, &ws);
        if (cudaMemcpyAsync(o_count_dev, ws.o_count, sizeof(int32_t), cudaMemcpyDeviceToDevice,
                            static_cast<cudaStream_t>(stream)) != cudaSuccess)
            return I8MM_ERR_CUDA;
    }
    return I8MM_OK;
}

// Device pointers into a linear-layer workspace (for tests / introspection).
int i8mm_linear_workspace_views(void* workspace, int64_t M, int64_t K, int64_t N, void** views,
                                int n_views) {
    if (!workspace || !views || n_views < 8) return I8MM_ERR_ARGUMENT;
    void* base = reinterpret_cast<void*>(round_up(reinterpret_cast<intptr_t>(workspace), 256));
    Workspace ws = carve(base, M, K, N, true);
    views[0] = ws.o_count;  // int32 |O|
    views[1] = ws.o_idx;    // int32 [K]
    views[2] = ws.xq;       // int8 [M x ldq]
    views[3] = ws.row_amax; // float [M]
    views[4] = ws.p_count;  // int32 patched-column count
    views[5] = ws.p_idx;    // int32 [N]
    views[6] = ws.p_amax;   // float [N]
    views[7] = ws.wq_p;     // int8 [N x ldq]
    return I8MM_OK;
}

int i8mm_linear_workspace_init(void* workspace, size_t workspace_bytes, int64_t M, int64_t K, int64_t N,
                               void* stream) {
    if (!workspace || M <= 0 || K <= 0 || N <= 0) return I8MM_ERR_ARGUMENT;
    Workspace ws;
    if (int s = linear_ws(workspace, workspace_bytes, M, K, N, &ws)) return s;
    if (!ws.decode) return I8MM_OK;  // the prefill routing zeroes its counters every call
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // split-tile partial slots start empty (byte 0x80: dec::kPartEmpty); every
    // decode call leaves them empty and its counters zero
    if (cudaMemsetAsync(ws.c32, 0x80, sizeof(int32_t) * static_cast<size_t>(ws.c32_words), st) != cudaSuccess)
        return I8MM_ERR_CUDA;
    return cuda_status(cudaMemsetAsync(ws.tile_cnt, 0, sizeof(int32_t) * (ws.n_tiles + 2), st));
}

int i8mm_linear_patch_stats(const void* w, int64_t ldw, const void* wbuf, int64_t M, int64_t K, int64_t N,
                            void* workspace, size_t workspace_bytes, void* stream) {
    if (!w || !wbuf || !workspace || M <= 0 || K <= 0 || N <= 0 || ldw < N) return I8MM_ERR_ARGUMENT;
    Workspace ws;
    if (int s = linear_ws(workspace, workspace_bytes, M, K, N, &ws)) return s;
    if (!ws.decode) return I8MM_OK;  // the prefill prologue wrote the patch list
    const WeightBuf b = carve_weight(reinterpret_cast<void*>(round_up(reinterpret_cast<intptr_t>(wbuf), 256)), K, N);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // the decode kernel decides patched columns per tile; the list the prefill
    // prologue publishes (weights.cu fixup) is recomputed here from its mask / O
    if (cudaMemsetAsync(ws.p_count, 0, sizeof(int32_t) * fixup_zero_words(N), st) != cudaSuccess)
        return I8MM_ERR_CUDA;
    return cuda_status(launch_gather_fixup(static_cast<const __half*>(w), K, N, ldw, ws.mask, ws.o_idx, ws.o_count,
                                           ws.o_cap, ws.wo, round_up(N, 8), b.col_amax, b.cand_v, b.cand_r,
                                           ws.p_count, ws.p_idx, ws.p_amax, ws.p_src, st));
}

int i8mm_linear_weight_views(void* wbuf, int64_t K, int64_t N, void** views, int n_views) {
    if (!wbuf || !views || n_views < 4) return I8MM_ERR_ARGUMENT;
    if (n_views >= 5)
        views[4] = carve_weight(reinterpret_cast<void*>(round_up(reinterpret_cast<intptr_t>(wbuf), 256)),
                                K, N).q2;
    WeightBuf b = carve_weight(reinterpret_cast<void*>(round_up(reinterpret_cast<intptr_t>(wbuf), 256)),
                               K, N);
    views[0] = b.wq_t;
    views[1] = b.col_amax;
    views[2] = b.cand_v;
    views[3] = b.cand_r;
    return I8MM_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- sibling schemes
// Tensor-wise absmax / zeropoint pipelines (quantize.py:120-171,
// gemm.py:85-104, 150-187) on the same tcgen05 int8 GEMM.
namespace {
struct ScalarWs {
    int8_t* xq;
    int8_t* wq_t;
    int32_t* c;
    int32_t* stats;   // 2 x 4 int32
    float* fstats;    // 2 x 4 floats: [amax, min, max, -]
    int32_t* rowsum;  // M
    int32_t* colsum;  // N
    int32_t* flag;    // overflow
    int64_t ldq;
    size_t bytes;
};
ScalarWs carve_scalar(void* base, int64_t M, int64_t K, int64_t N) {
    ScalarWs w{};
    w.ldq = round_up(K, 16);
    uintptr_t p = reinterpret_cast<uintptr_t>(base);
    const uintptr_t p0 = p;
    auto take = [&](size_t bytes) {
        uintptr_t r = p;
        p += static_cast<uintptr_t>(round_up(static_cast<int64_t>(bytes), 256));
        return r;
    };
    w.xq = reinterpret_cast<int8_t*>(take(static_cast<size_t>(M * w.ldq)));
    w.wq_t = reinterpret_cast<int8_t*>(take(static_cast<size_t>(N * w.ldq)));
    w.c = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * static_cast<size_t>(M * N)));
    w.stats = reinterpret_cast<int32_t*>(take(8 * sizeof(int32_t)));
    w.fstats = reinterpret_cast<float*>(take(8 * sizeof(float)));
    w.rowsum = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * M));
    w.colsum = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * N));
    w.flag = reinterpret_cast<int32_t*>(take(sizeof(int32_t)));
    w.bytes = p - p0;
    return w;
}

double rha(double v) { return std::copysign(std::floor(std::fabs(v) + 0.5), v); }
}  // namespace

extern "C" {

int i8mm_tensor_stats(const void* x, int64_t rows, int64_t cols, int64_t ld, int32_t* scratch,
                      float* out3, void* stream) {
    if (int s = check_device()) return s;
    if (rows <= 0 || cols <= 0 || ld < cols || !x || !scratch || !out3) return I8MM_ERR_ARGUMENT;
    return cuda_status(launch_tensor_stats(static_cast<const __half*>(x), rows, cols, ld, scratch, out3,
                                           static_cast<cudaStream_t>(stream)));
}

int i8mm_absmax_quantize(const void* x, int64_t rows, int64_t cols, int64_t ld, const float* amax,
                         int8_t* q, int64_t ldq, int transpose, void* stream) {
    if (int s = check_device()) return s;
    const int64_t need = transpose ? rows : cols;
    if (rows <= 0 || cols <= 0 || ld < cols || ldq < need || !x || !amax || !q) return I8MM_ERR_ARGUMENT;
    return cuda_status(launch_quantize_scalar(static_cast<const __half*>(x), rows, cols, ld, 0, amax, 0.0, 0,
                                              q, ldq, transpose, static_cast<cudaStream_t>(stream)));
}

int i8mm_zeropoint_params(float lo, float hi, double* nd, int32_t* zp, double* offset) {
    if (!nd || !zp || !offset) return I8MM_ERR_ARGUMENT;
    if (hi == lo) {  // quantize.py:156-160: constant tensor -> offset, nd 1, zp 0
        *nd = 1.0;
        *zp = 0;
        *offset = static_cast<double>(lo);
        return I8MM_OK;
    }
    const double n = 254.0 / (static_cast<double>(hi) - static_cast<double>(lo));
    const double z = rha(n * static_cast<double>(lo)) + 127.0;  // quantize.py:162
    if (!(z >= -32768.0 && z <= 32767.0)) return I8MM_ERR_ZEROPOINT;
    *nd = n;
    *zp = static_cast<int32_t>(z);
    *offset = 0.0;
    return I8MM_OK;
}

int i8mm_zeropoint_quantize(const void* x, int64_t rows, int64_t cols, int64_t ld, double nd, int32_t zp,
                            int8_t* q, int64_t ldq, int transpose, void* stream) {
    if (int s = check_device()) return s;
    const int64_t need = transpose ? rows : cols;
    if (rows <= 0 || cols <= 0 || ld < cols || ldq < need || !x || !q || !(nd > 0.0)) return I8MM_ERR_ARGUMENT;
    return cuda_status(launch_quantize_scalar(static_cast<const __half*>(x), rows, cols, ld, 1, nullptr, nd, zp,
                                              q, ldq, transpose, static_cast<cudaStream_t>(stream)));
}

// float32-operand forms (the reference's DenseMatrix is float32, tensors.py:31-49)
int i8mm_tensor_stats_f32(const float* x, int64_t rows, int64_t cols, int64_t ld, int32_t* scratch,
                          float* out3, void* stream) {
    if (int s = check_device()) return s;
    if (rows <= 0 || cols <= 0 || ld < cols || !x || !scratch || !out3) return I8MM_ERR_ARGUMENT;
    return cuda_status(launch_tensor_stats(x, rows, cols, ld, scratch, out3, static_cast<cudaStream_t>(stream)));
}

int i8mm_absmax_quantize_f32(const float* x, int64_t rows, int64_t cols, int64_t ld, const float* amax,
                             int8_t* q, int64_t ldq, int transpose, void* stream) {
    if (int s = check_device()) return s;
    const int64_t need = transpose ? rows : cols;
    if (rows <= 0 || cols <= 0 || ld < cols || ldq < need || !x || !amax || !q) return I8MM_ERR_ARGUMENT;
    return cuda_status(launch_quantize_scalar(x, rows, cols, ld, 0, amax, 0.0, 0, q, ldq, transpose,
                                              static_cast<cudaStream_t>(stream)));
}

int i8mm_zeropoint_quantize_f32(const float* x, int64_t rows, int64_t cols, int64_t ld, double nd, int32_t zp,
                                int8_t* q, int64_t ldq, int transpose, void* stream) {
    if (int s = check_device()) return s;
    const int64_t need = transpose ? rows : cols;
    if (rows <= 0 || cols <= 0 || ld < cols || ldq < need || !x || !q || !(nd > 0.0)) return I8MM_ERR_ARGUMENT;
    return cuda_status(launch_quantize_scalar(x, rows, cols, ld, 1, nullptr, nd, zp, q, ldq, transpose,
                                              static_cast<cudaStream_t>(stream)));
}

int i8mm_rowsum_i8(const int8_t* q, int64_t rows, int64_t cols, int64_t ld, int32_t* out, void* stream) {
    if (int s = check_device()) return s;
    if (rows < 0 || cols < 0 || ld < cols || !q || !out) return I8MM_ERR_ARGUMENT;
    return cuda_status(launch_rowsum_i8(q, rows, cols, ld, out, static_cast<cudaStream_t>(stream)));
}

int i8mm_dequantize_absmax(const int32_t* c, int64_t M, int64_t N, int64_t ldc, const float* amax_x,
                           const float* amax_w, float* out, int64_t ldo, void* stream) {
    if (int s = check_device()) return s;
    if (M <= 0 || N <= 0 || ldc < N || ldo < N || !c || !amax_x || !amax_w || !out) return I8MM_ERR_ARGUMENT;
    return cuda_status(launch_dequant_absmax(c, M, N, ldc, amax_x, amax_w, out, ldo,
                                             static_cast<cudaStream_t>(stream)));
}

int i8mm_zeropoint_combine(const int32_t* c, int64_t M, int64_t N, int64_t ldc, const int32_t* rowsum_a,
                           const int32_t* colsum_b, int64_t K, int32_t zp_a, int32_t zp_b, double nd_a,
                           double nd_b, double off_a, double off_b, float* out, int64_t ldo,
                           int32_t* acc_out, int32_t* overflow, void* stream) {
    if (int s = check_device()) return s;
    if (M <= 0 || N <= 0 || ldc < N || !c || !rowsum_a || !colsum_b || !overflow || (out && ldo < N))
        return I8MM_ERR_ARGUMENT;
    return cuda_status(launch_zeropoint_combine(c, M, N, ldc, rowsum_a, colsum_b, K, zp_a, zp_b, nd_a, nd_b,
                                                off_a, off_b, out, ldo, acc_out, overflow,
                                                static_cast<cudaStream_t>(stream)));
}

size_t i8mm_scalar_workspace_size(int64_t M, int64_t K, int64_t N) {
    if (M <= 0 || K <= 0 || N <= 0) return 0;
    return carve_scalar(nullptr, M, K, N).bytes + 256;
}

static int scalar_ws(void* workspace, size_t bytes, int64_t M, int64_t K, int64_t N, ScalarWs* ws) {
    void* base = reinterpret_cast<void*>(round_up(reinterpret_cast<intptr_t>(workspace), 256));
    *ws = carve_scalar(base, M, K, N);
    if (ws->bytes + (static_cast<char*>(base) - static_cast<char*>(workspace)) > bytes)
        return I8MM_ERR_ARGUMENT;
    return I8MM_OK;
}

static int gemm_codes(const ScalarWs& ws, int64_t M, int64_t K, int64_t N, cudaStream_t st) {
    GemmArgs g{};
    g.a = ws.xq;
    g.lda = ws.ldq;
    g.b = ws.wq_t;
    g.ldb = ws.ldq;
    g.M = M;
    g.N = N;
    g.K = K;
    g.y = ws.c;
    g.ldy = N;
    return launch_gemm_sm100(g, EPI_I32, st) == cudaSuccess ? I8MM_OK : I8MM_ERR_CUDA;
}

// absmax_matmul (gemm.py:150-156): never synchronizes the host
int i8mm_absmax_matmul(const void* x, int64_t ldx, const void* w, int64_t ldw, int64_t M, int64_t K,
                       int64_t N, float* y, int64_t ldy, void* workspace, size_t workspace_bytes,
                       void* stream) {
    if (int s = check_device()) return s;
    if (int s = check_inner(K)) return s;
    if (M <= 0 || K <= 0 || N <= 0 || ldx < K || ldw < N || ldy < N || !x || !w || !y || !workspace)
        return I8MM_ERR_ARGUMENT;
    ScalarWs ws;
    if (int s = scalar_ws(workspace, workspace_bytes, M, K, N, &ws)) return s;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const __half* xh = static_cast<const __half*>(x);
    const __half* wh = static_cast<const __half*>(w);
    if (launch_tensor_stats(xh, M, K, ldx, ws.stats, ws.fstats, st)) return I8MM_ERR_CUDA;
    if (launch_tensor_stats(wh, K, N, ldw, ws.stats + 4, ws.fstats + 4, st)) return I8MM_ERR_CUDA;
    if (launch_quantize_scalar(xh, M, K, ldx, 0, ws.fstats, 0.0, 0, ws.xq, ws.ldq, 0, st)) return I8MM_ERR_CUDA;
    if (launch_quantize_scalar(wh, K, N, ldw, 0, ws.fstats + 4, 0.0, 0, ws.wq_t, ws.ldq, 1, st))
        return I8MM_ERR_CUDA;
    if (int s = gemm_codes(ws, M, K, N, st)) return s;
    return cuda_status(launch_dequant_absmax(ws.c, M, N, N, ws.fstats, ws.fstats + 4, y, ldy, st));
}

// zeropoint_matmul (gemm.py:159-187). The zeropoints are validated on the host
// exactly as quantize.py:162-166 and the int32 range as gemm.py:71-75, so this
// entry synchronizes the stream twice (after the min/max pass and at the end).
int i8mm_zeropoint_matmul(const void* x, int64_t ldx, const void* w, int64_t ldw, int64_t M, int64_t K,
                          int64_t N, float* y, int64_t ldy, void* workspace, size_t workspace_bytes,
                          void* stream) {
    if (int s = check_device()) return s;
    if (int s = check_inner(K)) return s;
    if (M <= 0 || K <= 0 || N <= 0 || ldx < K || ldw < N || ldy < N || !x || !w || !y || !workspace)
        return I8MM_ERR_ARGUMENT;
    ScalarWs ws;
    if (int s = scalar_ws(workspace, workspace_bytes, M, K, N, &ws)) return s;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const __half* xh = static_cast<const __half*>(x);
    const __half* wh = static_cast<const __half*>(w);
    if (launch_tensor_stats(xh, M, K, ldx, ws.stats, ws.fstats, st)) return I8MM_ERR_CUDA;
    if (launch_tensor_stats(wh, K, N, ldw, ws.stats + 4, ws.fstats + 4, st)) return I8MM_ERR_CUDA;
    float h[8];
    if (cudaMemcpyAsync(h, ws.fstats, sizeof(h), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        return I8MM_ERR_CUDA;
    double nd_x, nd_w, off_x, off_w;
    int32_t zp_x, zp_w;
    if (int s = i8mm_zeropoint_params(h[1], h[2], &nd_x, &zp_x, &off_x)) return s;
    if (int s = i8mm_zeropoint_params(h[5], h[6], &nd_w, &zp_w, &off_w)) return s;
    if (off_x != 0.0 || h[1] == h[2]) {
        if (cudaMemsetAsync(ws.xq, 0, static_cast<size_t>(M * ws.ldq), st) != cudaSuccess) return I8MM_ERR_CUDA;
    } else if (launch_quantize_scalar(xh, M, K, ldx, 1, nullptr, nd_x, zp_x, ws.xq, ws.ldq, 0, st)) {
        return I8MM_ERR_CUDA;
    }
    if (off_w != 0.0 || h[5] == h[6]) {
        if (cudaMemsetAsync(ws.wq_t, 0, static_cast<size_t>(N * ws.ldq), st) != cudaSuccess) return I8MM_ERR_CUDA;
    } else if (launch_quantize_scalar(wh, K, N, ldw, 1, nullptr, nd_w, zp_w, ws.wq_t, ws.ldq, 1, st)) {
        return I8MM_ERR_CUDA;
    }
    if (int s = gemm_codes(ws, M, K, N, st)) return s;
    if (launch_rowsum_i8(ws.xq, M, K, ws.ldq, ws.rowsum, st)) return I8MM_ERR_CUDA;
    if (launch_rowsum_i8(ws.wq_t, N, K, ws.ldq, ws.colsum, st)) return I8MM_ERR_CUDA;
    if (cudaMemsetAsync(ws.flag, 0, sizeof(int32_t), st) != cudaSuccess) return I8MM_ERR_CUDA;
    if (launch_zeropoint_combine(ws.c, M, N, N, ws.rowsum, ws.colsum, K, zp_x, zp_w, nd_x, nd_w, off_x, off_w,
                                 y, ldy, nullptr, ws.flag, st))
        return I8MM_ERR_CUDA;
    int32_t flag = 0;
    if (cudaMemcpyAsync(&flag, ws.flag, sizeof(flag), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        return I8MM_ERR_CUDA;
    return flag ? I8MM_ERR_OVERFLOW : I8MM_OK;
}

}  // extern "C"
