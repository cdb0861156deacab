// Decode path of the weight-stationary LLM.int8() linear layer (SURVEY.md 8f
// rank 2, config 3: M = 1..256 tokens). At these sizes the layer is bound by
// the stream of int8 weights from HBM (K*N bytes per call), so the design is
// ONE cooperative launch (one CTA per SM) that keeps HBM busy from its first
// cycle: the TMA producer starts streaming weight tiles into the shared-memory
// ring before the activation prologue has even run, and the remaining per-call
// work (patched columns) runs on otherwise idle warps under the weight stream.
//
// Same arithmetic as the prefill path, so outputs are bit-identical to it:
//   Xq / row amax / outlier set  : prologue.cu semantics (quantize.py:168-179,
//                                   gemm.py:203-211, 242)
//   column scales                : weights.cu weight-stationary fixup
//                                   (quantize.py:182-187 on w[keep, :])
//   epilogue                     : gemm_sm100.cu (gemm.py:120-147, 238, 244-247)
//
// decode_fused_kernel (256 threads, grid = #SMs, cooperative):
//   W0  barriers, TMEM, and thread 0 issues the weight (A operand) TMA loads
//       of the first ring stages; their token (B operand) halves follow later
//   P1  zero the per-call state; outlier scan of 16-row x 128-column items
//       into partial mask words (no atomics, no pre-zeroed memory)   grid.sync
//   P2  CTA 0: final mask + sorted outlier list (gemm.py:211); the others:
//       row absmax over keep columns (atomicMax on fp16 bits)        grid.sync
//   P3  row codes (fast exact rounding, quant_common.cuh) and the column
//       fixup -> patched columns (amax changed because the cached
//       maximiser is an outlier row)                                 grid.sync
//   then, concurrently:
//   warp 0  TMA producer: token tiles for the prefilled stages, then both
//   warp 1  MMA: D[n, m] += WqT[n, k] Xq[m, k]  (tcgen05 kind::i8, swap-AB:
//           M = 128 weight rows, N = tokens padded to 16, K = 32)
//   warps 2-7  patched columns: re-derived codes dotted with Xq (exact int32
//           atomics into the workspace)
//   warps 4-7  epilogue, one thread per weight row n: dequant + outlier term,
//           stores coalesced along n
// The (n-tile, k-block) space is split evenly over the CTAs (stream-K); tiles
// split between CTAs reduce exactly through int32 red.add, and the CTA that
// completes a tile runs its epilogue.
#include <cooperative_groups.h>
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <mutex>

#include "kernels.cuh"
#include "quant_common.cuh"
#include "sm100_ptx.cuh"

namespace cg = cooperative_groups;

namespace i8mm {

bool make_tmap_i8_rows(CUtensorMap* map, const int8_t* base, int64_t rows, int64_t K, int64_t ld,
                       int box_rows);  // gemm_sm100.cu

namespace dec {

constexpr int THREADS = 256;    // warp 0 TMA, 1 MMA, 2 TMEM alloc, 2-7 patches, 4-7 epilogue
constexpr int NWARPS = THREADS / 32;
constexpr int ITEM_ROWS = 16;   // rows per scan / quantize item (one warp)
constexpr int ITEM_COLS = 128;  // columns per item: 16 lanes x 8 halves, 2 row parities
constexpr int WO_CAP = 16;      // outlier rows of W held in registers by the epilogue
constexpr int TILE_N = 128;     // weight rows per tile (the MMA's M)
constexpr int BK = 128;         // K bytes per stage (one SWIZZLE_128B row)
constexpr int UMMA_K = 32;
constexpr int MAX_STAGES = 12;
constexpr int A_BYTES = TILE_N * BK;
constexpr uint32_t TMEM_COLS = 512;  // two accumulators at column 0 and 256
constexpr int MAX_M = 256;
constexpr int LOCAL_CAP = 512;  // fixup columns per CTA (N <= LOCAL_CAP * grid)
constexpr int PATCH_ROWS = 128; // patched columns handled by the extra tile of the stream
// the first PT_GATHER_ROWS rows of the patch tile are gathered from q2 (tile::gather4)
// after the barrier; the rest (many patches) are copied to pq in P2 and box-loaded
constexpr int PT_GATHER_ROWS = 8;

__device__ __forceinline__ bool bit_of(const uint32_t* m, int64_t k) {
    return (m[k >> 5] >> (k & 31)) & 1u;
}
__device__ __forceinline__ float hbits_to_float(uint32_t b) {
    return __half2float(__ushort_as_half(static_cast<unsigned short>(b)));
}
__device__ __forceinline__ float amax_or_127(float a) { return a == 0.0f ? 127.0f : a; }

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// timeline stamp i of this CTA (dev tool: i8mm_debug_decode_timeline)
// (dev build only: see gemm_sm100.cu, I8MM_GEMM_DEVTOOLS)
#ifdef I8MM_GEMM_DEVTOOLS
constexpr bool kDevStamps = true;
#else
constexpr bool kDevStamps = false;
#endif
#define DSTAMP(ptr, i)                                                               \
    do {                                                                             \
        if (kDevStamps && (ptr) != nullptr) (ptr)[blockIdx.x * 16 + (i)] = gtimer(); \
    } while (0)

__device__ __forceinline__ void st_release(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// 8 consecutive fp16 of a row starting at `col` (zeros past K); 16-byte load
// when the row is aligned, element loads otherwise.
__device__ __forceinline__ uint4 load8(const __half* row, int64_t col, int64_t K, bool vec) {
    if (vec && col + 8 <= K) return ld_stream_u4(row + col);
    uint32_t h[8];
#pragma unroll
    for (int e = 0; e < 8; ++e)
        h[e] = col + e < K ? static_cast<uint32_t>(__half_as_ushort(row[col + e])) : 0u;
    return make_uint4(h[0] | h[1] << 16, h[2] | h[3] << 16, h[4] | h[5] << 16, h[6] | h[7] << 16);
}

// one block: prefix popcount over the mask words, sorted outlier indices
__device__ void compact_block(const uint32_t* __restrict__ mask, int64_t nwords,
                              int32_t* __restrict__ o_idx, int32_t* __restrict__ o_count,
                              int32_t* warp_sums) {
    const int64_t per = (static_cast<uint32_t>(nwords) + blockDim.x - 1) / blockDim.x;
    const int64_t w0 = threadIdx.x * per;
    const int64_t w1 = w0 + per < nwords ? w0 + per : nwords;
    int32_t local = 0;
    for (int64_t w = w0; w < w1; ++w) local += __popc(mask[w]);
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
        int32_t s = lane < nw ? warp_sums[lane] : 0;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int32_t t = __shfl_up_sync(0xffffffffu, s, d);
            if (lane >= d) s += t;
        }
        if (lane < nw) warp_sums[lane] = s;
    }
    __syncthreads();
    int32_t pos = incl - local + (wid > 0 ? warp_sums[wid - 1] : 0);
    for (int64_t w = w0; w < w1; ++w) {
        uint32_t m = mask[w];
        while (m) {
            const int b = __ffs(m) - 1;
            m &= m - 1;
            o_idx[pos++] = static_cast<int32_t>((w << 5) + b);
        }
    }
    if (threadIdx.x == blockDim.x - 1) *o_count = pos;
}

// same scan, but only the first WO_CAP indices (to shared memory) and the count
__device__ void compact_block_smem(const uint32_t* __restrict__ mask, int64_t nwords, int32_t* o_s,
                                   int32_t* n_s, int32_t* warp_sums) {
    const int64_t per = (static_cast<uint32_t>(nwords) + blockDim.x - 1) / blockDim.x;
    const int64_t w0 = threadIdx.x * per;
    const int64_t w1 = w0 + per < nwords ? w0 + per : nwords;
    int32_t local = 0;
    for (int64_t w = w0; w < w1; ++w) local += __popc(__ldcg(mask + w));
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
        int32_t s = lane < nw ? warp_sums[lane] : 0;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int32_t t = __shfl_up_sync(0xffffffffu, s, d);
            if (lane >= d) s += t;
        }
        if (lane < nw) warp_sums[lane] = s;
    }
    __syncthreads();
    int32_t pos = incl - local + (wid > 0 ? warp_sums[wid - 1] : 0);
    for (int64_t w = w0; w < w1 && pos < WO_CAP; ++w) {
        uint32_t m = __ldcg(mask + w);
        while (m && pos < WO_CAP) {
            const int b = __ffs(m) - 1;
            m &= m - 1;
            o_s[pos++] = static_cast<int32_t>((w << 5) + b);
        }
    }
    if (threadIdx.x == blockDim.x - 1) *n_s = incl + (wid > 0 ? warp_sums[wid - 1] : 0);
}

struct __align__(8) Bars {
    uint64_t full[MAX_STAGES];
    uint64_t empty[MAX_STAGES];
    uint64_t tmem_full[2];
    uint64_t tmem_empty[2];
    uint32_t tmem_slot;
    int32_t finisher;
    int32_t n_out;
    int32_t o_s[WO_CAP];            // first outlier columns (this CTA's compaction)
    int32_t n_local;                // patched columns found in this CTA's fixup range:
    int32_t local_j[LOCAL_CAP];     //   column,
    int32_t local_p[LOCAL_CAP];     //   patch index (row of the patch tile),
    float local_a[LOCAL_CAP];       //   amax over keep rows,
    int32_t local_src[LOCAL_CAP];   //   1 = its codes are the cached q2 row
    int32_t red[16 * NWARPS];       // per-warp partial dot products (patched columns)
    int32_t pt_rows[PATCH_ROWS];    // producer: q2 row (patched column) of each patch-tile row
    int32_t warp_sums[NWARPS];
};

struct Params {
    DecodeArgs a;
    int mpad, num_kb, n_tiles, stages;
    int n_acc;     // accumulators per tile buffer (n_acc * mpad <= 256 TMEM columns)
    int prefetch;  // weight stages loaded before the prologue (<= stages)
    int64_t total_units;
    uint32_t b_bytes;
    unsigned long long* dbg;  // per-CTA %globaltimer stamps (dev tool), nullable
};

// srow (per-token factor) + a union of {this CTA's X column slice (prologue),
// x[:, O] factors (epilogue)} + barriers
constexpr size_t SMEM_UNION = 24576;
constexpr int MAX_OWNED_WORDS = 64;
__host__ __device__ constexpr size_t smem_extra() {
    return MAX_M * sizeof(float) + SMEM_UNION + MAX_M * sizeof(uint32_t) +
           MAX_OWNED_WORDS * sizeof(uint32_t) + sizeof(Bars) + 64;
}

template <int EPI>
__device__ __forceinline__ void store_out(const DecodeArgs& a, int64_t m, int64_t n, float v) {
    if constexpr (EPI == EPI_F16)
        reinterpret_cast<__half*>(a.y)[m * a.ldy + n] = __float2half_rn(v);
    else
        reinterpret_cast<float*>(a.y)[m * a.ldy + n] = v;
}

// y[m, n] from the exact int32 accumulator c (same op order as gemm_sm100.cu)
template <int EPI>
__device__ __forceinline__ float epi_value(const DecodeArgs& a, int32_t c, int64_t m, int64_t n,
                                           float rowf, float colf, float aw, int n_out,
                                           const float* sxo, const float (&wr)[WO_CAP]) {
    if constexpr (EPI == EPI_F32_EXACT) {
        const double sx = 127.0 / static_cast<double>(rowf);
        const double sw = 127.0 / static_cast<double>(amax_or_127(aw));
        const double d = __dmul_rn(sx, sw);
        float v = __double2float_rn(__ddiv_rn(static_cast<double>(c), d));
        if (n_out > 0) {
            double hacc = 0.0;
            for (int o = 0; o < n_out; ++o) {
                const int64_t k = a.o_idx[o];
                const double xv = __half2float(a.x[m * a.ldx + k]);
                const double wv = __half2float(a.w[k * a.ldw + n]);
                hacc = __dadd_rn(hacc, __dmul_rn(xv, wv));
            }
            v = __double2float_rn(__dadd_rn(static_cast<double>(v), hacc));
        }
        return v;
    } else {
        float v = (static_cast<float>(c) * rowf) * colf;
        if (n_out > 0 && n_out <= WO_CAP) {
#pragma unroll
            for (int o = 0; o < WO_CAP; ++o)
                if (o < n_out) v = fmaf(sxo[m * WO_CAP + o], wr[o], v);
        } else {
            for (int o = 0; o < n_out; ++o) {
                const int64_t k = a.o_idx[o];
                v = fmaf(__half2float(a.x[m * a.ldx + k]), __half2float(a.w[k * a.ldw + n]), v);
            }
        }
        return v;
    }
}

// 16 token columns of this thread's weight row: sum of the n_acc accumulators
__device__ __forceinline__ void tmem_row16(uint32_t taddr, int n_acc, int mpad, uint32_t (&r)[16]) {
    tmem_ld_32x32b_x16(taddr, r);
    for (int j = 1; j < n_acc; ++j) {
        uint32_t t[16];
        tmem_ld_32x32b_x16(taddr + static_cast<uint32_t>(j * mpad), t);
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 16; ++e) r[e] += t[e];
    }
    tmem_ld_wait();
}

// mask words owned by CTA c (whole words: the owner sees every row of its
// columns, so its outlier bits are final without a cross-CTA reduction)
__host__ __device__ __forceinline__ void owned_words(int64_t nwords, int64_t G, int64_t c,
                                                     int64_t& w0, int64_t& w1) {
    w0 = nwords * c / G;
    w1 = nwords * (c + 1) / G;
}

template <int EPI>
__global__ void __launch_bounds__(THREADS, 1)
    decode_fused_kernel(const __grid_constant__ CUtensorMap tmap_w,
                        const __grid_constant__ CUtensorMap tmap_x,
                        const __grid_constant__ CUtensorMap tmap_p,
                        const __grid_constant__ CUtensorMap tmap_q2,
                        const __grid_constant__ CUtensorMap tmap_pb, const Params p) {
    cg::grid_group grid = cg::this_grid();
    const DecodeArgs& a = p.a;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u);
    const uint32_t stage_bytes = A_BYTES + p.b_bytes;
    uint8_t* ring = smem;
    float* srow = reinterpret_cast<float*>(smem + static_cast<size_t>(p.stages) * stage_bytes);
    float* sxo = srow + MAX_M;                                   // epilogue
    __half* xs = reinterpret_cast<__half*>(sxo);                 // prologue (same bytes)
    uint32_t* sram = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(sxo) + SMEM_UNION);
    uint32_t* smw = sram + MAX_M;                                // owned mask words
    Bars* bars = reinterpret_cast<Bars*>(smw + MAX_OWNED_WORDS);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t G = gridDim.x;
    // unit indices fit 32 bits (decode_fits bounds T * G < 2^31): 32-bit division on
    // the producer / MMA / finisher paths (a 64-bit one is a ~100-instruction call)
    const uint32_t T = static_cast<uint32_t>(p.total_units);
    const uint32_t Gu = gridDim.x;
    const int u_begin = static_cast<int>(T * blockIdx.x / Gu);
    const int u_end = static_cast<int>(T * (blockIdx.x + 1) / Gu);
    const int num_kb = p.num_kb;
    // the last tile (index n_tiles) is the patch tile: its A rows are the q2 rows
    // of this call's patched columns, written in P2, so it is never prefetched
    const int main_units = p.n_tiles * num_kb;
    const int n_pre = max(0, min(p.prefetch, min(u_end, main_units) - u_begin));

    if (threadIdx.x == 0) DSTAMP(p.dbg, 0);
    // ================= W0: setup + weight prefetch (independent of X)
    if (threadIdx.x == 0) {
        tma_prefetch_desc(&tmap_w);
        tma_prefetch_desc(&tmap_x);
        tma_prefetch_desc(&tmap_p);
        tma_prefetch_desc(&tmap_q2);
        tma_prefetch_desc(&tmap_pb);
        for (int s = 0; s < p.stages; ++s) {
            mbar_init(&bars->full[s], 1);
            mbar_init(&bars->empty[s], 1);
        }
        for (int q = 0; q < 2; ++q) {
            mbar_init(&bars->tmem_full[q], 1);
            mbar_init(&bars->tmem_empty[q], 4);
        }
        fence_mbarrier_init();
        bars->n_local = 0;
        const uint64_t pol_w = l2_policy_evict_normal();
        for (int i = 0; i < n_pre; ++i) {
            const int u = u_begin + i;
            mbar_arrive_expect_tx(&bars->full[i], stage_bytes);
            tma_load_2d(&tmap_w, &bars->full[i], ring + static_cast<size_t>(i) * stage_bytes,
                        (u % num_kb) * BK, (u / num_kb) * TILE_N,
                        pol_w);
        }
    }
    if (warp == 2) tmem_alloc<TMEM_COLS>(&bars->tmem_slot);
    // programmatic dependent launch: the weight prefetch above (weights are
    // never written by the preceding kernels) overlaps the previous layer's
    // tail; X, the threshold word and the workspace only after the wait
    pdl_wait();
    pdl_trigger();

    // ================= prologue (warps 1-7; warp 0 is issuing the prefetch)
    constexpr int PT = (NWARPS - 1) * 32;
    const bool pro = warp >= 1;
    const int pt = threadIdx.x - 32;  // 0..PT-1 for prologue threads
    const int64_t M = a.M, K = a.K, N = a.N;
    const int64_t nwords = (K + 31) >> 5;
    int64_t w0, w1;
    // 32-bit division (decode_fits bounds nwords * G and N * G below 2^32)
    w0 = static_cast<uint32_t>(nwords) * blockIdx.x / Gu;
    w1 = static_cast<uint32_t>(nwords) * (blockIdx.x + 1) / Gu;
    const int64_t c0 = w0 * 32;
    const int64_t c1 = min(w1 * 32, K);
    const int64_t ncols = c1 > c0 ? c1 - c0 : 0;
    const int64_t nvec = (ncols + 7) / 8;         // 8-column vectors of the slice
    const int64_t xs_ld = (w1 - w0) * 32;          // halves per smem row
    const uint32_t thr_bits = a.thr_bits_dev != nullptr ? *a.thr_bits_dev : a.thr_bits;

    // fixup candidates of this CTA's column range (weight-side data: fetched now,
    // consumed after barrier 1)
    const int64_t j0 = static_cast<uint32_t>(N) * blockIdx.x / Gu, j1 = static_cast<uint32_t>(N) * (blockIdx.x + 1) / Gu;
    int32_t crA[kTopT], crB[kTopT];
#pragma unroll
    for (int i = 0; i < kTopT; ++i) {
        const int64_t ja = j0 + threadIdx.x, jb = ja + THREADS;
        crA[i] = ja < j1 ? a.cand_r[i * N + ja] : -1;
        crB[i] = jb < j1 ? a.cand_r[i * N + jb] : -1;
    }

    // ---------------- P1: load this CTA's column slice of X (all M rows) into
    // smem; its outlier bits (final) and per-row partial absmax over keep columns
    if (pro) {
        const int nv = static_cast<int>(nvec);  // 32-bit index math (see u_begin)
        for (int i = pt; i < static_cast<int>(M) * nv; i += PT) {
            const int m = i / nv, v8 = i - m * nv;
            const uint4 q = load8(a.x + m * a.ldx, c0 + v8 * 8, K, a.x_vec);
            *reinterpret_cast<uint4*>(xs + m * xs_ld + v8 * 8) = q;
        }
        for (int64_t i = static_cast<int64_t>(blockIdx.x) * PT + pt; i <= a.n_tiles; i += G * PT)
            a.tile_cnt[i] = 0;  // main tiles + the patch tile
        for (int64_t i = static_cast<int64_t>(blockIdx.x) * PT + pt; i < N; i += G * PT)
            a.patch_pos[i] = 0;
        if (blockIdx.x == 0 && pt == 0) *a.p_count = 0;
        for (int64_t i = static_cast<int64_t>(blockIdx.x) * PT + pt; i < PATCH_ROWS; i += G * PT)
            a.pq_ready[i] = 0;
    }
    __syncthreads();
    // one warp per owned word: lane = column, OR over rows
    for (int64_t w = w0 + (warp - 1); pro && w < w1; w += NWARPS - 1) {
        const int64_t col = (w - w0) * 32 + lane;
        uint32_t hit = 0;
        if (w * 32 + lane < K)
            for (int64_t m = 0; m < M; ++m)
                hit |= (__half_as_ushort(xs[m * xs_ld + col]) & 0x7FFFu) >= thr_bits ? 1u : 0u;
        const uint32_t word = __ballot_sync(0xffffffffu, hit != 0);
        if (lane == 0) {
            a.mask[w] = word;
            smw[w - w0] = word;
        }
    }
    __syncthreads();
    // per-row partial absmax over this slice's keep columns -> part[cta][row]
    // (warp per row, lanes over columns)
    for (int64_t m = pro ? warp - 1 : M; m < M; m += NWARPS - 1) {
        uint32_t mx = 0;
        for (int64_t col = lane; col < ncols; col += 32)
            if (!((smw[col >> 5] >> (col & 31)) & 1u))
                mx = max(mx, static_cast<uint32_t>(__half_as_ushort(xs[m * xs_ld + col])) & 0x7FFFu);
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, d));
        if (lane == 0) a.part[static_cast<int64_t>(blockIdx.x) * M + m] = mx;
    }
    if (threadIdx.x == 32) DSTAMP(p.dbg, 1);
    grid.sync();

    // ---------------- P2: row absmax (every CTA reduces the partials), sorted
    // outlier list (CTA 0), codes of this CTA's slice, column fixup
    // the mask words the fixup tests first (its candidates' rows are known since
    // P1): loaded now, in flight with the partials below
    const uint32_t fmA = crA[0] >= 0 ? __ldcg(a.mask + (crA[0] >> 5)) : 0u;
    const uint32_t fmB = crB[0] >= 0 ? __ldcg(a.mask + (crB[0] >> 5)) : 0u;
    // warp per 4 rows, lanes over the CTAs' partials (all loads in flight first)
    for (int64_t m0 = warp * 4; m0 < M; m0 += NWARPS * 4) {
        uint32_t mx[4] = {0u, 0u, 0u, 0u};
        for (int64_t c = lane; c < G; c += 32)
#pragma unroll
            for (int r = 0; r < 4; ++r)
                if (m0 + r < M) mx[r] = max(mx[r], __ldcg(a.part + c * M + m0 + r));
#pragma unroll
        for (int r = 0; r < 4; ++r) {
#pragma unroll
            for (int d = 16; d > 0; d >>= 1) mx[r] = max(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], d));
            if (lane == 0 && m0 + r < M) sram[m0 + r] = mx[r];
        }
    }
    if (blockIdx.x == 0) compact_block(a.mask, nwords, a.o_idx, a.o_count, bars->warp_sums);
    else compact_block_smem(a.mask, nwords, bars->o_s, &bars->n_out, bars->warp_sums);
    __syncthreads();
    if (blockIdx.x == 0 && threadIdx.x == 0) bars->n_out = *a.o_count;
    if (blockIdx.x == 0 && threadIdx.x < WO_CAP && threadIdx.x < *a.o_count)
        bars->o_s[threadIdx.x] = a.o_idx[threadIdx.x];  // only written entries (initcheck)
    __syncthreads();
    const int n_out = bars->n_out;
    // x[:, O] factor of this thread's first item: loaded before the codes (stored
    // after them, when the X slice's shared memory is free)
    const bool xo_on = n_out > 0 && n_out <= WO_CAP;
    const int xo_items = xo_on ? static_cast<int>(M) * n_out : 0;
    float xo_first = 0.0f;
    if (static_cast<int>(threadIdx.x) < xo_items) {
        const int m = threadIdx.x / n_out, o = threadIdx.x - m * n_out;
        xo_first = __half2float(a.x[m * a.ldx + bars->o_s[o]]);
    }
    // codes: 8 consecutive columns per thread item, stored as 8 bytes
    {
        const int nv = static_cast<int>(nvec);
        for (int i = threadIdx.x; i < static_cast<int>(M) * nv; i += THREADS) {
            const int m = i / nv, v8 = i - m * nv;
            const float amax = hbits_to_float(sram[m]);
            const double s = scale_of(amax);
            const float s32 = static_cast<float>(s);
            const uint32_t mb = (smw[(v8 * 8) >> 5] >> ((v8 * 8) & 31)) & 0xFFu;
            const __half* h = xs + m * xs_ld + v8 * 8;
            uint32_t b[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const int c = (((mb >> e) & 1u) || c0 + v8 * 8 + e >= K) ? 0 : code_fast(__half2float(h[e]), s32, s);
                b[e] = static_cast<uint32_t>(c) & 0xFFu;
            }
            *reinterpret_cast<uint2*>(a.xq + m * a.ldq + c0 + v8 * 8) =
                make_uint2(b[0] | b[1] << 8 | b[2] << 16 | b[3] << 24, b[4] | b[5] << 8 | b[6] << 16 | b[7] << 24);
        }
        if (blockIdx.x == G - 1) {  // K..ldq padding
            const int64_t pad0 = (K + 7) / 8 * 8;
            for (int64_t i = threadIdx.x; i < M * ((a.ldq - pad0) / 8); i += THREADS) {
                const int64_t per = (a.ldq - pad0) / 8;
                *reinterpret_cast<uint2*>(a.xq + (i / per) * a.ldq + pad0 + (i % per) * 8) = make_uint2(0u, 0u);
            }
        }
        if (blockIdx.x == 0)
            for (int64_t m = threadIdx.x; m < M; m += THREADS) {
                a.row_amax[m] = hbits_to_float(sram[m]);
                a.ramax_bits[m] = sram[m];
            }
    }
    __syncthreads();  // the X slice (xs) is consumed: its bytes become sxo
    // x[:, O] factors for the epilogue (X is read-only: no need to wait for anyone)
    if (static_cast<int>(threadIdx.x) < xo_items) {
        const int m = threadIdx.x / n_out, o = threadIdx.x - m * n_out;
        sxo[m * WO_CAP + o] = xo_first;
    }
    for (int i = threadIdx.x + THREADS; i < xo_items; i += THREADS) {
        const int m = i / n_out, o = i - m * n_out;
        sxo[m * WO_CAP + o] = __half2float(a.x[m * a.ldx + bars->o_s[o]]);
    }
    // weight-stationary fixup (weights.cu fixup_kernel semantics) over this
    // CTA's column range; the four candidates were fetched during P1
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int64_t j = j0 + threadIdx.x + h * THREADS;
        if (j >= j1) continue;
        int32_t cr[kTopT];
#pragma unroll
        for (int i = 0; i < kTopT; ++i) cr[i] = h ? crB[i] : crA[i];
        if (cr[0] < 0 || !(((h ? fmB : fmA) >> (cr[0] & 31)) & 1u)) continue;
        float a_new = -1.0f;
        bool exhausted = true;
        int src = 0;  // 1: the cached q2 row holds this column's new codes
#pragma unroll
        for (int i = 1; i < kTopT; ++i) {
            if (!exhausted) break;
            if (cr[i] < 0) {
                exhausted = false;
                a_new = 0.0f;
                src = i == 1;
            } else if (!bit_of(a.mask, cr[i])) {
                exhausted = false;
                a_new = hbits_to_float(a.cand_v[i * N + j]);
                src = i == 1;
            }
        }
        if (exhausted) {
            uint32_t m = 0;
            for (int64_t k = 0; k < K; ++k)
                if (!bit_of(a.mask, k))
                    m = max(m, static_cast<uint32_t>(__half_as_ushort(a.w[k * a.ldw + j])) & 0x7FFFu);
            a_new = hbits_to_float(m);
        }
        if (a_new != a.amax_full[j]) {
            const int32_t pidx = atomicAdd(a.p_count, 1);
            a.p_idx[pidx] = static_cast<int32_t>(j);
            a.p_amax[pidx] = a_new;
            a.patch_pos[j] = pidx + 1;
            a.p_src[pidx] = src;
            // the patch tile gathers this row from q2 after the barrier: pull it into
            // L2 now (asynchronous; nothing here waits for it)
            if (src && pidx < PT_GATHER_ROWS)
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.q2 + j * a.ldq),
                             "r"(static_cast<uint32_t>(a.ldq & ~int64_t(15)))
                             : "memory");
            const int li = atomicAdd(&bars->n_local, 1);
            bars->local_j[li] = static_cast<int32_t>(j);
            bars->local_p[li] = pidx;
            bars->local_a[li] = a_new;
            bars->local_src[li] = src;
        }
    }
    __syncthreads();
    // patch-tile rows: a patched column whose codes are its cached q2 row (the
    // common case) is gathered straight from q2 by the patch tile's producer
    // (TMA tile::gather4, no copy here); only re-derived codes (its top-2 rows
    // are both outlier rows: rare) are written to pq now
    for (int li = 0; li < bars->n_local; ++li) {
        const int pidx = bars->local_p[li];
        if (pidx >= PATCH_ROWS || (bars->local_src[li] && pidx < PT_GATHER_ROWS)) continue;
        const int64_t j = bars->local_j[li];
        int8_t* dst = a.pq + static_cast<int64_t>(pidx) * a.ldq;
        if (bars->local_src[li]) {  // rows >= PT_GATHER_ROWS: one box load of pq after the barrier
            const uint4* srcq = reinterpret_cast<const uint4*>(a.q2 + j * a.ldq);
            for (int64_t v = threadIdx.x; v < a.ldq / 16; v += THREADS)
                reinterpret_cast<uint4*>(dst)[v] = __ldcs(srcq + v);
        } else {
            const double sc = scale_of(bars->local_a[li]);
            const float s32 = static_cast<float>(sc);
            for (int64_t k = threadIdx.x; k < a.ldq; k += THREADS)
                dst[k] = (k < K && !bit_of(a.mask, k))
                             ? static_cast<int8_t>(code_fast(__half2float(a.w[k * a.ldw + j]), s32, sc)) : int8_t(0);
        }
    }
    // Xq and the patch rows are read back by TMA (async proxy) after the barrier
    asm volatile("fence.proxy.async.global;" ::: "memory");
    if (threadIdx.x == 32) DSTAMP(p.dbg, 3);
    grid.sync();
    if (threadIdx.x == 0) DSTAMP(p.dbg, 4);
    // per-token factors (rows of X) staged once; x[:, O] was staged in P2
    for (int64_t m = threadIdx.x; m < M; m += THREADS) srow[m] = amax_or_127(hbits_to_float(sram[m]));
    __syncthreads();
    // ---------------- this CTA's patched columns, complete, before its weight
    // stream resumes (memory is quiet; nothing downstream waits on them): exact
    // int32 dots of the re-derived codes (q2 row, or W's column in the rare
    // multi-outlier case) with Xq, then the same epilogue math
    if (threadIdx.x == 0 && (kDevStamps && p.dbg != nullptr)) {
        p.dbg[blockIdx.x * 16 + 12] = static_cast<unsigned long long>(bars->n_local);
        p.dbg[blockIdx.x * 16 + 13] = static_cast<unsigned long long>(bars->n_local ? bars->local_src[0] : 9);
    }
    for (int li = 0; li < bars->n_local; ++li) {
        if (bars->local_p[li] < PATCH_ROWS) continue;  // handled by the patch tile
        const int64_t j = bars->local_j[li];
        const float aw = bars->local_a[li];
        const bool src = bars->local_src[li] != 0;
        const double s = scale_of(aw);
        const float s32 = static_cast<float>(s);
        const int64_t nk16 = a.ldq / 16;
        for (int64_t m0 = 0; m0 < M; m0 += 16) {
            int acc[16];
#pragma unroll
            for (int mm = 0; mm < 16; ++mm) acc[mm] = 0;
            for (int64_t kv = threadIdx.x; kv < nk16; kv += THREADS) {
                uint4 cw;
                if (src) {
                    cw = __ldcs(reinterpret_cast<const uint4*>(a.q2 + j * a.ldq + kv * 16));
                } else {  // rare: re-derive 16 codes from the strided W column
                    uint32_t b[16];
#pragma unroll
                    for (int e = 0; e < 16; ++e) {
                        const int64_t k = kv * 16 + e;
                        const int c = (k < K && !bit_of(a.mask, k))
                                          ? code_fast(__half2float(a.w[k * a.ldw + j]), s32, s) : 0;
                        b[e] = static_cast<uint32_t>(c) & 0xFFu;
                    }
                    cw = make_uint4(b[0] | b[1] << 8 | b[2] << 16 | b[3] << 24,
                                    b[4] | b[5] << 8 | b[6] << 16 | b[7] << 24,
                                    b[8] | b[9] << 8 | b[10] << 16 | b[11] << 24,
                                    b[12] | b[13] << 8 | b[14] << 16 | b[15] << 24);
                }
                // predicated (branch-free) loads: all rows' bytes in flight at once
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    uint4 xv[8];
#pragma unroll
                    for (int mm = 0; mm < 8; ++mm) {
                        const int64_t m = m0 + h * 8 + mm;
                        xv[mm] = m < M ? __ldcg(reinterpret_cast<const uint4*>(a.xq + m * a.ldq + kv * 16))
                                       : make_uint4(0u, 0u, 0u, 0u);
                    }
#pragma unroll
                    for (int mm = 0; mm < 8; ++mm) {
                        int& ac = acc[h * 8 + mm];
                        ac = __dp4a(static_cast<int>(xv[mm].x), static_cast<int>(cw.x), ac);
                        ac = __dp4a(static_cast<int>(xv[mm].y), static_cast<int>(cw.y), ac);
                        ac = __dp4a(static_cast<int>(xv[mm].z), static_cast<int>(cw.z), ac);
                        ac = __dp4a(static_cast<int>(xv[mm].w), static_cast<int>(cw.w), ac);
                    }
                }
            }
            if (threadIdx.x == 0 && li == 0 && m0 == 0) DSTAMP(p.dbg, 10);
#pragma unroll
            for (int mm = 0; mm < 16; ++mm) {
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) acc[mm] += __shfl_xor_sync(0xffffffffu, acc[mm], o);
                if (lane == 0) bars->red[mm * NWARPS + warp] = acc[mm];
            }
            __syncthreads();
            if (threadIdx.x < 16 && m0 + threadIdx.x < M) {
                const int64_t m = m0 + threadIdx.x;
                int32_t c = 0;
#pragma unroll
                for (int w = 0; w < NWARPS; ++w) c += bars->red[threadIdx.x * NWARPS + w];
                const float colf = amax_or_127(aw) * (1.0f / 16129.0f);
                float wr[WO_CAP];
#pragma unroll
                for (int o = 0; o < WO_CAP; ++o)
                    wr[o] = (EPI != EPI_F32_EXACT && o < n_out && n_out <= WO_CAP)
                                ? __half2float(a.w[static_cast<int64_t>(bars->o_s[o]) * a.ldw + j])
                                : 0.0f;
                store_out<EPI>(a, m, j, epi_value<EPI>(a, c, m, j, srow[m], colf, aw, n_out, sxo, wr));
            }
            __syncthreads();
        }
    }
    // patched columns read L2/HBM with a few dependent round trips: keep the
    // weight streams of all CTAs paused until they are done (one more grid
    // barrier, only when the call has patched columns at all)

    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x == 0) DSTAMP(p.dbg, 9);
    const uint32_t tmem_base = bars->tmem_slot;

    if (warp == 0) {
        // ---------------- TMA producer
        if (lane == 0) {
            const uint64_t pol_w = l2_policy_evict_normal();
            const uint64_t pol_x = l2_policy_evict_last();
            for (int i = 0; i < n_pre; ++i) {  // token halves of the prefilled stages
                const int u = u_begin + i;
                tma_load_2d(&tmap_x, &bars->full[i], ring + static_cast<size_t>(i) * stage_bytes + A_BYTES,
                            (u % num_kb) * BK, 0, pol_x);
            }
            int stage = n_pre % p.stages;
            uint32_t phase = n_pre == p.stages ? 1u : 0u;
            int pt_groups = -1;  // patch tile: gathered 4-row groups (set at its first unit)
            bool pt_rest = false;  // rows >= PT_GATHER_ROWS present (box load from pq)
            uint32_t pt_pq = 0;  // bit g: group g is gathered from pq
            for (int u = u_begin + n_pre; u < u_end; ++u) {
                const int tile = u / num_kb;
                const int kb = u - tile * num_kb;
                mbar_wait(&bars->empty[stage], phase ^ 1u);
                uint8_t* dst = ring + static_cast<size_t>(stage) * stage_bytes;
                if (tile < p.n_tiles) {
                    mbar_arrive_expect_tx(&bars->full[stage], stage_bytes);
                    tma_load_2d(&tmap_w, &bars->full[stage], dst, kb * BK, tile * TILE_N, pol_w);
                } else {
                    // the patch tile: row r = patched column p_idx[r]; groups of 4 rows
                    // are gathered (tile::gather4) from the cached q2 rows, or from pq
                    // when a group holds a re-derived row (its q2-sourced rows are then
                    // copied to pq after the barrier, each published with a ready flag)
                    if (pt_groups < 0) {
                        // one round trip: the count and the first rows' column / source
                        // (entries past the count are ignored)
                        int32_t pr[PT_GATHER_ROWS], ps[PT_GATHER_ROWS];
                        const int np_raw = __ldcg(a.p_count);
#pragma unroll
                        for (int r = 0; r < PT_GATHER_ROWS; ++r) {
                            pr[r] = __ldcg(a.p_idx + r);
                            ps[r] = __ldcg(a.p_src + r);
                        }
                        const int np = min(np_raw, PATCH_ROWS);
                        pt_rest = np > PT_GATHER_ROWS;
                        pt_groups = (min(np, PT_GATHER_ROWS) + 3) / 4;
                        bool waited = false;
                        for (int g = 0; g < pt_groups; ++g) {
                            int n0 = 0;
#pragma unroll
                            for (int i = 0; i < 4; ++i) {
                                const int r = 4 * g + i;
                                if (r < np) {
                                    bars->pt_rows[r] = pr[r];
                                    n0 += ps[r] == 0 ? 1 : 0;
                                }
                            }
                            for (int r = np; r < 4 * g + 4; ++r) bars->pt_rows[r] = bars->pt_rows[4 * g];
                            if (n0 > 0) {
                                pt_pq |= 1u << g;
#pragma unroll
                                for (int i = 0; i < 4; ++i) {
                                    const int r = 4 * g + i;
                                    if (r < np && ps[r] != 0)
                                        while (ld_acquire(a.pq_ready + r) == 0) {
                                        }
                                }
                                waited = true;
                            }
                        }
                        if (waited) asm volatile("fence.proxy.async.global;" ::: "memory");
                    }
                    mbar_arrive_expect_tx(&bars->full[stage], static_cast<uint32_t>(pt_groups) * 4u * BK + p.b_bytes +
                                                                  (pt_rest ? static_cast<uint32_t>(PATCH_ROWS - PT_GATHER_ROWS) * BK : 0u));
                    if (pt_rest)  // rows PT_GATHER_ROWS.. : copied to pq in P2 (many patches)
                        tma_load_2d(&tmap_pb, &bars->full[stage], dst + PT_GATHER_ROWS * BK, kb * BK, 0, pol_x);
                    for (int g = 0; g < pt_groups; ++g) {
                        uint8_t* gd = dst + g * 4 * BK;
                        if ((pt_pq >> g) & 1u)
                            tma_gather4(&tmap_p, &bars->full[stage], gd, kb * BK, 4 * g, 4 * g + 1, 4 * g + 2, 4 * g + 3);
                        else
                            tma_gather4(&tmap_q2, &bars->full[stage], gd, kb * BK, bars->pt_rows[4 * g],
                                        bars->pt_rows[4 * g + 1], bars->pt_rows[4 * g + 2], bars->pt_rows[4 * g + 3]);
                    }
                }
                tma_load_2d(&tmap_x, &bars->full[stage], dst + A_BYTES, kb * BK, 0, pol_x);
                if (++stage == p.stages) {
                    stage = 0;
                    phase ^= 1u;
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer
        const uint32_t idesc = idesc_i8(TILE_N, static_cast<uint32_t>(p.mpad));
        int stage = 0;
        uint32_t phase = 0;
        int seg = 0;
        for (int u = u_begin; u < u_end; ++seg) {
            const int tile = u / num_kb;
            const int seg_end = min(u_end, (tile + 1) * num_kb);
            const int acc = seg & 1;
            mbar_wait(&bars->tmem_empty[acc], ((seg >> 1) & 1) ^ 1u);
            tc_fence_after();
            const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * 256);
            for (int kk = 0; u < seg_end; ++u, ++kk) {
                mbar_wait(&bars->full[stage], phase);
                tc_fence_after();
                if (lane == 0 && u == u_begin) DSTAMP(p.dbg, 5);
                if (lane == 0 && u == u_end - 1) DSTAMP(p.dbg, 14);  // last unit's operands landed
                if (lane == 0) {
                    const uint32_t a0 = smem_addr(ring + static_cast<size_t>(stage) * stage_bytes);
                    const uint32_t b0 = a0 + A_BYTES;
                    // K-steps rotate over n_acc independent accumulators (the
                    // epilogue adds them back, exact int32)
#pragma unroll
                    for (int k = 0; k < BK / UMMA_K; ++k)
                        mma_i8(d_tmem + static_cast<uint32_t>((k % p.n_acc) * p.mpad),
                               smem_desc_k_sw128(a0 + k * UMMA_K), smem_desc_k_sw128(b0 + k * UMMA_K),
                               idesc, (kk > 0 || k >= p.n_acc) ? 1u : 0u);
                    mma_commit(&bars->empty[stage]);
                }
                __syncwarp();
                if (++stage == p.stages) {
                    stage = 0;
                    phase ^= 1u;
                }
            }
            if (lane == 0) mma_commit(&bars->tmem_full[acc]);
            __syncwarp();
        }
        if (lane == 0) DSTAMP(p.dbg, 6);
    } else {
        if (warp == 2 || warp == 3) {
            // ---------------- rare: a q2-sourced patch row whose 4-row group also holds
            // a re-derived row must be in pq too (the group is gathered from pq)
            const int t64 = threadIdx.x - 64;
            const int np = min(__ldcg(a.p_count), PATCH_ROWS);
            for (int li = 0; li < bars->n_local; ++li) {
                const int pidx = bars->local_p[li];
                if (pidx >= PT_GATHER_ROWS || !bars->local_src[li]) continue;
                bool mixed = false;
                for (int r = pidx & ~3; r < min((pidx & ~3) + 4, np); ++r) mixed |= __ldcg(a.p_src + r) == 0;
                if (!mixed) continue;
                const int64_t j = bars->local_j[li];
                const uint4* srcq = reinterpret_cast<const uint4*>(a.q2 + j * a.ldq);
                uint4* dst = reinterpret_cast<uint4*>(a.pq + static_cast<int64_t>(pidx) * a.ldq);
                for (int64_t v = t64; v < a.ldq / 16; v += 64) dst[v] = __ldcs(srcq + v);
                __threadfence();
                named_bar_sync(3, 64);
                if (t64 == 0) st_release(a.pq_ready + pidx, 1);
            }
        } else if (warp >= 4) {
            // ---------------- epilogue: thread = weight row n of the tile
            const int np_all = __ldcg(a.p_count);  // final after barrier 2
            const int quad = warp & 3;
            const int n_local = quad * 32 + lane;
            const int chunks = p.mpad / 16;
            int seg = 0;
            for (int u = u_begin; u < u_end; ++seg) {
                const int tile = u / num_kb;
                const int seg_end = min(u_end, (tile + 1) * num_kb);
                const int len = static_cast<int>(seg_end - u);
                const bool full = len == num_kb;
                u = seg_end;
                const int acc = seg & 1;
                int64_t n;
                bool n_ok;
                int32_t pp;
                float aw;
                if (tile < p.n_tiles) {
                    n = tile * TILE_N + n_local;
                    n_ok = n < N;
                    pp = n_ok ? __ldcg(a.patch_pos + n) : 0;  // patched: written by the patch tile
                    aw = n_ok ? a.amax_full[n] : 127.0f;
                } else {  // patch tile: row n_local is patched column p_idx[n_local]
                    n_ok = n_local < min(np_all, PATCH_ROWS);
                    n = n_ok ? __ldcg(a.p_idx + n_local) : 0;
                    pp = 0;
                    aw = n_ok ? __ldcg(a.p_amax + n_local) : 127.0f;
                }
                const float colf = amax_or_127(aw) * (1.0f / 16129.0f);
                float wr[WO_CAP];
#pragma unroll
                for (int o = 0; o < WO_CAP; ++o) {
                    float wv = 0.0f;
                    if (EPI != EPI_F32_EXACT && o < n_out && n_out <= WO_CAP && n_ok)
                        wv = __half2float(a.w[static_cast<int64_t>(bars->o_s[o]) * a.ldw + n]);
                    wr[o] = wv;
                }
                mbar_wait(&bars->tmem_full[acc], (seg >> 1) & 1);
                tc_fence_after();
                const uint32_t t_row = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) +
                                       static_cast<uint32_t>(acc * 256);
                bool finisher = full;
                if (!full) {
                    // partial sums: plain coalesced stores into this CTA's slot
                    // (slot 0 = its first segment, 1 = its last), no atomics
                    int32_t* slot = a.c32 + (blockIdx.x * 2 + (seg == 0 ? 0 : 1)) * (M * TILE_N) + n_local;
                    for (int ch = 0; ch < chunks; ++ch) {
                        uint32_t r[16];
                        tmem_row16(t_row + ch * 16, p.n_acc, p.mpad, r);
#pragma unroll
                        for (int jj = 0; jj < 16; ++jj)
                            if (ch * 16 + jj < M) __stcg(slot + (ch * 16 + jj) * TILE_N, static_cast<int32_t>(r[jj]));
                    }
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&bars->tmem_empty[acc]);
                    __threadfence();
                    named_bar_sync(1, 128);
                    if (threadIdx.x == 128) {
                        bars->finisher = atomicAdd(a.tile_cnt + tile, len) + len == num_kb ? 1 : 0;
                        __threadfence();
                    }
                    named_bar_sync(1, 128);
                    finisher = bars->finisher != 0;
                    named_bar_sync(1, 128);
                    if (finisher) __threadfence();
                }
                if (full) {
                    for (int ch = 0; ch < chunks; ++ch) {
                        uint32_t r[16];
                        tmem_row16(t_row + ch * 16, p.n_acc, p.mpad, r);
                        if (!n_ok || pp) continue;  // patched columns: written by their dot products
#pragma unroll
                        for (int jj = 0; jj < 16; ++jj) {
                            const int64_t m = ch * 16 + jj;
                            if (m >= M) break;
                            store_out<EPI>(a, m, n, epi_value<EPI>(a, static_cast<int32_t>(r[jj]), m, n,
                                                                  srow[m], colf, aw, n_out, sxo, wr));
                        }
                    }
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&bars->tmem_empty[acc]);
                } else if (finisher && n_ok && !pp) {
                    // contributors: the CTAs whose unit ranges intersect this tile
                    const uint32_t t0 = static_cast<uint32_t>(tile * num_kb), t1 = t0 + num_kb;
                    const uint32_t cf = ((t0 + 1) * Gu - 1) / T;
                    const uint32_t cl = (t1 * Gu - 1) / T;
                    for (int64_t m0 = 0; m0 < M; m0 += 16) {
                        int32_t cv[16];
#pragma unroll
                        for (int jj = 0; jj < 16; ++jj) cv[jj] = 0;
                        for (uint32_t c = cf; c <= cl; ++c) {
                            const int first_tile = static_cast<int>(T * c / Gu) / num_kb;
                            const int32_t* src = a.c32 + (static_cast<int64_t>(c) * 2 + (first_tile == tile ? 0 : 1)) * (M * TILE_N) + n_local;
#pragma unroll
                            for (int jj = 0; jj < 16; ++jj)
                                if (m0 + jj < M) cv[jj] += __ldcg(src + (m0 + jj) * TILE_N);
                        }
#pragma unroll
                        for (int jj = 0; jj < 16; ++jj) {
                            const int64_t m = m0 + jj;
                            if (m >= M) break;
                            store_out<EPI>(a, m, n, epi_value<EPI>(a, cv[jj], m, n, srow[m], colf, aw,
                                                                  n_out, sxo, wr));
                        }
                    }
                }
            }
            if (threadIdx.x == 128) DSTAMP(p.dbg, 7);
        }
    }
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc<TMEM_COLS>(tmem_base);
    }
    if (threadIdx.x == 0) DSTAMP(p.dbg, 8);
}

}  // namespace dec

// ------------------------------------------------------------------ host
int decode_stages(int64_t M) {
    const int mpad = static_cast<int>((M + 15) / 16 * 16);
    const int stage = dec::A_BYTES + mpad * dec::BK;
    const size_t budget = 227 * 1024 - 1024 - dec::smem_extra();
    int s = static_cast<int>(budget / stage);
    if (s > dec::MAX_STAGES) s = dec::MAX_STAGES;
    return s;
}

int decode_grid(int64_t K, int64_t N) {
    const int64_t units = ((N + dec::TILE_N - 1) / dec::TILE_N + 1) * ((K + dec::BK - 1) / dec::BK);
    return static_cast<int>(units < num_sms() ? units : num_sms());
}

bool decode_fits(int64_t M, int64_t K, int64_t N) {
    if (M <= 0 || M > dec::MAX_M || K <= 0 || N <= 0) return false;
    const int64_t G = decode_grid(K, N);
    const int64_t nwords = (K + 31) / 32;
    const int64_t wpc = (nwords + G - 1) / G;  // owned words per CTA (max)
    return M * wpc * 32 * 2 <= static_cast<int64_t>(dec::SMEM_UNION) && wpc <= 64 &&
           (N + G - 1) / G <= dec::LOCAL_CAP;
}

__global__ void set_word_kernel(uint32_t* dst, uint32_t value) { *dst = value; }

cudaError_t launch_set_word(uint32_t* dst, uint32_t value, cudaStream_t st) {
    set_word_kernel<<<1, 1, 0, st>>>(dst, value);
    count_launch();
    return cudaGetLastError();
}

// weight stages prefetched before the prologue (default 3: deeper prefetch
// queues the prologue's latency-bound round trips behind the weight stream);
// env I8MM_DECODE_PREFETCH for A/B measurements
static int decode_prefetch() {
    static int v = -2;
    if (v == -2) {
        const char* e = getenv("I8MM_DECODE_PREFETCH");
        v = (e && e[0]) ? atoi(e) : -1;
    }
    return v;
}

static unsigned long long* g_dbg = nullptr;
void set_decode_timeline(unsigned long long* stamps) { g_dbg = stamps; }
unsigned long long* debug_timeline() { return g_dbg; }

template <int EPI>
static cudaError_t launch_fused(const CUtensorMap& tw, const CUtensorMap& tx, const CUtensorMap& tp,
                                const CUtensorMap& tq, const CUtensorMap& tb,
                                const dec::Params& prm, size_t smem, int grid, cudaStream_t st) {
    static std::once_flag once;
    static cudaError_t attr_err = cudaSuccess;
    std::call_once(once, [] {
        attr_err = cudaFuncSetAttribute(dec::decode_fused_kernel<EPI>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    });
    if (attr_err != cudaSuccess) return attr_err;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(grid));
    cfg.blockDim = dim3(dec::THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, dec::decode_fused_kernel<EPI>, tw, tx, tp, tq, tb, prm);
    count_launch();
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

cudaError_t launch_decode(const DecodeArgs& a, int epi, cudaStream_t st) {
    using namespace dec;
    if (!decode_fits(a.M, a.K, a.N)) return cudaErrorInvalidValue;
    Params prm{};
    prm.a = a;
    prm.mpad = static_cast<int>((a.M + 15) / 16 * 16);
    prm.num_kb = static_cast<int>((a.K + BK - 1) / BK);
    prm.n_tiles = static_cast<int>((a.N + TILE_N - 1) / TILE_N);
    prm.total_units = static_cast<int64_t>(prm.n_tiles + 1) * prm.num_kb;  // + the patch tile
    prm.stages = decode_stages(a.M);
    prm.b_bytes = static_cast<uint32_t>(prm.mpad * BK);
    prm.n_acc = prm.mpad <= 64 ? 4 : (prm.mpad <= 128 ? 2 : 1);
    const int pf = decode_prefetch() < 0 ? 3 : decode_prefetch();
    prm.prefetch = pf < prm.stages ? pf : prm.stages;
    prm.dbg = g_dbg;
    CUtensorMap tw, tx, tp;
    if (!make_tmap_i8_rows(&tw, a.wq_t, a.N, a.K, a.ldq, TILE_N)) return cudaErrorInvalidValue;
    if (!make_tmap_i8_rows(&tx, a.xq, a.M, a.K, a.ldq, prm.mpad)) return cudaErrorInvalidValue;
    // patch tile A rows: 1-row boxes for tile::gather4 from pq and from q2
    CUtensorMap tq;
    if (!make_tmap_i8_rows(&tp, a.pq, PATCH_ROWS, a.K, a.ldq, 1)) return cudaErrorInvalidValue;
    if (!make_tmap_i8_rows(&tq, a.q2, a.N, a.K, a.ldq, 1)) return cudaErrorInvalidValue;
    CUtensorMap tb;  // pq rows PT_GATHER_ROWS..PATCH_ROWS-1 as one box
    if (!make_tmap_i8_rows(&tb, a.pq + PT_GATHER_ROWS * a.ldq, PATCH_ROWS - PT_GATHER_ROWS, a.K, a.ldq,
                           PATCH_ROWS - PT_GATHER_ROWS))
        return cudaErrorInvalidValue;
    const size_t smem =
        1024 + static_cast<size_t>(prm.stages) * (A_BYTES + prm.b_bytes) + smem_extra();
    const int grid = decode_grid(a.K, a.N);
    switch (epi) {
        case EPI_F16: return launch_fused<EPI_F16>(tw, tx, tp, tq, tb, prm, smem, grid, st);
        case EPI_F32: return launch_fused<EPI_F32>(tw, tx, tp, tq, tb, prm, smem, grid, st);
        case EPI_F32_EXACT: return launch_fused<EPI_F32_EXACT>(tw, tx, tp, tq, tb, prm, smem, grid, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace i8mm
