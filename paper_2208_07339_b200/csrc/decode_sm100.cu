// Decode path of the weight-stationary LLM.int8() linear layer (SURVEY.md 8f
// rank 2, config 3: M = 1..16 tokens). At these sizes the layer is bound by the
// stream of int8 weights from HBM (K*N bytes per call); the token side (outlier
// scan, row scales, codes, column fixup) is a few hundred KB at most, but it is a
// reduction over all of X that every weight tile's MMA depends on.
//
// ONE launch of 8-CTA thread-block clusters, one CTA per SM, no grid barrier and
// no cross-kernel hand-off: every cluster derives the token side itself, with
// the reduction in distributed shared memory, so the only global round trip
// before the first MMA is the read of X (L2-resident: the previous layer's
// output). Per CTA (256 threads):
//   setup   barriers + TMEM; the TMA producer fills the weight ring with the
//           CTA's first weight tiles before the dependency wait (the cached codes
//           are never written by a preceding kernel), so HBM streams from the
//           first microsecond
//   T1      rank r of the cluster owns k-blocks [num_kb*r/8, num_kb*(r+1)/8):
//           its X columns (all M rows) -> smem by bulk copies; outlier bits of its
//           columns are final (the owner sees every row); per-row partial absmax
//           over its keep columns; both broadcast to every rank (st.shared::cluster)
//                                                               cluster barrier
//   T2      row absmax = max of the 8 partials (identical in every rank); codes of
//           its k-blocks, each written ONCE into the shared-memory B-operand
//           panel of every rank whose stream-K units use it   cluster barrier
//   then    warp 0  TMA producer of the remaining weight tiles
//           warp 1  MMA: D[n, m] += WqT[n, k] Xq[m, k]  (tcgen05 kind::i8, swap-AB:
//                   M = 128 weight rows, N = 16 token rows, K = 32; B from the panel)
//           warps 4-7  epilogue, one thread per weight row n: the column fixup
//                   (a column whose cached maximiser row is an outlier row gets its
//                   keep-row amax from the cached candidates and its exact int32 dot
//                   from the cached second-candidate codes q2, on CUDA cores while
//                   the MMAs run), dequant + outlier term, stores coalesced along n
// The (n-tile, k-block) space is split evenly over the CTAs (stream-K); a tile
// split between CTAs is finished by the CTA holding its first k-block, which
// adds the others' int32 partials (handed over through the workspace with
// per-tile arrival counters that the finisher resets: the counters must be zero
// when a workspace is first used, i8mm_linear_workspace_init).
//
// Same arithmetic as the prefill path, so outputs are bit-identical to it:
//   Xq / row amax / outlier set  : prologue.cu semantics (quantize.py:168-179,
//                                   gemm.py:203-211, 242)
//   column scales                : weights.cu weight-stationary fixup
//                                   (quantize.py:182-187 on w[keep, :])
//   epilogue                     : gemm_sm100.cu (gemm.py:120-147, 238, 244-247)
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <mutex>

#include "kernels.cuh"
#include "quant_common.cuh"
#include "sm100_ptx.cuh"

namespace i8mm {

bool make_tmap_i8_rows(CUtensorMap* map, const int8_t* base, int64_t rows, int64_t K, int64_t ld,
                       int box_rows);  // gemm_sm100.cu

namespace dec {

#ifndef DECODE_CL
#define DECODE_CL 8
#endif
constexpr int THREADS = 256;    // warp 0 TMA, 1 MMA, 2 TMEM alloc, 4-7 epilogue; all in T1/T2
constexpr int NWARPS = THREADS / 32;
constexpr int CL = DECODE_CL;   // cluster size (portable)
constexpr int WO_CAP = 16;      // outlier rows of W held in registers by the epilogue
constexpr int TILE_N = 128;     // weight rows per tile (the MMA's M)
constexpr int BK = 128;         // K bytes per stage (one SWIZZLE_128B row)
constexpr int UMMA_K = 32;
constexpr int A_BYTES = TILE_N * BK;  // 16 KB weight tile
constexpr int MAX_M = 16;       // token rows (the MMA's N is 16)
constexpr int MPAD = 16;
constexpr int B_BYTES = MPAD * BK;    // 2 KB panel slot (one k-block of codes)
// independent accumulators per tile buffer: consecutive MMAs into one accumulator
// serialise on the tensor pipe's latency (~0.1 us each at N = 16), so the 4 K-steps
// of a unit and the next units rotate over N_ACC accumulators (the epilogue adds
// them back, exact int32)
constexpr int N_ACC = 16;  // a power of two (rotation by mask)
constexpr uint32_t TMEM_COLS = 2 * N_ACC * 16;  // 2 tile buffers x N_ACC x 16 columns
constexpr int MAX_STAGES = 16;
constexpr int MAX_WORDS = 4096; // mask words (K <= 131072, the MAX_INNER_DIM guard)
constexpr int NSEG_PRE = 3;     // segments whose cached column data is loaded at kernel start
constexpr int WO_PRE_L2 = 16;   // outlier rows of W prefetched into L2 per segment
constexpr int SMEM_LIMIT = 227 * 1024;

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
// timeline stamp i of this CTA, 32 per CTA (dev tool: i8mm_debug_decode_timeline)
// (dev build only: see gemm_sm100.cu, I8MM_GEMM_DEVTOOLS)
#ifdef I8MM_GEMM_DEVTOOLS
constexpr bool kDevStamps = true;
#else
constexpr bool kDevStamps = false;
#endif
#define DSTAMP(ptr, i)                                                                 \
    do {                                                                               \
        if (kDevStamps && (ptr) != nullptr) (ptr)[blockIdx.x * 64 + (i)] = gtimer(); \
    } while (0)

// 8 consecutive fp16 of a row starting at `col` (zeros past K); 16-byte load
// when the row is aligned, element loads otherwise.
__device__ __forceinline__ uint4 load8(const __half* row, int64_t col, int64_t K, bool vec) {
    if (vec && col + 8 <= K) return *reinterpret_cast<const uint4*>(row + col);
    uint32_t h[8];
#pragma unroll
    for (int e = 0; e < 8; ++e)
        h[e] = col + e < K ? static_cast<uint32_t>(__half_as_ushort(row[col + e])) : 0u;
    return make_uint4(h[0] | h[1] << 16, h[2] | h[3] << 16, h[4] | h[5] << 16, h[6] | h[7] << 16);
}
__device__ __forceinline__ uint32_t half_bits(const uint4& q, int e) {
    const uint32_t w = e < 2 ? q.x : e < 4 ? q.y : e < 6 ? q.z : q.w;
    return (e & 1) ? (w >> 16) : (w & 0xFFFFu);
}

// ---------------------------------------------------------------- cluster
__device__ __forceinline__ uint32_t mapa_shared(const void* p, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_addr(p)), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_cluster_u32(uint32_t addr, uint32_t v) {
    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void st_cluster_v4(uint32_t addr, const uint4& v) {
    asm volatile("st.shared::cluster.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w)
                 : "memory");
}
// split cluster barrier: arrive early, wait before the first access to a peer's
// shared memory (every CTA of the cluster has then started)
__device__ __forceinline__ void cluster_arrive_relaxed() {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_arrive_release() {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
    asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
}
__device__ __forceinline__ void red_cluster_add(uint32_t addr, uint32_t v) {
    asm volatile("red.relaxed.cluster.shared::cluster.add.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote_release(uint32_t addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(addr) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
    uint32_t ok = 0;
    while (!ok)
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(smem_addr(bar)), "r"(parity)
            : "memory");
}
// L2 policy of the single-use weight stream: evict_first keeps the kernel's code,
// X, the outputs and the workspace resident while 100+ MB of weights pass through
__device__ __forceinline__ uint64_t weight_policy(int mode) {
    return mode == 0 ? l2_policy_evict_first() : l2_policy_evict_normal();
}
// Cross-cluster split-tile partials are self-validating: a slot word holds
// kPartEmpty until its contributor stores the sum (|sum| <= 127 * 127 * K <
// 2^31 - kPartEmpty's magnitude for K <= 131072, so no sum equals it), and the
// finisher puts kPartEmpty back after reading. No flag, fence or barrier: the
// finisher polls the data words themselves (relaxed, single-copy atomic).
constexpr int32_t kPartEmpty = static_cast<int32_t>(0x80808080u);  // byte-memset pattern 0x80
__device__ __forceinline__ int32_t ld_relaxed(const int32_t* p) {
    int32_t v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(int32_t* p, int32_t v) {
    asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Weight-stationary column fixup (weights.cu fixup_kernel semantics, quantize.py:
// 182-187 on w[keep, :]) for a column whose cached maximiser row cr[0] is an
// outlier row: the amax over the keep rows from the cached candidates cr/cv
// (rows / |w| bits, descending), or -1 when every candidate is an outlier row
// (the column must be scanned). src = 1: the column's new codes are its cached
// second-candidate row (q2).
__device__ __forceinline__ float fixup_amax(const int32_t (&cr)[kTopT], const uint16_t (&cv)[kTopT],
                                            const uint32_t* mask, int& src) {
    src = 0;
#pragma unroll
    for (int t = 1; t < kTopT; ++t) {
        if (cr[t] < 0) {
            src = t == 1;
            return 0.0f;
        }
        if (!bit_of(mask, cr[t])) {
            src = t == 1;
            return hbits_to_float(cv[t]);
        }
    }
    return -1.0f;
}

// 16 codes of one token row at columns k0..k0+15, from 16 fp16 values; outlier
// columns and columns past K give 0 (prologue.cu semantics). The token phase
// runs at 8 warps per SM, so it is latency-bound: the 16 fast roundings are
// straight-line, independent chains (code_fast without its branch), and the
// exact f64 tie-break runs afterwards for the ~1e-4 of elements that need it.
__device__ __noinline__ uint32_t codes16_fixup(uint32_t word, uint32_t bad, uint4 lo, uint4 hi, int base,
                                               double s) {  // by value: no stack copy of lo / hi per item
    for (int e = base; e < base + 4; ++e)
        if ((bad >> e) & 1u) {
            const float x = hbits_to_float(half_bits(e < 8 ? lo : hi, e & 7));
            const uint32_t c = static_cast<uint32_t>(static_cast<int>(code_of(x, s))) & 0xFFu;
            const int sh = (e - base) * 8;
            word = (word & ~(0xFFu << sh)) | (c << sh);
        }
    return word;
}

__device__ __forceinline__ uint4 codes16(const uint4& lo, const uint4& hi, uint32_t mbits, int64_t k0,
                                         int64_t K, float s32, double s) {
    // packed f32x2 arithmetic (FMUL2 / FADD2, round-to-nearest per lane: the same
    // values as the scalar form), code bytes gathered with byte permutes: the low
    // byte of t = pf + 1.5 * 2^23 is rint(pf) as two's complement
    constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23: t - kMagic = rint(pf)
    constexpr float kTie = 0.5f - 6.103515625e-05f;
    const int lim = K - k0 < 16 ? static_cast<int>(K - k0) : 16;
    uint32_t zmask = mbits & 0xFFFFu;  // bit e: code e is 0 (outlier column or past K)
    if (lim < 16) zmask |= (0xFFFFu << (lim > 0 ? lim : 0)) & 0xFFFFu;
    const uint32_t hw[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
    const float2 s2 = make_float2(s32, s32), mg = make_float2(kMagic, kMagic), nmg = make_float2(-kMagic, -kMagic);
    uint32_t tb[16];
    uint32_t bad = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const float2 x2 = __half22float2(*reinterpret_cast<const __half2*>(&hw[q]));
        const float2 pf = __fmul2_rn(x2, s2);
        const float2 t = __fadd2_rn(pf, mg);
        const float2 r = __fadd2_rn(t, nmg);
        const float2 d = __fadd2_rn(pf, make_float2(-r.x, -r.y));
        tb[2 * q] = __float_as_uint(t.x);
        tb[2 * q + 1] = __float_as_uint(t.y);
        bad |= (fabsf(d.x) < kTie ? 0u : 1u) << (2 * q);
        bad |= (fabsf(d.y) < kTie ? 0u : 1u) << (2 * q + 1);
    }
    bad &= ~zmask;
    uint32_t w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const uint32_t p01 = __byte_perm(tb[4 * q], tb[4 * q + 1], 0x0040);
        const uint32_t p23 = __byte_perm(tb[4 * q + 2], tb[4 * q + 3], 0x0040);
        w[q] = __byte_perm(p01, p23, 0x5410);
    }
    if (zmask) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint32_t z4 = (zmask >> (4 * q)) & 0xFu;
            w[q] &= ~(((z4 * 0x00204081u) & 0x01010101u) * 0xFFu);
        }
    }
    if (bad) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if ((bad >> (q * 4)) & 0xFu) w[q] = codes16_fixup(w[q], bad, lo, hi, q * 4, s);
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
}

struct __align__(8) Bars {
    uint64_t full[MAX_STAGES];   // weight tile landed
    uint64_t empty[MAX_STAGES];  // stage consumed by the MMAs
    uint64_t tmem_full[2];
    uint64_t tmem_empty[2];
    uint64_t xbar;               // bulk copies of the X slice landed
    uint64_t pbar;               // split-tile finisher: same-cluster contributors' partials added
    uint32_t tmem_slot;
    uint32_t nonfinite[CL];      // rank 0: every rank's NaN/Inf flag
    int32_t n_out;
    int32_t o_s[WO_CAP];         // first outlier columns (sorted)
    int32_t warp_sums[NWARPS];
    int32_t peer_start[CL];      // each rank's first k-block and unit count (panel slots)
    int32_t peer_len[CL];
    // epilogue: patched columns of the current segment
    int32_t n_ent;
    int32_t ent_j[TILE_N];       // tile row
    int32_t ent_src[TILE_N];     // 1: codes = cached q2 row, 0: re-derived from W, -1: needs a scan, -2: not patched
    float ent_a[TILE_N];         // the column's amax over the keep rows
    int32_t ent_of[TILE_N];      // per tile row: its entry or -1
    int32_t red[NWARPS * MAX_M];
};

struct Params {
    DecodeArgs a;
    int num_kb, n_tiles;
    int s1, s2;          // weight stages before / after the X slice area is released
    int pre;             // weight tiles loaded before the token phase (<= s1)
    int l2_prefetch;     // the CTA's remaining weight tiles are prefetched into L2 at the start
    int w_policy;        // 0: weight tiles evict_first (default), 1: evict_normal (A/B)
    int slots;           // panel slots (k-blocks of codes) per CTA
    int xs_cached;       // the X slice is kept in smem (the ring's stages s1..s2-1) for T2
    int64_t xs_ld;       // halves per cached X-slice row
    int64_t total_units;
    unsigned long long* dbg;  // per-CTA %globaltimer stamps (dev tool), nullable
    int dbg_mode;             // dev build A/B: bit 0 local panel stores only, bit 1 no code math, bit 2 no Xq copy,
                              // bit 3 no token phase at all
};

// dynamic shared memory after the weight ring and the panel (kb_max: k-blocks a
// rank owns, at most; their panel destinations are a kb_max x CL int16 table)
__host__ __device__ inline size_t smem_tail(int64_t nwords, int64_t kb_max) {
    return static_cast<size_t>((nwords + 3) & ~int64_t(3)) * 4 + CL * MAX_M * 4 +
           MAX_M * (sizeof(double) + 3 * sizeof(float)) + MAX_M * WO_CAP * sizeof(float) +
           2 * TILE_N * MAX_M * sizeof(int32_t) + static_cast<size_t>((kb_max * CL + 3) & ~int64_t(3)) * 2 +
           sizeof(Bars) + 64;
}

template <int EPI>
__device__ __forceinline__ void store_out(const DecodeArgs& a, int64_t m, int64_t n, float v) {
    if constexpr (EPI == EPI_F16)
        reinterpret_cast<__half*>(a.y)[m * a.ldy + n] = __float2half_rn(v);
    else
        reinterpret_cast<float*>(a.y)[m * a.ldy + n] = v;
}

// y[m, n] from the exact int32 accumulator c (same op order as gemm_sm100.cu);
// the outlier term walks o_s (the first WO_CAP outlier columns), or the whole
// shared-memory mask in ascending column order when there are more
template <int EPI>
__device__ __forceinline__ float epi_value(const DecodeArgs& a, const int32_t* o_s, const uint32_t* smask,
                                           int64_t nwords, int32_t c, int64_t m, int64_t n, float rowf,
                                           float colf, float aw, int n_out, const float* sxo,
                                           const float (&wr)[WO_CAP]) {
    if constexpr (EPI == EPI_F32_EXACT) {
        const double sx = 127.0 / static_cast<double>(rowf);
        const double sw = 127.0 / static_cast<double>(amax_or_127(aw));
        const double d = __dmul_rn(sx, sw);
        float v = __double2float_rn(__ddiv_rn(static_cast<double>(c), d));
        if (n_out > 0) {
            double hacc = 0.0;
            auto term = [&](int64_t k) {
                const double xv = __half2float(a.x[m * a.ldx + k]);
                const double wv = __half2float(a.w[k * a.ldw + n]);
                hacc = __dadd_rn(hacc, __dmul_rn(xv, wv));
            };
            if (n_out <= WO_CAP) {
                for (int o = 0; o < n_out; ++o) term(o_s[o]);
            } else {
                for (int64_t w = 0; w < nwords; ++w)
                    for (uint32_t bits = smask[w]; bits; bits &= bits - 1) term((w << 5) + __ffs(bits) - 1);
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
        } else if (n_out > WO_CAP) {
            for (int64_t w = 0; w < nwords; ++w)
                for (uint32_t bits = smask[w]; bits; bits &= bits - 1) {
                    const int64_t k = (w << 5) + __ffs(bits) - 1;
                    v = fmaf(__half2float(a.x[m * a.ldx + k]), __half2float(a.w[k * a.ldw + n]), v);
                }
        }
        return v;
    }
}

// sorted outlier columns from the full mask in shared memory, by the nthr
// threads t = 0..nthr-1 (whole warps, synchronised on named barrier bar_id):
// the first WO_CAP to o_s, all of them to o_idx when non-null, the count to n_out
__device__ void compact_mask(const uint32_t* __restrict__ smask, int64_t nwords, Bars* bars,
                             int32_t* __restrict__ o_idx, int t, int nthr, uint32_t bar_id) {
    const int64_t per = (nwords + nthr - 1) / nthr;
    const int64_t w0 = t * per;
    const int64_t w1 = w0 + per < nwords ? w0 + per : nwords;
    int32_t local = 0;
    for (int64_t w = w0; w < w1; ++w) local += __popc(smask[w]);
    const int lane = t & 31, wid = t >> 5, nw = nthr >> 5;
    int32_t incl = local;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int32_t v = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += v;
    }
    if (lane == 31) bars->warp_sums[wid] = incl;
    named_bar_sync(bar_id, nthr);
    if (wid == 0) {
        int32_t v = lane < nw ? bars->warp_sums[lane] : 0;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int32_t u = __shfl_up_sync(0xffffffffu, v, d);
            if (lane >= d) v += u;
        }
        if (lane < nw) bars->warp_sums[lane] = v;
    }
    named_bar_sync(bar_id, nthr);
    int32_t pos = incl - local + (wid > 0 ? bars->warp_sums[wid - 1] : 0);
    for (int64_t w = w0; w < w1; ++w) {
        uint32_t m = smask[w];
        while (m) {
            const int b = __ffs(m) - 1;
            m &= m - 1;
            const int32_t k = static_cast<int32_t>((w << 5) + b);
            if (pos < WO_CAP) bars->o_s[pos] = k;
            if (o_idx != nullptr) o_idx[pos] = k;
            ++pos;
        }
    }
    if (t == nthr - 1) bars->n_out = pos;
    named_bar_sync(bar_id, nthr);
}

// 16 token columns of this thread's weight row: sum of the n_used accumulators
// the segment wrote (min(N_ACC, 4 x its units))
__device__ __forceinline__ void tmem_row16(uint32_t taddr, int n_used, uint32_t (&r)[16]) {
    // accumulator pairs (32 consecutive columns) per load, one wait per pair: a
    // wait per accumulator made the sum a chain of n_used TMEM round trips
    if (n_used & 1) {
        tmem_ld_32x32b_x16(taddr, r);
    } else {
#pragma unroll
        for (int e = 0; e < 16; ++e) r[e] = 0u;
    }
    for (int j = n_used & 1; j < n_used; j += 2) {
        uint32_t t[32];
        tmem_ld_32x32b_x32(taddr + static_cast<uint32_t>(j * MPAD), t);
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 16; ++e) r[e] += t[e] + t[16 + e];
    }
    tmem_ld_wait();
}

template <int EPI>
__global__ void __launch_bounds__(THREADS, 1)
    decode_kernel(const __grid_constant__ CUtensorMap tmap_w, const Params p) {
    const DecodeArgs& a = p.a;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u);
    const int64_t M = a.M, K = a.K, N = a.N;
    const int64_t nwords = (K + 31) >> 5;
    uint8_t* ring = smem;
    uint8_t* panel = ring + static_cast<size_t>(p.s2) * A_BYTES;
    uint32_t* smask = reinterpret_cast<uint32_t*>(panel + static_cast<size_t>(p.slots) * B_BYTES);
    uint32_t* spart = smask + ((nwords + 3) & ~int64_t(3));            // [CL][MAX_M] partial row amax bits
    double* sscale = reinterpret_cast<double*>(spart + CL * MAX_M);     // [M]
    float* sscale32 = reinterpret_cast<float*>(sscale + MAX_M);
    float* srow = sscale32 + MAX_M;                                     // amax_or_127(row amax)
    float* samax = srow + MAX_M;                                        // row amax
    float* sxo = samax + MAX_M;                                         // [M][WO_CAP] x[:, O]
    int32_t* pdot = reinterpret_cast<int32_t*>(sxo + MAX_M * WO_CAP);    // [TILE_N][MAX_M]
    const int kb_max = (p.num_kb + CL - 1) / CL;
    int32_t* racc = pdot + TILE_N * MAX_M;  // [MAX_M][TILE_N] same-cluster contributors' partial sums
    int16_t* sdst = reinterpret_cast<int16_t*>(racc + TILE_N * MAX_M);  // [kb_max][CL] panel slot or -1
    Bars* bars = reinterpret_cast<Bars*>(sdst + ((kb_max * CL + 3) & ~3));
    __half* xs = reinterpret_cast<__half*>(ring + static_cast<size_t>(p.s1) * A_BYTES);  // T1/T2 only

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t crank = cluster_ctarank();
    const uint32_t clu = blockIdx.x / CL;
    const bool lead = clu == 0;  // cluster 0 also publishes the call's token-side results
    // unit indices fit 32 bits (decode_fits bounds T * G < 2^31): 32-bit division on
    // the producer / MMA / finisher paths (a 64-bit one is a ~100-instruction call)
    const uint32_t T = static_cast<uint32_t>(p.total_units);
    const uint32_t Gu = gridDim.x;
    const int u_begin = static_cast<int>(T * blockIdx.x / Gu);
    const int u_end = static_cast<int>(T * (blockIdx.x + 1) / Gu);
    const int L = u_end - u_begin;
    const int num_kb = p.num_kb;
    const int S2 = p.s2;
    const bool all_kb = L >= num_kb;  // the panel holds every k-block (slot = kb)
    // k-blocks (and X columns, mask words) this rank owns in T1/T2
    const int kb_lo = num_kb * static_cast<int>(crank) / CL, kb_hi = num_kb * static_cast<int>(crank + 1) / CL;
    const int64_t c0 = static_cast<int64_t>(kb_lo) * BK, c1 = min(static_cast<int64_t>(kb_hi) * BK, K);
    const int64_t w0 = static_cast<int64_t>(kb_lo) * 4, w1 = min(static_cast<int64_t>(kb_hi) * 4, nwords);
    const int nv = c1 > c0 ? static_cast<int>((c1 - c0 + 7) / 8) : 0;  // 8-column vectors
    const int nfull = c1 > c0 ? static_cast<int>((c1 - c0) / 8) : 0;
    const bool cached = p.xs_cached != 0;
    const int64_t xs_ld = p.xs_ld;

    DSTAMP(p.dbg, 0);
    const bool bulk = cached && a.x_vec;
    // split tile this CTA finishes (at most one: the last tile start in its range
    // when that tile runs past the range), and its contributors: those in this
    // cluster add their partials into racc (distributed shared memory), the
    // others hand them over through the workspace
    int fin_local = 0, fin_cross = 0;
    {
        const int t_last = (u_end - 1) / num_kb;
        const int t0u = t_last * num_kb;
        if (t0u >= u_begin && t0u + num_kb > u_end) {
            const uint32_t cl = (static_cast<uint32_t>(t0u + num_kb) * Gu - 1) / T;
            const uint32_t cl_in = min(cl, clu * CL + CL - 1);
            fin_local = static_cast<int>(cl_in - blockIdx.x);
            fin_cross = static_cast<int>(cl - cl_in);
        }
    }
    // ================= setup: barriers, the weight prefetch (independent of this
    // call's tokens), then the X slice (written by the preceding kernel) first
    if (tid == 0) {
        tma_prefetch_desc(&tmap_w);
        for (int s = 0; s < S2; ++s) {
            mbar_init(&bars->full[s], 1);
            mbar_init(&bars->empty[s], 1);
        }
        for (int q = 0; q < 2; ++q) {
            mbar_init(&bars->tmem_full[q], 1);
            mbar_init(&bars->tmem_empty[q], 4);
        }
        mbar_init(&bars->xbar, 1);
        mbar_init(&bars->pbar, max(1, fin_local));
        fence_mbarrier_init();
        const uint64_t pol_w = weight_policy(p.w_policy);
        for (int i = 0; i < min(p.pre, L); ++i) {
            const int u = u_begin + i;
            mbar_arrive_expect_tx(&bars->full[i], A_BYTES);
            tma_load_2d(&tmap_w, &bars->full[i], ring + static_cast<size_t>(i) * A_BYTES, (u % num_kb) * BK,
                        (u / num_kb) * TILE_N, pol_w);
        }
    }
    // Everything up to the dependency wait touches only this call's immutable
    // inputs (the cached codes and candidates, written by i8mm_linear_prepare,
    // whose kernels never trigger early) and shared memory, so it overlaps the
    // preceding kernel's tail: CTAs of this grid start on SMs as they free up.
    // panel destinations of this rank's k-blocks: slot in each rank's panel, or -1
    for (int i = tid; i < (kb_hi - kb_lo) * CL; i += THREADS) {
        const int kbi = i / CL, q = i - kbi * CL;
        const uint32_t g = clu * CL + q;
        const int ub = static_cast<int>(T * g / Gu), len = static_cast<int>(T * (g + 1) / Gu) - ub;
        const int kb = kb_lo + kbi;
        int slot;
        if (len >= num_kb) {
            slot = kb;
        } else {
            slot = kb - ub % num_kb;
            if (slot < 0) slot += num_kb;
            if (slot >= len) slot = -1;
        }
        sdst[i] = static_cast<int16_t>(slot);
    }
    if (tid == 0) DSTAMP(p.dbg, 22);
    if (warp == 2) tmem_alloc<TMEM_COLS>(&bars->tmem_slot);
    if (tid == 64) DSTAMP(p.dbg, 23);
    // cached (immutable) candidates of the first segments' columns, in registers
    // through the token phase: the column fixup needs no global round trip
    int32_t pre_cr[NSEG_PRE][kTopT];
    uint16_t pre_cv[NSEG_PRE][kTopT];
    float pre_aw[NSEG_PRE];
    if (warp >= 4) {
        const int n_local = tid - 128;
        int u = u_begin;
#pragma unroll
        for (int sg = 0; sg < NSEG_PRE; ++sg) {
            const int tile = u / num_kb;
            const int64_t n = static_cast<int64_t>(tile) * TILE_N + n_local;
            const bool ok = u < u_end && n < N;
#pragma unroll
            for (int t = 0; t < kTopT; ++t) {
                pre_cr[sg][t] = ok ? __ldg(a.cand_r + t * N + n) : -1;
                pre_cv[sg][t] = ok && t > 0 ? __ldg(a.cand_v + t * N + n) : uint16_t(0);
            }
            pre_aw[sg] = ok ? __ldg(a.amax_full + n) : 127.0f;
            u = min(u_end, (tile + 1) * num_kb);
        }
    }
    if (tid == 128) DSTAMP(p.dbg, 24);
    // (token rows M..15 of the panel slots are left as they are: they only feed
    // accumulator columns m >= M, which no path reads)
    for (int64_t w = w0 + tid; w < w1; w += THREADS) smask[w] = 0u;
    if (fin_local > 0)  // contributors add into it after cluster barrier 2
        for (int i = tid; i < static_cast<int>(M) * TILE_N; i += THREADS) racc[i] = 0;
    if (tid == 0) DSTAMP(p.dbg, 19);
    // X and the workspace (written / read by the preceding kernels) after the wait
    pdl_wait();
    pdl_trigger();
    if (tid == 0) DSTAMP(p.dbg, 20);
    if (bulk && tid == 0) {
        const uint32_t row_bytes = static_cast<uint32_t>(nfull) * 16u;
        if (row_bytes > 0) {
            mbar_arrive_expect_tx(&bars->xbar, row_bytes * static_cast<uint32_t>(M));
            for (int64_t m = 0; m < M; ++m) bulk_load_1d(xs + m * xs_ld, a.x + m * a.ldx + c0, row_bytes, &bars->xbar);
        } else {
            mbar_arrive(&bars->xbar);
        }
    }
    if (tid == 0) DSTAMP(p.dbg, 21);
    // the rest of this CTA's weight tiles -> L2 now: a CTA's TMA engine keeps only
    // a few tiles in flight, L2 prefetches have no such cap, so HBM streams the
    // layer at full rate under the token phase and the ring's later loads hit L2
    if (warp == 3 && p.l2_prefetch)
        for (int i = min(p.pre, L) + lane; i < L; i += 32) {
            const int u = u_begin + i;
            tma_prefetch_l2_2d(&tmap_w, (u % num_kb) * BK, (u / num_kb) * TILE_N);
        }
    if (bulk && nv > nfull)  // ragged last vector (K % 8 != 0): element loads
        for (int64_t m = tid; m < M; m += THREADS)
            *reinterpret_cast<uint4*>(xs + m * xs_ld + nfull * 8) = load8(a.x + m * a.ldx, c0 + nfull * 8, K, false);
    if (tid == 0) DSTAMP(p.dbg, 25);
    cluster_arrive_relaxed();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = bars->tmem_slot;
    DSTAMP(p.dbg, 1);

    // ================= T1: X slice, outlier bits, row partials -> every rank
    {
    const uint32_t thr = a.thr_bits_dev != nullptr ? __ldcg(a.thr_bits_dev) : a.thr_bits;
    if (bulk) mbar_wait(&bars->xbar, 0);
    DSTAMP(p.dbg, 2);
    uint32_t nf = 0;
    for (int i = tid; i < static_cast<int>(M) * nv; i += THREADS) {
        const int m = i / nv, v = i - m * nv;
        uint4 q;
        if (bulk) {
            q = *reinterpret_cast<const uint4*>(xs + m * xs_ld + v * 8);
        } else {
            q = load8(a.x + m * a.ldx, c0 + v * 8, K, a.x_vec);
            if (cached) *reinterpret_cast<uint4*>(xs + m * xs_ld + v * 8) = q;
        }
        uint32_t fl = 0;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const uint32_t h = half_bits(q, e);
            fl |= ((h & 0x7FFFu) >= thr ? 1u : 0u) << e;
            nf |= (h & 0x7C00u) == 0x7C00u ? 1u : 0u;
        }
        if (fl) atomicOr(smask + w0 + (v >> 2), fl << ((v & 3) * 8));
    }
    if (tid == 0) DSTAMP(p.dbg, 10);
    nf = __syncthreads_or(nf);
    cluster_wait();  // every peer is running: its shared memory can be written
    if (tid == 0) DSTAMP(p.dbg, 11);
    for (int m = warp; m < static_cast<int>(M); m += NWARPS) {  // warp per row
        uint32_t mx = 0;
        for (int v = lane; v < nv; v += 32) {
            const uint4 q = cached ? *reinterpret_cast<const uint4*>(xs + m * xs_ld + v * 8)
                                   : load8(a.x + m * a.ldx, c0 + v * 8, K, a.x_vec);
            const uint32_t mb = smask[w0 + (v >> 2)] >> ((v & 3) * 8);
#pragma unroll
            for (int e = 0; e < 8; ++e)
                if (!((mb >> e) & 1u)) mx = max(mx, half_bits(q, e) & 0x7FFFu);
        }
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, d));
        if (lane < CL) st_cluster_u32(mapa_shared(spart + crank * MAX_M + m, lane), mx);
    }
    if (tid == 0) DSTAMP(p.dbg, 12);
    const int nown = static_cast<int>(w1 - w0);
    for (int i = tid; i < nown * CL; i += THREADS) {
        const int q = i / nown, w = static_cast<int>(w0) + (i - q * nown);
        if (q != static_cast<int>(crank)) st_cluster_u32(mapa_shared(smask + w, q), smask[w]);
    }
    if (tid == 0) st_cluster_u32(mapa_shared(&bars->nonfinite[crank], 0), nf);
    if (tid == 0) DSTAMP(p.dbg, 13);
    cluster_sync_all();  // 1: full mask and all partials in every rank
    DSTAMP(p.dbg, 3);

    // ================= T2: row scales, outlier list, codes -> every rank's panel
    for (int m = tid; m < static_cast<int>(M); m += THREADS) {
        uint32_t mx = 0;
#pragma unroll
        for (int q = 0; q < CL; ++q) mx = max(mx, spart[q * MAX_M + m]);
        const float amax = hbits_to_float(mx);
        const double s = scale_of(amax);
        sscale[m] = s;
        sscale32[m] = static_cast<float>(s);
        samax[m] = amax;
        srow[m] = amax_or_127(amax);
        if (lead && crank == 0) {
            a.row_amax[m] = amax;
            a.ramax_bits[m] = mx;
        }
    }
    __syncthreads();  // row scales (O is compacted by the epilogue warps after barrier 2)
    if (tid == 0) DSTAMP(p.dbg, 14);
    const int nkb = kb_hi - kb_lo;
    // codes of this rank's k-blocks: item = (k-block, row, 16-column chunk); row
    // and chunk from a multiply-shift (exact for the ranges here: rest < 2^13)
    const uint32_t m8 = static_cast<uint32_t>(M) * 8u;
    const uint32_t inv_m8 = (1u << 20) / m8 + 1u;
    // every rank's panel base in the cluster window, computed once: a store is
    // then base + slot offset, with no per-store address translation
    uint32_t peer_panel[CL];
#pragma unroll
    for (int q = 0; q < CL; ++q) peer_panel[q] = mapa_shared(panel, static_cast<uint32_t>(q));
    for (int it = tid; it < nkb * static_cast<int>(m8); it += THREADS) {
        if (tid == 0 && it == 0) DSTAMP(p.dbg, 32);
        if (tid == 0 && it == THREADS) DSTAMP(p.dbg, 34);
        const int kbi = static_cast<int>((static_cast<uint32_t>(it) * inv_m8) >> 20);
        const int rem = it - kbi * static_cast<int>(m8);
        const int m = rem >> 3, ch = rem & 7;
        const int kb = kb_lo + kbi;
        const int64_t k0 = static_cast<int64_t>(kb) * BK + ch * 16;
        uint4 code = make_uint4(0u, 0u, 0u, 0u);
        if (k0 < K && !(kDevStamps && (p.dbg_mode & 2))) {
            uint4 lo, hi;
            if (cached) {
                lo = *reinterpret_cast<const uint4*>(xs + m * xs_ld + (k0 - c0));
                hi = *reinterpret_cast<const uint4*>(xs + m * xs_ld + (k0 - c0) + 8);
            } else {
                lo = load8(a.x + m * a.ldx, k0, K, a.x_vec);
                hi = load8(a.x + m * a.ldx, k0 + 8, K, a.x_vec);
            }
            const uint32_t mbits = (smask[k0 >> 5] >> (k0 & 31)) & 0xFFFFu;
            code = codes16(lo, hi, mbits, k0, K, sscale32[m], sscale[m]);
            if (tid == 0 && it == 0) DSTAMP(p.dbg, 33);
            if (lead && !(kDevStamps && (p.dbg_mode & 4)))
                *reinterpret_cast<uint4*>(a.xq + m * a.ldq + k0) = code;  // workspace Xq (views)
        }
        const uint32_t off = static_cast<uint32_t>(m * BK + ((ch ^ (m & 7)) * 16));
        // the k-block's destination slots, read once (CL int16 = one 16-byte row
        // for CL = 8): the stores below carry no memory clobber, so nothing
        // forces a re-read between them (the proxy fence and cluster barrier 2
        // order them before any use)
        int16_t dsl[CL];
#pragma unroll
        for (int q = 0; q < CL; ++q) dsl[q] = sdst[kbi * CL + q];
#pragma unroll
        for (int q = 0; q < CL; ++q) {
            const int slot = dsl[q];
            if (slot < 0) continue;
            if (kDevStamps && (p.dbg_mode & 1))
                *reinterpret_cast<uint4*>(panel + static_cast<size_t>(slot) * B_BYTES + off) = code;
            else
                asm volatile("st.shared::cluster.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(
                                 peer_panel[q] + static_cast<uint32_t>(slot) * B_BYTES + off),
                             "r"(code.x), "r"(code.y), "r"(code.z), "r"(code.w));
        }
    }
    if (tid == 0) DSTAMP(p.dbg, 15);
    if (tid == 128) DSTAMP(p.dbg, 28);  // warp 4 codes done (dev: slot shared with the 3rd segment entry count)
    asm volatile("fence.proxy.async.shared::cluster;" ::: "memory");  // panels feed tcgen05.mma
    if (tid == 0) DSTAMP(p.dbg, 16);
    if (lead) {
        for (int64_t w = w0 + tid; w < w1; w += THREADS) a.mask[w] = smask[w];
        if (crank == CL - 1) {  // Xq padding columns K..ldq (whole 16-column chunks)
            const int64_t pad0 = (K + 15) / 16 * 16;
            for (int64_t i = tid; i < M * ((a.ldq - pad0) / 16); i += THREADS) {
                const int64_t per = (a.ldq - pad0) / 16;
                *reinterpret_cast<uint4*>(a.xq + (i / per) * a.ldq + pad0 + (i % per) * 16) = make_uint4(0u, 0u, 0u, 0u);
            }
        }
    }
    if (tid == 0) DSTAMP(p.dbg, 18);
    cluster_sync_all();  // 2: every panel complete; the X slice area becomes weight stages
    fence_proxy_async_smem();
    }
    DSTAMP(p.dbg, 4);

    // Producer and MMA loops keep their (tile, k-block, stage, phase) state
    // incrementally: a runtime integer division is a ~20-instruction dependent
    // chain, and at 4 small MMAs per unit it would pace the whole weight stream.
    if (warp == 0) {
        // ---------------- TMA producer: the remaining weight tiles
        if (lane == 0) {
            const uint64_t pol_w = weight_policy(p.w_policy);
            const int i0 = min(p.pre, L);
            int u = u_begin + i0;
            int tile = u / num_kb, kb = u - tile * num_kb;
            int s = i0 % S2;
            uint32_t ph = static_cast<uint32_t>((i0 / S2) & 1);
            for (int i = i0; i < L; ++i) {
                if (i >= S2) mbar_wait(&bars->empty[s], ph ^ 1u);
                mbar_arrive_expect_tx(&bars->full[s], A_BYTES);
                tma_load_2d(&tmap_w, &bars->full[s], ring + static_cast<size_t>(s) * A_BYTES, kb * BK, tile * TILE_N,
                            pol_w);
                if (++kb == num_kb) {
                    kb = 0;
                    ++tile;
                }
                if (++s == S2) {
                    s = 0;
                    ph ^= 1u;
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer. At N = 16 tokens a tcgen05.mma moves only 4 KB of
        // weights, so the issue loop itself paces the stream: descriptors are
        // precomputed (+2 per 32-byte K step, + one slot / stage stride per unit) and
        // the accumulator rotates by mask (~60 cycles per MMA instead of ~240)
        const uint32_t idesc = idesc_i8(TILE_N, MPAD);
        constexpr int KS = BK / UMMA_K;  // 4 K-steps per unit
        const uint64_t a_base = smem_desc_k_sw128(smem_addr(ring));
        const uint64_t b_base = smem_desc_k_sw128(smem_addr(panel));
        int s = 0;
        uint32_t ph = 0;
        int kb = u_begin % num_kb;  // the unit's k-block; panel slot = kb (all_kb) or i
        int seg = 0;
        for (int u = u_begin; u < u_end; ++seg) {
            const int seg_end = min(u_end, (u / num_kb + 1) * num_kb);
            const int acc = seg & 1;
            mbar_wait(&bars->tmem_empty[acc], ((seg >> 1) & 1) ^ 1u);
            tc_fence_after();
            const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * N_ACC * MPAD);
            for (int kk = 0; u < seg_end; ++u, ++kk) {
                mbar_wait(&bars->full[s], ph);
                tc_fence_after();
                if (lane == 0) {
                    if (u == u_begin) DSTAMP(p.dbg, 5);
                    const int slot = all_kb ? kb : u - u_begin;
                    const uint64_t ad = a_base + static_cast<uint64_t>(s * (A_BYTES >> 4));
                    const uint64_t bd = b_base + static_cast<uint64_t>(slot * (B_BYTES >> 4));
                    const uint32_t d = d_tmem + static_cast<uint32_t>(((kk * KS) & (N_ACC - 1)) * MPAD);
                    const uint32_t accum = kk * KS >= N_ACC ? 1u : 0u;  // fresh on the first use
#pragma unroll
                    for (int k = 0; k < KS; ++k)
                        mma_i8(d + static_cast<uint32_t>(k * MPAD), ad + 2 * k, bd + 2 * k, idesc, accum);
                    mma_commit(&bars->empty[s]);
                }
                __syncwarp();
                if (++kb == num_kb) kb = 0;
                if (++s == S2) {
                    s = 0;
                    ph ^= 1u;
                }
            }
            if (lane == 0) mma_commit(&bars->tmem_full[acc]);
            __syncwarp();
        }
        if (lane == 0) DSTAMP(p.dbg, 6);
    } else if (warp == 2 || warp == 3) {
        // ---------------- idle warps 2-3: the sorted outlier list (and the lead CTA's O
        // outputs), L2 prefetches of W[O, tile], x[:, O] into shared memory; the
        // epilogue waits for them (named barrier 4) only before its first finishing
        // segment, so a leading contributor segment hands its partials over first
        const int t = tid - 64;
        compact_mask(smask, nwords, bars, lead && crank == 0 ? a.o_idx : nullptr, t, 64, 3);
        if (lead && crank == 0 && t == 0) {
            *a.o_count = bars->n_out;
            uint32_t any = 0;  // every rank's NaN/Inf flag landed before barrier 1
            for (int q = 0; q < CL; ++q) any |= bars->nonfinite[q];
            if (a.nonfinite != nullptr) *a.nonfinite = any ? 1 : 0;
        }
        const int n_out = bars->n_out;
        const int n_o = n_out <= WO_CAP ? n_out : 0;
        const int n_o0 = min(n_out, WO_PRE_L2);
        int u = u_begin;
        for (int sg = 0; sg < NSEG_PRE && u < u_end; ++sg) {
            const int tile = u / num_kb;
            if (t < n_o0) {
                const int64_t n0 = static_cast<int64_t>(tile) * TILE_N;
                const int64_t cols = min(static_cast<int64_t>(TILE_N), N - n0);
                const uint32_t bytes = static_cast<uint32_t>(cols * 2) & ~15u;
                if (bytes && a.w_vec)
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                                     a.w + static_cast<int64_t>(bars->o_s[t]) * a.ldw + n0),
                                 "r"(bytes)
                                 : "memory");
            }
            u = min(u_end, (tile + 1) * num_kb);
        }
        for (int i = t; i < static_cast<int>(M) * n_o; i += 64) {
            const int m = i / n_o, o = i - m * n_o;
            sxo[m * WO_CAP + o] = __half2float(a.x[m * a.ldx + bars->o_s[o]]);
        }
        asm volatile("bar.arrive 4, 192;" ::: "memory");
    } else if (warp >= 4) {
        // ---------------- epilogue: thread = weight row n of the tile
        const int et = tid - 128;
        // the patched columns' cached q2 rows -> L2 while the first MMAs run
        // (the outlier list, W[O, tile] prefetches and x[:, O] are warps 2-3's)
        {
            int u = u_begin;
#pragma unroll
            for (int sg = 0; sg < NSEG_PRE; ++sg) {
                const int tile = u / num_kb;
                const int seg_end = min(u_end, (tile + 1) * num_kb);
                if (u < u_end) {
                    const int64_t n = static_cast<int64_t>(tile) * TILE_N + et;
                    if (n < N && pre_cr[sg][0] >= 0 && bit_of(smask, pre_cr[sg][0])) {
                        int src;
                        const float an = fixup_amax(pre_cr[sg], pre_cv[sg], smask, src);
                        if (src == 1 && an != pre_aw[sg]) {
                            const int k_lo = (u % num_kb) * BK, k_hi = min((seg_end - 1) % num_kb + 1, num_kb) * BK;
                            if (k_hi > k_lo)
                                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.q2 + n * a.ldq + k_lo),
                                             "r"(static_cast<uint32_t>(k_hi - k_lo))
                                             : "memory");
                        }
                    }
                }
                u = seg_end;
            }
        }
        int n_out = 0, n_o = 0;
        bool o_ready = false;  // warps 2-3's outlier list (named barrier 4)
        const int n_local = et;
        const int quad = warp & 3;
        // closing barrier, split: a CTA adds into a peer's shared memory only in its
        // first segment, and only when that segment continues a tile an earlier CTA of
        // this cluster started; every other epilogue thread arrives right away (the
        // wait is at the very end)
        bool arrived = true;
        {
            const uint32_t t0 = static_cast<uint32_t>(u_begin / num_kb * num_kb);
            const uint32_t cf0 = ((t0 + 1) * Gu - 1) / T;
            if (L > 0 && static_cast<uint32_t>(u_begin) != t0 && cf0 / CL == clu) arrived = false;
        }
        if (arrived) cluster_arrive_release();
        if (et == 0) DSTAMP(p.dbg, 35);
        int seg = 0;
        for (int u = u_begin; u < u_end; ++seg) {
            const int tile = u / num_kb;
            const int su0 = u;
            const int seg_end = min(u_end, (tile + 1) * num_kb);
            const bool full = seg_end - u == num_kb;
            u = seg_end;
            const int acc = seg & 1;
            const int64_t n = static_cast<int64_t>(tile) * TILE_N + n_local;
            const bool n_ok = n < N;
            int32_t cr[kTopT];
            uint16_t cv[kTopT];
            float aw;
            if (seg < NSEG_PRE) {
#pragma unroll
                for (int t = 0; t < kTopT; ++t) {
                    cr[t] = seg == 0 ? pre_cr[0][t] : seg == 1 ? pre_cr[1][t] : pre_cr[2][t];
                    cv[t] = seg == 0 ? pre_cv[0][t] : seg == 1 ? pre_cv[1][t] : pre_cv[2][t];
                }
                aw = seg == 0 ? pre_aw[0] : seg == 1 ? pre_aw[1] : pre_aw[2];
            } else {
#pragma unroll
                for (int t = 0; t < kTopT; ++t) {
                    cr[t] = n_ok ? __ldg(a.cand_r + t * N + n) : -1;
                    cv[t] = n_ok && t > 0 ? __ldg(a.cand_v + t * N + n) : uint16_t(0);
                }
                aw = n_ok ? __ldg(a.amax_full + n) : 127.0f;
            }
            float wr[WO_CAP];
            const int64_t n0 = static_cast<int64_t>(tile) * TILE_N;
            // a contributor segment (not full, tile started by another CTA) hands raw
            // partials over: it needs no W[O, tile]
            const bool contrib_seg = !full && ((static_cast<uint32_t>(tile * num_kb) + 1) * Gu - 1) / T != blockIdx.x;
            if (!contrib_seg && !o_ready) {
                named_bar_sync(4, 192);
                o_ready = true;
                n_out = bars->n_out;
                n_o = n_out <= WO_CAP ? n_out : 0;
            }
            if (contrib_seg) {
#pragma unroll
                for (int o = 0; o < WO_CAP; ++o) wr[o] = 0.0f;
            } else if (EPI != EPI_F32_EXACT && n_o > 0 && a.w_vec && n0 + TILE_N <= N) {
                // W[O, tile] staged through the (idle) pdot area with 16-byte loads: one
                // load round trip instead of one per outlier row
                __half* sw = reinterpret_cast<__half*>(pdot);  // [WO_CAP][TILE_N]
                named_bar_sync(1, 128);  // the previous segment's pdot readers are done
                for (int i = et; i < n_o * (TILE_N / 8); i += 128) {
                    const int o = i / (TILE_N / 8), c8 = i - o * (TILE_N / 8);
                    *reinterpret_cast<uint4*>(sw + o * TILE_N + c8 * 8) = *reinterpret_cast<const uint4*>(
                        a.w + static_cast<int64_t>(bars->o_s[o]) * a.ldw + n0 + c8 * 8);
                }
                named_bar_sync(1, 128);
#pragma unroll
                for (int o = 0; o < WO_CAP; ++o) wr[o] = (o < n_o && n_ok) ? __half2float(sw[o * TILE_N + n_local]) : 0.0f;
                if (et == 0 && seg == 0) DSTAMP(p.dbg, 38);
            } else {
#pragma unroll
                for (int o = 0; o < WO_CAP; ++o)
                    wr[o] = (EPI != EPI_F32_EXACT && o < n_o && n_ok)
                                ? __half2float(a.w[static_cast<int64_t>(bars->o_s[o]) * a.ldw + n]) : 0.0f;
            }
            // -- column fixup: patched when the cached maximiser row is an outlier row
            //    and the keep-row amax differs (weights.cu fixup_kernel semantics)
            if (et == 0) bars->n_ent = 0;
            bars->ent_of[n_local] = -1;
            named_bar_sync(1, 128);
            if (n_ok && cr[0] >= 0 && bit_of(smask, cr[0])) {
                int src;
                const float a_new = fixup_amax(cr, cv, smask, src);
                if (a_new < 0.0f || a_new != aw) {
                    const int e = atomicAdd(&bars->n_ent, 1);
                    bars->ent_j[e] = n_local;
                    bars->ent_a[e] = a_new;
                    bars->ent_src[e] = a_new < 0.0f ? -1 : src;
                }
            }
            named_bar_sync(1, 128);
            const int n_ent = bars->n_ent;
            if (kDevStamps && et == 0 && p.dbg != nullptr) p.dbg[blockIdx.x * 64 + 26 + min(seg, 2)] = n_ent;
            if (n_ent > 0) {
                // every cached candidate an outlier row (rare): scan the column, warp per entry
                for (int e = quad; e < n_ent; e += 4) {
                    if (bars->ent_src[e] != -1) continue;
                    const int64_t j = static_cast<int64_t>(tile) * TILE_N + bars->ent_j[e];
                    uint32_t mx = 0;
                    for (int64_t k = lane; k < K; k += 32)
                        if (!bit_of(smask, k))
                            mx = max(mx, static_cast<uint32_t>(__half_as_ushort(a.w[k * a.ldw + j])) & 0x7FFFu);
#pragma unroll
                    for (int d = 16; d > 0; d >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, d));
                    __syncwarp();  // every lane has read ent_src[e]
                    if (lane == 0) {
                        const float an = hbits_to_float(mx);
                        bars->ent_a[e] = an;
                        bars->ent_src[e] = an != __ldg(a.amax_full + j) ? 0 : -2;
                    }
                }
                named_bar_sync(1, 128);
                for (int e = et; e < n_ent; e += 128)
                    if (bars->ent_src[e] >= 0) bars->ent_of[bars->ent_j[e]] = e;
                // exact int32 dots of the patched columns' codes with this segment's
                // panel codes (all 128 threads per column, on CUDA cores)
                const int nch = (seg_end - su0) * 8;
                for (int e = 0; e < n_ent; ++e) {
                    const int src = bars->ent_src[e];
                    if (src < 0) continue;
                    const int64_t j = static_cast<int64_t>(tile) * TILE_N + bars->ent_j[e];
                    const double sc = scale_of(bars->ent_a[e]);
                    const float s32 = static_cast<float>(sc);
                    int accd[MAX_M];
#pragma unroll
                    for (int m = 0; m < MAX_M; ++m) accd[m] = 0;
                    for (int c = et; c < nch; c += 128) {
                        const int uu = su0 + (c >> 3), ch = c & 7;
                        const int kb = uu % num_kb;
                        const int64_t k = static_cast<int64_t>(kb) * BK + ch * 16;
                        const int slot = all_kb ? kb : uu - u_begin;
                        uint4 cw;
                        if (src == 1) {
                            cw = __ldg(reinterpret_cast<const uint4*>(a.q2 + j * a.ldq + k));
                        } else {  // re-derived from W's column (its top-2 rows are outlier rows)
                            uint32_t b[16];
#pragma unroll
                            for (int e2 = 0; e2 < 16; ++e2) {
                                const int64_t kk = k + e2;
                                const int cd = (kk < K && !bit_of(smask, kk))
                                                   ? code_fast(__half2float(a.w[kk * a.ldw + j]), s32, sc) : 0;
                                b[e2] = static_cast<uint32_t>(cd) & 0xFFu;
                            }
                            cw = make_uint4(b[0] | b[1] << 8 | b[2] << 16 | b[3] << 24,
                                            b[4] | b[5] << 8 | b[6] << 16 | b[7] << 24,
                                            b[8] | b[9] << 8 | b[10] << 16 | b[11] << 24,
                                            b[12] | b[13] << 8 | b[14] << 16 | b[15] << 24);
                        }
                        const uint8_t* ps = panel + static_cast<size_t>(slot) * B_BYTES;
#pragma unroll
                        for (int m = 0; m < MAX_M; ++m) {
                            if (m >= M) break;
                            const uint4 xv = *reinterpret_cast<const uint4*>(ps + m * BK + ((ch ^ (m & 7)) * 16));
                            accd[m] = __dp4a(static_cast<int>(xv.x), static_cast<int>(cw.x), accd[m]);
                            accd[m] = __dp4a(static_cast<int>(xv.y), static_cast<int>(cw.y), accd[m]);
                            accd[m] = __dp4a(static_cast<int>(xv.z), static_cast<int>(cw.z), accd[m]);
                            accd[m] = __dp4a(static_cast<int>(xv.w), static_cast<int>(cw.w), accd[m]);
                        }
                    }
#pragma unroll
                    for (int m = 0; m < MAX_M; ++m) {
#pragma unroll
                        for (int d = 16; d > 0; d >>= 1) accd[m] += __shfl_xor_sync(0xffffffffu, accd[m], d);
                        if (lane == 0) bars->red[quad * MAX_M + m] = accd[m];
                    }
                    named_bar_sync(1, 128);
                    if (et < MAX_M)
                        pdot[e * MAX_M + et] = bars->red[et] + bars->red[MAX_M + et] + bars->red[2 * MAX_M + et] +
                                               bars->red[3 * MAX_M + et];
                    named_bar_sync(1, 128);
                }
            }
            const int my_ent = bars->ent_of[n_local];
            if (my_ent >= 0) aw = bars->ent_a[my_ent];
            const float colf = amax_or_127(aw) * (1.0f / 16129.0f);
            // split tile: the CTA holding its first unit finishes it (that unit range
            // is its last segment, or its only one); the others are their first
            // segments and hand over int32 partials
            const uint32_t t0 = static_cast<uint32_t>(tile * num_kb), t1 = t0 + num_kb;
            const uint32_t cf = ((t0 + 1) * Gu - 1) / T;
            const uint32_t cl = (t1 * Gu - 1) / T;
            // the finisher's cross-cluster partials: usually long ready (they are the
            // next cluster's first segments), so fetched while this segment's MMAs run
            uint32_t xpart[16];
#pragma unroll
            for (int jj = 0; jj < 16; ++jj) xpart[jj] = 0u;
            if (!full && cf == blockIdx.x && fin_cross > 0) {
                // each thread polls its own words of the contributors' slots until none
                // is kPartEmpty (bounded: a workspace never initialised traps instead
                // of hanging the GPU), then empties them for the next call
                // two contributors' slots per polling round (their words in flight together)
                const uint32_t need1 = (1u << M) - 1u;
                for (uint32_t c = cl - fin_cross + 1; c <= cl; c += 2) {
                    const bool two = c + 1 <= cl;
                    int32_t* src0 = a.c32 + static_cast<int64_t>(c) * (MAX_M * TILE_N) + n_local;
                    int32_t* src1 = src0 + MAX_M * TILE_N;
                    const uint32_t need = need1 | (two ? need1 << 16 : 0u);
                    uint32_t got = 0;
                    for (uint32_t spin = 0; got != need; ++spin) {
                        int32_t v[32];
#pragma unroll
                        for (int jj = 0; jj < 32; ++jj) {
                            const int row = jj & 15;
                            v[jj] = ((need >> jj) & 1u) && !((got >> jj) & 1u)
                                        ? ld_relaxed((jj < 16 ? src0 : src1) + row * TILE_N) : kPartEmpty;
                        }
#pragma unroll
                        for (int jj = 0; jj < 32; ++jj)
                            if (v[jj] != kPartEmpty) {
                                xpart[jj & 15] += static_cast<uint32_t>(v[jj]);
                                got |= 1u << jj;
                            }
                        if (spin > (1u << 22)) __trap();
                    }
#pragma unroll
                    for (int jj = 0; jj < 16; ++jj)
                        if (jj < M) {
                            st_relaxed(src0 + jj * TILE_N, kPartEmpty);
                            if (two) st_relaxed(src1 + jj * TILE_N, kPartEmpty);
                        }
                }
                if (et == 0 && seg == 0) DSTAMP(p.dbg, 36);
            }
            mbar_wait(&bars->tmem_full[acc], (seg >> 1) & 1);
            tc_fence_after();
            if (et == 0 && seg == 0) DSTAMP(p.dbg, 7);
            const uint32_t t_row = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) +
                                   static_cast<uint32_t>(acc * N_ACC * MPAD);
            uint32_t r[16];
            tmem_row16(t_row, min(N_ACC, (seg_end - su0) * (BK / UMMA_K)), r);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bars->tmem_empty[acc]);
            if (my_ent >= 0) {
#pragma unroll
                for (int jj = 0; jj < 16; ++jj) r[jj] = static_cast<uint32_t>(pdot[my_ent * MAX_M + jj]);
            }
            if (!full && cf != blockIdx.x && cf / CL == clu) {
                // the finisher is in this cluster: add into its racc, then one
                // release-arrive on its pbar per contributor CTA
                const uint32_t dst = mapa_shared(racc + n_local, cf % CL);
#pragma unroll
                for (int jj = 0; jj < 16; ++jj)
                    if (jj < M) red_cluster_add(dst + jj * TILE_N * 4, r[jj]);
                named_bar_sync(1, 128);
                if (et == 0) mbar_arrive_remote_release(mapa_shared(&bars->pbar, cf % CL));
                if (!arrived) {
                    cluster_arrive_release();
                    arrived = true;
                }
                continue;
            }
            if (!full && cf != blockIdx.x) {
                // self-validating partial words (kPartEmpty): no flag, no barrier
                int32_t* slotp = a.c32 + static_cast<int64_t>(blockIdx.x) * (MAX_M * TILE_N) + n_local;
#pragma unroll
                for (int jj = 0; jj < 16; ++jj)
                    if (jj < M) st_relaxed(slotp + jj * TILE_N, static_cast<int32_t>(r[jj]));
                if (et == 0) DSTAMP(p.dbg, 37);
                continue;
            }
            if (kDevStamps && et == 0 && p.dbg != nullptr) p.dbg[blockIdx.x * 64 + 29 + min(seg, 2)] = full ? 2 : (cf != blockIdx.x ? 0 : 1);
            if (!full) {  // finisher: the contributors' partials (this cluster's in racc, the others' global)
                if (fin_local > 0) {
                    mbar_wait_cluster(&bars->pbar, 0);
#pragma unroll
                    for (int jj = 0; jj < 16; ++jj)
                        if (jj < M) r[jj] += static_cast<uint32_t>(racc[jj * TILE_N + n_local]);
                }
#pragma unroll
                for (int jj = 0; jj < 16; ++jj) r[jj] += xpart[jj];
            }
            if (n_ok) {
#pragma unroll
                for (int jj = 0; jj < 16; ++jj) {
                    if (jj >= M) break;
                    store_out<EPI>(a, jj, n, epi_value<EPI>(a, bars->o_s, smask, nwords, static_cast<int32_t>(r[jj]),
                                                           jj, n, srow[jj], colf, aw, n_out, sxo, wr));
                }
            }
        }
        if (!o_ready) named_bar_sync(4, 192);  // pairs warps 2-3's arrive
        if (!arrived) cluster_arrive_release();
        if (et == 0) DSTAMP(p.dbg, 8);
    }
    if (warp < 4) cluster_arrive_release();
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc<TMEM_COLS>(tmem_base);
    }
    // Closing cluster barrier, split. After barrier 2 the only distributed-shared-
    // memory traffic is contributors adding into a finisher's racc and arriving on
    // its pbar, all in the contributors' first segment; every thread arrives once
    // its part of that is done (warps 0-3 after their roles, the epilogue after its
    // first segment), so no CTA leaves while a peer may still write its shared
    // memory, and a CTA waits only for its peers' first segments, not for the
    // cluster's slowest finisher (a full barrier here cost ~4 us per layer).
    cluster_wait();
    DSTAMP(p.dbg, 9);
}

}  // namespace dec

// ------------------------------------------------------------------ host
namespace {
struct DecodeGeom {
    int grid, s1, s2, slots, xs_cached;
    int64_t xs_ld, units;
    size_t smem;
    bool ok;
};

// active 8-CTA clusters of the decode kernel (one CTA per SM), measured once
int decode_clusters() {
    static int n = -1;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaFuncSetAttribute(dec::decode_kernel<EPI_F16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             dec::SMEM_LIMIT);
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(dec::CL * 64);
        cfg.blockDim = dim3(dec::THREADS);
        cfg.dynamicSmemBytes = dec::SMEM_LIMIT;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = dec::CL;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int c = 0;
        if (cudaOccupancyMaxActiveClusters(&c, dec::decode_kernel<EPI_F16>, &cfg) != cudaSuccess) c = 0;
        cudaGetLastError();
        n = c > 0 ? c : num_sms() / dec::CL;
    });
    return n;
}

DecodeGeom decode_geom(int64_t M, int64_t K, int64_t N) {
    using namespace dec;
    DecodeGeom g{};
    g.ok = false;
    if (M <= 0 || M > MAX_M || K <= 0 || N <= 0) return g;
    const int64_t nwords = (K + 31) / 32;
    if (nwords > MAX_WORDS) return g;
    const int64_t num_kb = (K + BK - 1) / BK;
    const int64_t n_tiles = (N + TILE_N - 1) / TILE_N;
    g.units = n_tiles * num_kb;
    int64_t grid = static_cast<int64_t>(decode_clusters()) * CL;
    const int64_t max_grid = (g.units / CL) * CL;  // every CTA gets at least one unit
    if (grid > max_grid) grid = max_grid;
    if (grid < CL) return g;
    g.grid = static_cast<int>(grid);
    if (g.units * grid >= (int64_t(1) << 31)) return g;
    const int64_t per = (g.units + grid - 1) / grid;
    g.slots = static_cast<int>(per < num_kb ? per : num_kb);
    const int64_t kb_max = (num_kb + CL - 1) / CL;  // k-blocks per rank (max)
    g.xs_ld = kb_max * BK;
    static int env_kb = -2;
    if (env_kb == -2) {
        const char* e = getenv("I8MM_DECODE_SMEM_KB");
        env_kb = (e && e[0]) ? atoi(e) : -1;
    }
    const size_t limit = env_kb > 0 ? static_cast<size_t>(env_kb) * 1024 : SMEM_LIMIT;
    const size_t fixed = 1024 + static_cast<size_t>(g.slots) * B_BYTES + smem_tail(nwords, kb_max);
    if (fixed + 2 * A_BYTES > limit) return g;
    int s2 = static_cast<int>((limit - fixed) / A_BYTES);
    if (s2 > MAX_STAGES) s2 = MAX_STAGES;
    const size_t xs_bytes = static_cast<size_t>(M * g.xs_ld) * 2;
    const int xs_stages = static_cast<int>((xs_bytes + A_BYTES - 1) / A_BYTES);
    // the X slice lives in the ring's last stages while T1/T2 run
    // keep the X slice in the ring whenever it fits, even if no stage is left for
    // the weight prefetch: re-reading X from global in T1/T2 costs more (fc2 M = 16:
    // 67.6 -> 57.4 us, profiles/r2/decode/notes_r2.md); I8MM_DECODE_XS_MIN_FREE for A/B
    static const int min_free = [] {
        const char* e = getenv("I8MM_DECODE_XS_MIN_FREE");
        return (e && e[0]) ? atoi(e) : 0;
    }();
    g.xs_cached = s2 - xs_stages >= min_free ? 1 : 0;
    g.s2 = s2;
    g.s1 = g.xs_cached ? s2 - xs_stages : s2;
    g.smem = fixed + static_cast<size_t>(s2) * A_BYTES;
    g.ok = true;
    return g;
}
}  // namespace

int decode_stages(int64_t M) { return decode_geom(M, 4096, 4096).s2; }

int decode_grid(int64_t K, int64_t N) { return decode_geom(1, K, N).grid; }

bool decode_fits(int64_t M, int64_t K, int64_t N) { return decode_geom(M, K, N).ok; }

__global__ void set_word_kernel(uint32_t* dst, uint32_t value) { *dst = value; }

cudaError_t launch_set_word(uint32_t* dst, uint32_t value, cudaStream_t st) {
    set_word_kernel<<<1, 1, 0, st>>>(dst, value);
    count_launch();
    return cudaGetLastError();
}

static unsigned long long* g_dbg = nullptr;
void set_decode_timeline(unsigned long long* stamps) { g_dbg = stamps; }
unsigned long long* debug_timeline() { return g_dbg; }

static int env_int_once(const char* name, int dflt) {
    const char* e = getenv(name);
    return (e && e[0]) ? atoi(e) : dflt;
}

template <int EPI>
static cudaError_t launch_decode_epi(const CUtensorMap& tw, const dec::Params& prm, const DecodeGeom& g,
                                     cudaStream_t st) {
    static std::once_flag once;
    static cudaError_t attr_err = cudaSuccess;
    std::call_once(once, [] {
        attr_err = cudaFuncSetAttribute(dec::decode_kernel<EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        dec::SMEM_LIMIT);
    });
    if (attr_err != cudaSuccess) return attr_err;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(g.grid));
    cfg.blockDim = dim3(dec::THREADS);
    cfg.dynamicSmemBytes = g.smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = dec::CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, dec::decode_kernel<EPI>, tw, prm);
    count_launch();
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

cudaError_t launch_decode(const DecodeArgs& a, int epi, cudaStream_t st) {
    using namespace dec;
    const DecodeGeom g = decode_geom(a.M, a.K, a.N);
    if (!g.ok) return cudaErrorInvalidValue;
    Params prm{};
    prm.a = a;
    prm.num_kb = static_cast<int>((a.K + BK - 1) / BK);
    prm.n_tiles = static_cast<int>((a.N + TILE_N - 1) / TILE_N);
    prm.total_units = g.units;
    prm.s1 = g.s1;
    prm.s2 = g.s2;
    // weight tiles prefetched before the token phase (env I8MM_DECODE_PREFETCH, A/B)
    static const int env_pre = env_int_once("I8MM_DECODE_PREFETCH", -1);
    prm.pre = env_pre >= 0 && env_pre < g.s1 ? env_pre : g.s1;
    static const int env_l2 = env_int_once("I8MM_DECODE_L2_PREFETCH", 0);
    prm.l2_prefetch = env_l2;
    static const int env_wp = env_int_once("I8MM_DECODE_W_POLICY", 0);
    prm.w_policy = env_wp;
    prm.slots = g.slots;
    prm.xs_cached = g.xs_cached;
    prm.xs_ld = g.xs_ld;
    prm.dbg = g_dbg;
    static const int env_dbg = env_int_once("I8MM_DECODE_DBG_MODE", 0);
    prm.dbg_mode = env_dbg;
    CUtensorMap tw;
    if (!make_tmap_i8_rows(&tw, a.wq_t, a.N, a.K, a.ldq, TILE_N)) return cudaErrorInvalidValue;
    switch (epi) {
        case EPI_F16: return launch_decode_epi<EPI_F16>(tw, prm, g, st);
        case EPI_F32: return launch_decode_epi<EPI_F32>(tw, prm, g, st);
        case EPI_F32_EXACT: return launch_decode_epi<EPI_F32_EXACT>(tw, prm, g, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace i8mm
