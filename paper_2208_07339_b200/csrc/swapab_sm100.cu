// Mid-size token counts (17..128 rows) of the weight-stationary prefill path:
// after the row prologue (O, row scales, Xq, x[:, O], W[O, :], patched columns;
// prologue.cu), the int8 product runs swap-AB so the tensor core's 128-row
// operand is the weights, not a mostly empty token tile:
//
//   D[n, m] = sum_k WqT[n, k] * Xq[m, k]    tcgen05.mma kind::i8, M = 128 weight
//                                            rows, N = MP >= M tokens, K = 32
//
// A 128-row token tile at M = 32 spent 3/4 of every MMA on zero rows and left
// all but n_tiles SMs idle (qkvo M = 32: 40 CTAs, 27 us for 26 MB). Here the
// (n-tile, k-block) units are split evenly over one CTA per SM (stream-K, as in
// decode_sm100.cu), each stage carries the weight tile and the k-block's MP
// token rows by TMA, and a tile split between CTAs is finished by the CTA
// holding its first k-block, which adds the others' int32 partials handed over
// through the workspace (per-tile arrival counters zeroed by the prologue).
// Patched columns (weight-stationary fixup, gemm.py:243 semantics) run as extra
// tiles over their re-derived codes; the main tiles skip them.
//
// The epilogue is the prefill kernel's fast one, element for element:
//   y = (f32(c) * rowf) * colf, then fma(xo[m, o], wo[o, n], y) for o ascending
// (gemm_sm100.cu emit), so outputs are bitwise those of the prefill GEMM.
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

namespace sab {

constexpr int THREADS = 256;  // warp 0 TMA, 1 MMA, 2 TMEM, 4-7 epilogue
constexpr int TILE_N = 128;   // weight rows per tile (the MMA's M)
constexpr int BK = 128;       // K bytes per stage
constexpr int UMMA_K = 32;
constexpr int KS = BK / UMMA_K;
constexpr int A_BYTES = TILE_N * BK;
constexpr int WO_CAP = 16;  // outlier rows of W held in registers
constexpr int MAX_STAGES = 16;
constexpr int SMEM_LIMIT = 227 * 1024;

struct Params {
    const float* row_amax;
    const float* col_amax;
    const __half* xo;
    int64_t o_cap;
    const int32_t* o_idx;
    const int32_t* o_count;
    const __half* x;
    int64_t ldx;
    const __half* w;
    int64_t ldw;
    const __half* wo;
    int64_t ldwo, wo_cap;
    const int32_t* patch_count;
    const int32_t* patch_idx;
    const float* patch_amax;
    const uint32_t* patch_mask;
    void* y;
    int64_t ldy;
    int64_t M, N;
    int num_kb, n_tiles, stages;
    int32_t* c32;       // [grid][MP][TILE_N] partial sums of split tiles
    int32_t* tile_cnt;  // [n_tiles + patch tiles] arrival counters (zeroed)
    unsigned long long* dbg;  // dev build: 16 %globaltimer stamps per CTA, nullable
};

#ifdef I8MM_GEMM_DEVTOOLS
constexpr bool kStamps = true;
#else
constexpr bool kStamps = false;
#endif
__device__ __forceinline__ void stamp(const Params& p, int i) {
    if constexpr (kStamps) {
        if (p.dbg != nullptr) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            p.dbg[blockIdx.x * 16 + i] = t;
        }
    }
}

struct __align__(8) Bars {
    uint64_t full[MAX_STAGES];
    uint64_t empty[MAX_STAGES];
    uint64_t tmem_full[2];
    uint64_t tmem_empty[2];
    uint32_t tmem_slot;
};

__device__ __forceinline__ float amax_or_127(float a) { return a == 0.0f ? 127.0f : a; }
__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

template <int MP>
constexpr int n_acc() { return 256 / MP; }  // 2 buffers x n_acc x MP = 512 TMEM columns
template <int MP>
constexpr int b_bytes() { return MP * BK; }
template <int MP>
constexpr int stage_bytes() { return A_BYTES + b_bytes<MP>(); }

template <int MP, int EPI>
__global__ void __launch_bounds__(THREADS, 1)
    swapab_kernel(const __grid_constant__ CUtensorMap tmap_w, const __grid_constant__ CUtensorMap tmap_p,
                  const __grid_constant__ CUtensorMap tmap_x, const Params p) {
    constexpr int NACC = n_acc<MP>();
    constexpr int STAGE = stage_bytes<MP>();
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u);
    const int S = p.stages;
    uint8_t* ring = smem;  // stage s: A (weights) then B (tokens)
    float* sxo = reinterpret_cast<float*>(ring + static_cast<size_t>(S) * STAGE);  // [MP][WO_CAP]
    float* srow = sxo + MP * WO_CAP;                                                 // [MP]
    float* swo = srow + MP;  // [WO_CAP][TILE_N] W[O, tile] of the current segment
    Bars* bars = reinterpret_cast<Bars*>(swo + WO_CAP * TILE_N);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int num_kb = p.num_kb;

    if (tid == 0) {
        tma_prefetch_desc(&tmap_w);
        tma_prefetch_desc(&tmap_p);
        tma_prefetch_desc(&tmap_x);
        for (int s = 0; s < S; ++s) {
            mbar_init(&bars->full[s], 1);
            mbar_init(&bars->empty[s], 1);
        }
        for (int q = 0; q < 2; ++q) {
            mbar_init(&bars->tmem_full[q], 1);
            mbar_init(&bars->tmem_empty[q], 4);
        }
        fence_mbarrier_init();
    }
    if (warp == 2) tmem_alloc<512>(&bars->tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = bars->tmem_slot;
    if (tid == 0) stamp(p, 0);
    // everything below reads the prologue's outputs
    pdl_wait();
    pdl_trigger();
    if (tid == 0) stamp(p, 1);
    const int n_patch = min(static_cast<int>(*p.patch_count), static_cast<int>(p.N));
    const int n_pt = (n_patch + TILE_N - 1) / TILE_N;
    const uint32_t T = static_cast<uint32_t>((p.n_tiles + n_pt) * num_kb);
    const uint32_t G = gridDim.x;
    const int u_begin = static_cast<int>(T * blockIdx.x / G);
    const int u_end = static_cast<int>(T * (blockIdx.x + 1) / G);

    if (warp == 0) {
        // ---------------- TMA producer: weight tile (main or patch) + the k-block's token rows
        if (lane == 0) {
            const uint64_t pol_w = l2_policy_evict_first();  // single-use weight stream
            const uint64_t pol_x = l2_policy_evict_last();   // Xq is re-read by every n-tile
            int tile = u_begin / num_kb, kb = u_begin - tile * num_kb;
            int s = 0;
            uint32_t ph = 0;
            for (int i = 0; i < u_end - u_begin; ++i) {
                if (i >= S) mbar_wait(&bars->empty[s], ph ^ 1u);
                uint8_t* st = ring + static_cast<size_t>(s) * STAGE;
                mbar_arrive_expect_tx(&bars->full[s], STAGE);
                if (tile < p.n_tiles)
                    tma_load_2d(&tmap_w, &bars->full[s], st, kb * BK, tile * TILE_N, pol_w);
                else
                    tma_load_2d(&tmap_p, &bars->full[s], st, kb * BK, (tile - p.n_tiles) * TILE_N, pol_w);
                tma_load_2d(&tmap_x, &bars->full[s], st + A_BYTES, kb * BK, 0, pol_x);
                if (++kb == num_kb) {
                    kb = 0;
                    ++tile;
                }
                if (++s == S) {
                    s = 0;
                    ph ^= 1u;
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer: 4 K-steps per unit, rotating over NACC accumulators
        const uint32_t idesc = idesc_i8(TILE_N, MP);
        const uint64_t base = smem_desc_k_sw128(smem_addr(ring));
        int s = 0;
        uint32_t ph = 0;
        int seg = 0;
        for (int u = u_begin; u < u_end; ++seg) {
            const int seg_end = min(u_end, (u / num_kb + 1) * num_kb);
            const int acc = seg & 1;
            mbar_wait(&bars->tmem_empty[acc], ((seg >> 1) & 1) ^ 1u);
            tc_fence_after();
            const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * NACC * MP);
            for (int kk = 0; u < seg_end; ++u, ++kk) {
                mbar_wait(&bars->full[s], ph);
                tc_fence_after();
                if (lane == 0) {
                    const uint64_t ad = base + static_cast<uint64_t>((s * STAGE) >> 4);
                    const uint64_t bd = ad + static_cast<uint64_t>(A_BYTES >> 4);
#pragma unroll
                    for (int k = 0; k < KS; ++k) {
                        const int j = kk * KS + k;
                        mma_i8(d_tmem + static_cast<uint32_t>((j & (NACC - 1)) * MP), ad + 2 * k, bd + 2 * k, idesc,
                               j >= NACC ? 1u : 0u);
                    }
                    mma_commit(&bars->empty[s]);
                }
                __syncwarp();
                if (++s == S) {
                    s = 0;
                    ph ^= 1u;
                }
            }
            if (lane == 0) mma_commit(&bars->tmem_full[acc]);
            __syncwarp();
            if (lane == 0 && seg < 3) stamp(p, 2 + seg);  // MMAs of segment issued
        }
    } else if (warp >= 4) {
        // ---------------- epilogue: thread = weight row n of the tile
        const int et = tid - 128;
        const int quad = warp & 3;
        const int n_out = *p.o_count;
        const int n_o = min(n_out, WO_CAP);
        for (int i = et; i < MP * WO_CAP; i += 128) {
            const int m = i / WO_CAP, o = i - m * WO_CAP;
            float v = 0.0f;
            if (m < p.M && o < n_o)
                v = o < p.o_cap ? __half2float(p.xo[m * p.o_cap + o]) : __half2float(p.x[m * p.ldx + p.o_idx[o]]);
            sxo[i] = v;
        }
        for (int m = et; m < MP; m += 128) srow[m] = m < p.M ? amax_or_127(p.row_amax[m]) : 127.0f;
        named_bar_sync(1, 128);
        int seg = 0;
        for (int u = u_begin; u < u_end; ++seg) {
            const int tile = u / num_kb;
            const int su0 = u;
            const int seg_end = min(u_end, (tile + 1) * num_kb);
            const bool full = su0 == tile * num_kb && seg_end == (tile + 1) * num_kb;
            u = seg_end;
            const int acc = seg & 1;
            // this thread's output column
            const bool patch = tile >= p.n_tiles;
            int64_t n;
            bool n_ok;
            float aw;
            if (!patch) {
                n = static_cast<int64_t>(tile) * TILE_N + et;
                n_ok = n < p.N && !((p.patch_mask[n >> 5] >> (n & 31)) & 1u);  // patched: its patch tile
                aw = n < p.N ? p.col_amax[n] : 127.0f;
            } else {
                const int pi = (tile - p.n_tiles) * TILE_N + et;
                n_ok = pi < n_patch;
                n = n_ok ? p.patch_idx[pi] : 0;
                aw = n_ok ? p.patch_amax[pi] : 127.0f;
            }
            const float colf = amax_or_127(aw) * (1.0f / 16129.0f);
            // split tile: first-unit holder finishes, the others hand over partials
            const uint32_t t0 = static_cast<uint32_t>(tile * num_kb), t1 = t0 + num_kb;
            const uint32_t cf = ((t0 + 1) * G - 1) / T;
            const uint32_t cl = (t1 * G - 1) / T;
            const bool finisher = !full && cf == blockIdx.x;
            float wr[WO_CAP];
            const int64_t n0 = static_cast<int64_t>(tile) * TILE_N;
            if (!full && !finisher) {  // contributor: raw partials only, no outlier term
#pragma unroll
                for (int o = 0; o < WO_CAP; ++o) wr[o] = 0.0f;
            } else if (!patch && n_o > 0 && n_o <= p.wo_cap && n0 + TILE_N <= p.N && (p.ldwo % 8) == 0) {
                // W[O, tile] staged with 16-byte loads (two per thread), then read from
                // shared memory: one load round trip instead of one per outlier row
                named_bar_sync(1, 128);  // the previous segment's readers are done
                for (int i = et; i < n_o * (TILE_N / 8); i += 128) {
                    const int o = i / (TILE_N / 8), c8 = i - o * (TILE_N / 8);
                    const uint4 q = *reinterpret_cast<const uint4*>(p.wo + static_cast<int64_t>(o) * p.ldwo + n0 + c8 * 8);
                    const __half2* h2 = reinterpret_cast<const __half2*>(&q);
                    float4* dst = reinterpret_cast<float4*>(swo + o * TILE_N + c8 * 8);
                    const float2 f0 = __half22float2(h2[0]), f1 = __half22float2(h2[1]);
                    const float2 f2 = __half22float2(h2[2]), f3 = __half22float2(h2[3]);
                    dst[0] = make_float4(f0.x, f0.y, f1.x, f1.y);
                    dst[1] = make_float4(f2.x, f2.y, f3.x, f3.y);
                }
                named_bar_sync(1, 128);
#pragma unroll
                for (int o = 0; o < WO_CAP; ++o) wr[o] = (o < n_o && n_ok) ? swo[o * TILE_N + et] : 0.0f;
            } else {
#pragma unroll
                for (int o = 0; o < WO_CAP; ++o)
                    wr[o] = (o < n_o && n_ok) ? (o < p.wo_cap ? __half2float(p.wo[static_cast<int64_t>(o) * p.ldwo + n])
                                                              : __half2float(p.w[static_cast<int64_t>(p.o_idx[o]) * p.ldw + n]))
                                              : 0.0f;
            }
            if (et == 0 && seg < 3) stamp(p, 5 + seg);  // epilogue reaches the segment
            if (finisher) {
                if (et == 0) {
                    for (uint32_t spin = 0; ld_acquire(p.tile_cnt + tile) < static_cast<int>(cl - cf); ++spin)
                        if (spin > (1u << 22)) __trap();
                    p.tile_cnt[tile] = 0;  // ready for the next call's prologue-free reuse
                }
                named_bar_sync(1, 128);
            }
            if (et == 0 && seg < 3) stamp(p, 8 + seg);  // finisher's partials ready (or no wait)
            mbar_wait(&bars->tmem_full[acc], (seg >> 1) & 1);
            tc_fence_after();
            if (et == 0 && seg < 3) stamp(p, 11 + seg);  // accumulator ready
            const uint32_t t_row = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) +
                                   static_cast<uint32_t>(acc * NACC * MP);
            const int n_used = min(NACC, (seg_end - su0) * KS);
#pragma unroll 1
            for (int c0 = 0; c0 < MP; c0 += 16) {
                if (c0 >= p.M) break;
                uint32_t r[16];
                tmem_ld_32x32b_x16(t_row + static_cast<uint32_t>(c0), r);
                tmem_ld_wait();
                for (int j = 1; j < n_used; ++j) {
                    uint32_t t[16];
                    tmem_ld_32x32b_x16(t_row + static_cast<uint32_t>(j * MP + c0), t);
                    tmem_ld_wait();
#pragma unroll
                    for (int e = 0; e < 16; ++e) r[e] += t[e];
                }
                if (!full && !finisher) {  // contributor: partials to this CTA's slot
                    int32_t* slot = p.c32 + (static_cast<int64_t>(blockIdx.x) * MP + c0) * TILE_N + et;
#pragma unroll
                    for (int e = 0; e < 16; ++e) __stcg(slot + e * TILE_N, static_cast<int32_t>(r[e]));
                    continue;
                }
                if (finisher) {
                    for (uint32_t c = cf + 1; c <= cl; ++c) {
                        const int32_t* src = p.c32 + (static_cast<int64_t>(c) * MP + c0) * TILE_N + et;
#pragma unroll
                        for (int e = 0; e < 16; ++e) r[e] += static_cast<uint32_t>(__ldcg(src + e * TILE_N));
                    }
                }
                if (n_ok) {
#pragma unroll
                    for (int e = 0; e < 16; ++e) {
                        const int m = c0 + e;
                        if (m >= p.M) break;
                        float v = (static_cast<float>(static_cast<int32_t>(r[e])) * srow[m]) * colf;
                        if (n_out <= WO_CAP) {
#pragma unroll
                            for (int o = 0; o < WO_CAP; ++o)
                                if (o < n_out) v = fmaf(sxo[m * WO_CAP + o], wr[o], v);
                        } else {
                            for (int o = 0; o < n_out; ++o) {
                                const float xv = o < p.o_cap ? __half2float(p.xo[m * p.o_cap + o])
                                                             : __half2float(p.x[m * p.ldx + p.o_idx[o]]);
                                const float wv = o < p.wo_cap ? __half2float(p.wo[static_cast<int64_t>(o) * p.ldwo + n])
                                                              : __half2float(p.w[static_cast<int64_t>(p.o_idx[o]) * p.ldw + n]);
                                v = fmaf(xv, wv, v);
                            }
                        }
                        if constexpr (EPI == EPI_F16)
                            reinterpret_cast<__half*>(p.y)[m * p.ldy + n] = __float2half_rn(v);
                        else
                            reinterpret_cast<float*>(p.y)[m * p.ldy + n] = v;
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bars->tmem_empty[acc]);
            if (!full && !finisher) {
                // the barrier orders every thread's partial stores before thread 0's release
                named_bar_sync(1, 128);
                if (et == 0) asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(p.tile_cnt + tile) : "memory");
            }
        }
    }
    if (tid == 128) stamp(p, 15);  // epilogue done (before the closing barrier; timer reads
                                   // right after a BAR.SYNC can complete before it resolves)
    tc_fence_before();
    __syncthreads();
    if (tid == 0) stamp(p, 14);
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc<512>(tmem_base);
    }
}

}  // namespace sab

namespace {
int sab_stages(int mp) {
    const size_t stage = static_cast<size_t>(sab::A_BYTES) + static_cast<size_t>(mp) * sab::BK;
    const size_t fixed = 1024 + static_cast<size_t>(mp) * (sab::WO_CAP + 1) * sizeof(float) +
                         static_cast<size_t>(sab::WO_CAP) * sab::TILE_N * sizeof(float) + sizeof(sab::Bars) + 64;
    int s = static_cast<int>((sab::SMEM_LIMIT - fixed) / stage);
    return s > sab::MAX_STAGES ? sab::MAX_STAGES : s;
}
int g_swapab = -1;  // -1: env I8MM_SWAPAB (default on)
unsigned long long* g_sab_dbg = nullptr;
}  // namespace

int swapab_mp(int64_t M) { return M <= 32 ? 32 : (M <= 64 ? 64 : 128); }

// Routing (measured, profiles/r2/decode/notes_r2.md, single calls on the OPT-13B
// projections): swap-AB wins at M <= 32 for every shape and at M <= 64 while the
// row-tile GEMM would have fewer 256-column tiles than half the SMs; above that
// the row-tile GEMM's overlapped epilogue wins. M <= 16 stays on the decode kernel.
bool swapab_route(int64_t M, int64_t K, int64_t N) {
    static const int min_m = [] {  // A/B overrides, read once (independently of set_swapab)
        const char* lo = getenv("I8MM_SWAPAB_MIN_M");
        return (lo && lo[0]) ? atoi(lo) : 0;
    }();
    static const int max_m = [] {
        const char* hi = getenv("I8MM_SWAPAB_MAX_M");
        return (hi && hi[0]) ? atoi(hi) : 64;
    }();
    if (g_swapab < 0) {
        const char* e = getenv("I8MM_SWAPAB");
        g_swapab = (e && e[0] == '0') ? 0 : 1;
    }
    // below 17 rows only small weight matrices (<= 32 MiB of codes), from 12 rows:
    // measured against the decode kernel (qkvo 5120 x 5120: M = 12 / 16: 37.9 / 41.8 ->
    // 36.9 us; fc1 / fc2 (105 MB) stay faster on the decode kernel up to M = 16)
    const int64_t lo_m = min_m > 0 ? min_m : (K * N <= (32LL << 20) ? 12 : 17);
    if (g_swapab != 1 || M < lo_m || M > max_m || M > 128 || K < sab::BK || N < 1 || (K % 16) != 0) return false;
    if (M <= 32 || max_m > 64) return true;
    return (N + 255) / 256 < num_sms() / 2;
}

void set_swapab(int on) { g_swapab = on; }

void set_swapab_timeline(unsigned long long* stamps) { g_sab_dbg = stamps; }

int64_t swapab_c32_words(int64_t M) { return static_cast<int64_t>(num_sms()) * swapab_mp(M) * sab::TILE_N; }

int64_t swapab_cnt_words(int64_t N) { return 2 * ((N + sab::TILE_N - 1) / sab::TILE_N); }

template <int MP, int EPI>
static cudaError_t launch_sab(const CUtensorMap& tw, const CUtensorMap& tp, const CUtensorMap& tx,
                              const sab::Params& prm, int grid, size_t smem, cudaStream_t st) {
    static std::once_flag once;
    static cudaError_t attr_err = cudaSuccess;
    std::call_once(once, [] {
        attr_err = cudaFuncSetAttribute(sab::swapab_kernel<MP, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        sab::SMEM_LIMIT);
    });
    if (attr_err != cudaSuccess) return attr_err;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(grid));
    cfg.blockDim = dim3(sab::THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    cudaError_t e = cudaLaunchKernelEx(&cfg, sab::swapab_kernel<MP, EPI>, tw, tp, tx, prm);
    count_launch();
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

cudaError_t launch_swapab(const GemmArgs& a, int32_t* c32, int32_t* tile_cnt, int epi, cudaStream_t st) {
    if (a.M < 1 || a.M > 128 || a.N <= 0 || a.K <= 0 || (epi != EPI_F16 && epi != EPI_F32)) return cudaErrorInvalidValue;
    const int mp = swapab_mp(a.M);
    sab::Params prm{};
    prm.row_amax = a.row_amax;
    prm.col_amax = a.col_amax;
    prm.xo = a.xo;
    prm.o_cap = a.o_cap;
    prm.o_idx = a.o_idx;
    prm.o_count = a.o_count;
    prm.x = a.x;
    prm.ldx = a.ldx;
    prm.w = a.w;
    prm.ldw = a.ldw;
    prm.wo = a.wo;
    prm.ldwo = a.ldwo;
    prm.wo_cap = a.wo_cap;
    prm.patch_count = a.patch_count;
    prm.patch_idx = a.patch_idx;
    prm.patch_amax = a.patch_amax;
    prm.patch_mask = a.patch_mask;
    prm.y = a.y;
    prm.ldy = a.ldy;
    prm.M = a.M;
    prm.N = a.N;
    prm.num_kb = static_cast<int>((a.K + sab::BK - 1) / sab::BK);
    prm.n_tiles = static_cast<int>((a.N + sab::TILE_N - 1) / sab::TILE_N);
    prm.stages = sab_stages(mp);
    prm.c32 = c32;
    prm.tile_cnt = tile_cnt;
    prm.dbg = g_sab_dbg;
    CUtensorMap tw, tp, tx;
    if (!make_tmap_i8_rows(&tw, a.b, a.N, a.K, a.ldb, sab::TILE_N)) return cudaErrorInvalidValue;
    if (!make_tmap_i8_rows(&tp, a.b_patch, a.N, a.K, a.ldb, sab::TILE_N)) return cudaErrorInvalidValue;
    if (!make_tmap_i8_rows(&tx, a.a, a.M, a.K, a.lda, mp)) return cudaErrorInvalidValue;
    // one CTA per SM; every CTA gets at least one unit of the main tiles
    const int64_t units = static_cast<int64_t>(prm.n_tiles) * prm.num_kb;
    const int grid = static_cast<int>(units < num_sms() ? units : num_sms());
    const size_t smem = 1024 + static_cast<size_t>(prm.stages) * (sab::A_BYTES + mp * sab::BK) +
                        static_cast<size_t>(mp) * (sab::WO_CAP + 1) * sizeof(float) +
                        static_cast<size_t>(sab::WO_CAP) * sab::TILE_N * sizeof(float) + sizeof(sab::Bars) + 64;
    switch (mp * 4 + epi) {
        case 32 * 4 + EPI_F16: return launch_sab<32, EPI_F16>(tw, tp, tx, prm, grid, smem, st);
        case 64 * 4 + EPI_F16: return launch_sab<64, EPI_F16>(tw, tp, tx, prm, grid, smem, st);
        case 128 * 4 + EPI_F16: return launch_sab<128, EPI_F16>(tw, tp, tx, prm, grid, smem, st);
        case 32 * 4 + EPI_F32: return launch_sab<32, EPI_F32>(tw, tp, tx, prm, grid, smem, st);
        case 64 * 4 + EPI_F32: return launch_sab<64, EPI_F32>(tw, tp, tx, prm, grid, smem, st);
        case 128 * 4 + EPI_F32: return launch_sab<128, EPI_F32>(tw, tp, tx, prm, grid, smem, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace i8mm
