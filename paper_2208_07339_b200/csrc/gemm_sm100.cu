// K4: int8 x int8 -> int32 GEMM on the 5th-gen tensor cores (tcgen05, sm_100a)
// with the LLM.int8() epilogue fused in: vector-wise dequantization by the
// outer product of row/column absmax (gemm.py:120-147, row x col branch) plus
// the high-precision outlier term sum_{o in O} X[:,o] W[o,:] (gemm.py:238,
// 244-247), written straight to the output tile.
//
// Structure (persistent, warp-specialised, 384 threads per CTA). CG=2 (the
// default for M > 128) runs CTA pairs (cluster 2x1) on cta_group::2 MMAs:
// a 256x256 output tile per pair, each CTA loading 128 rows of Xq and 128 rows
// of WqT per stage, which halves the per-SM shared-memory operand traffic of
// the 1-CTA (CG=1) 128x256 tile.
//   warp 0      TMA producer   : Xq / WqT K-blocks of 128 B into a SWIZZLE_128B
//                                smem ring (4 stages CG=1, 6 stages CG=2); in a
//                                pair both CTAs load, the leader's mbarrier
//                                counts both CTAs' bytes
//   warp 1      MMA issuer     : one elected lane of the leader CTA issues
//                                tcgen05.mma.cta_group::{1,2}.kind::i8
//                                (M = 128 CG, N = 256, K = 32) into TMEM
//   warp 2      TMEM allocator : 512 columns = two 128x256 int32 accumulators
//   warps 4..11 epilogue       : tcgen05.ld -> dequant + outlier FMAs ->
//                                global stores, overlapping the next tile's
//                                mainloop (double-buffered TMEM)
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <mutex>

#include "kernels.cuh"
#include "sm100_ptx.cuh"

namespace i8mm {

namespace gemm {
constexpr int BM = 128;  // rows of the output tile per CTA
constexpr int BN = 256;  // columns of the output tile (per CTA pair when CG=2)
constexpr int BK = 128;  // bytes == int8 elements: one SWIZZLE_128B atom row
constexpr int UMMA_K = 32;
constexpr int MAX_STAGES = 6;
constexpr int A_BYTES = BM * BK;

// CG = CTAs per MMA (cta_group), MC = CTA pairs per cluster sharing each WqT
// tile through TMA multicast (cluster = CG * MC CTAs along M).
// TS: fp16 output through per-warp shared-memory staging tiles and TMA bulk
// stores (full 64-byte row segments per box row instead of 32 scattered
// 16-byte stores per warp instruction); costs one operand stage of smem.
// NW: N=256 MMA halves per tile (2: the pair tile is 256 x 512 with one 512-column
// accumulator -- each A panel feeds twice the outputs, 0.75x the L2 -> SM bytes)
template <int CG, int MC = 1, bool TS = false, int NW = 1>
struct Cfg {
    static constexpr int TBN = BN * NW;           // output columns per (pair) tile
    static constexpr int STAGES = NW == 2 ? (TS ? 3 : 4) : (CG == 1 ? 4 : (TS ? 5 : 6));
    static constexpr int B_ROWS = TBN / CG;       // WqT rows resident in each CTA
    static constexpr int B_LOAD_ROWS = B_ROWS / MC;  // rows each CTA fetches (then multicasts)
    static constexpr int B_BYTES = B_ROWS * BK;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr size_t SMEM_OPERANDS = static_cast<size_t>(STAGES) * STAGE_BYTES;
    static constexpr int GROUP_M = CG == 1 ? 16 : 8 / MC;
    static constexpr int CLUSTER = CG * MC;
    static constexpr int TILE_M = BM * CG * MC;    // output rows per cluster tile
};
constexpr int WO_CAP = 16;  // outlier rows of W staged in smem per tile
constexpr int EPI_WARP0 = 4;
constexpr int EPI_WARPS = 8;  // two warps per TMEM lane quadrant, each half of BN
constexpr int EPI_THREADS = EPI_WARPS * 32;
constexpr int THREADS = (EPI_WARP0 + EPI_WARPS) * 32;
constexpr uint32_t TMEM_COLS = 2 * BN;

struct __align__(8) Barriers {
    uint64_t full[MAX_STAGES];
    uint64_t empty[MAX_STAGES];
    uint64_t tmem_full[2];
    uint64_t tmem_empty[2];
    uint32_t tmem_slot;
};

// outlier rows of W staged per tile (the 512-wide tile stages up to 8; more take
// the global-load path) and the per-column factors
__host__ __device__ constexpr int wo_cap_of(int nw) { return nw == 2 ? 8 : WO_CAP; }
__host__ __device__ constexpr size_t smem_wo_of(int nw) {
    return static_cast<size_t>(wo_cap_of(nw)) * BN * nw * sizeof(float);
}
__host__ __device__ constexpr size_t smem_cols_of(int nw) { return static_cast<size_t>(BN) * nw * sizeof(double); }
constexpr int STG_BYTES = 32 * 32 * 2;  // one 32 x 32 fp16 staging tile
constexpr size_t SMEM_STG = static_cast<size_t>(EPI_WARPS) * 2 * STG_BYTES;  // double-buffered per warp
template <int CG, int MC, bool TS = false, int NW = 1>
constexpr size_t smem_total() {
    return 1024 /*align slack*/ + Cfg<CG, MC, TS, NW>::SMEM_OPERANDS + (TS ? SMEM_STG : 0) + smem_wo_of(NW) +
           smem_cols_of(NW) + sizeof(Barriers) + 64;
}

struct Params {
    int64_t M, N, K;
    int num_kb;
    int m_tiles;
    void* y;
    int64_t ldy;
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
    const __half* wo;
    int64_t ldwo;
    int64_t wo_cap;
    // weight-stationary patches: extra N-tiles appended after the main tiles,
    // B from the patch codes (tmap_p), output column j -> Y column patch_idx[j],
    // column amax patch_amax[j], live count *patch_count (read on the device)
    const int32_t* patch_count;
    const int32_t* patch_idx;
    const float* patch_amax;
    const uint32_t* patch_mask;  // bit j: Y column j is written by a patch tile instead
    int vec_store;  // 1: y rows 16-byte aligned and row pitch a multiple of 16 B
    int dbg_epi;    // A/B knob (I8MM_DBG_EPI): bit 0 skips the outlier FMAs, bit 1 the stores
    int tma_y;      // tmap_y is valid (fp16 Y, 16-byte aligned rows)
    int group_m;    // raster: m-tiles per group sharing each B panel in L2
    int l2_pol;     // raster L2 policy (A/B): bit 0 A panels evict_last, bit 1 B panels evict_first
    // split-K (CG = 1 only): ksplit units per tile, each over a K-block range;
    // partials are added into c32 (column-major, c32_rows rows: one red per
    // lane covers 32 consecutive rows), the last unit of a tile runs the epilogue
    int ksplit;
    int32_t* c32;
    int64_t c32_rows;
    int32_t* c32_cnt;
    unsigned long long* dbg;  // per-CTA %globaltimer stamps (dev tool), nullable
    // fused output all-gather (EPI_F16): every output row segment is also
    // stored to n_peer peer buffers (NVLink peer memory of the other ranks'
    // full Y, column offset peer_col); peer_vec: 16-byte aligned peer rows
    void* y_peer[kMaxPeers];
    int n_peer;
    int64_t peer_ldy, peer_col;
    int peer_vec;
};

// Dev instrumentation (timeline stamps, wait-cycle counters, the I8MM_DBG_EPI
// knob) is compiled only into the dev build (`build.py --devtools`, defines
// I8MM_GEMM_DEVTOOLS): even never taken, its branches in the producer / MMA /
// epilogue loops cost the production kernel 13-15 % (measured same-box A/B)
#ifdef I8MM_GEMM_DEVTOOLS
constexpr bool kDev = true;
#else
constexpr bool kDev = false;
#endif

__device__ __forceinline__ void gstamp(unsigned long long* dbg, int i) {
    if (kDev && dbg != nullptr) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        dbg[blockIdx.x * 16 + i] = t;
    }
}

struct TileSpace {
    int n_tiles, main_total, patch_n, total;
};

__device__ __forceinline__ TileSpace tile_space(const Params& p, int tbn) {
    TileSpace ts;
    ts.n_tiles = static_cast<int>((p.N + tbn - 1) / tbn);
    ts.main_total = p.m_tiles * ts.n_tiles;
    int64_t pn = 0;
    if (p.patch_count != nullptr) {
        pn = *p.patch_count;
        pn = pn < p.N ? pn : p.N;
    }
    ts.patch_n = static_cast<int>(pn);
    ts.total = ts.main_total + p.m_tiles * static_cast<int>((pn + tbn - 1) / tbn);
    return ts;
}

__device__ __forceinline__ bool tile_coords(const Params& p, const TileSpace& ts, int t,
                                            int& m_blk, int& n_blk) {
    const int GROUP_M = p.group_m;
    if (t >= ts.main_total) {  // patch tiles (weight-stationary fixup), m fastest
        const int local = t - ts.main_total;
        m_blk = local % p.m_tiles;
        n_blk = local / p.m_tiles;
        return true;
    }
    // grouped raster: GROUP_M m-tiles share each B panel while it is hot in L2
    const int per_group = GROUP_M * ts.n_tiles;
    const int g = t / per_group;
    const int first_m = g * GROUP_M;
    const int gm = min(GROUP_M, p.m_tiles - first_m);
    const int local = t - g * per_group;
    m_blk = first_m + local % gm;
    n_blk = local / gm;
    return false;
}

__device__ __forceinline__ float amax_or_127(float a) { return a == 0.0f ? 127.0f : a; }

// v[0..31] += sum_o xo[o] * wo[o][0..31] over NO staged (zero-padded) outlier
// rows: straight-line packed f32x2 FMAs, no per-row guards. The rows are staged
// widened to f32 once per tile: staging them as fp16 halves the shared-memory
// wavefronts but costs two conversions per pair in every chunk (+58 M warp
// instructions on fc1, +31 %, which a power-capped part pays in clock)
template <int NO, int TBN>
__device__ __forceinline__ void outlier_fma(float2* v2, const float* xo_r, const float* wrow) {
#pragma unroll
    for (int o = 0; o < NO; ++o) {
        const float2 xv2 = make_float2(xo_r[o], xo_r[o]);
        const float4* wr = reinterpret_cast<const float4*>(wrow + o * TBN);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const float4 f = wr[u];
            v2[2 * u] = __ffma2_rn(xv2, make_float2(f.x, f.y), v2[2 * u]);
            v2[2 * u + 1] = __ffma2_rn(xv2, make_float2(f.z, f.w), v2[2 * u + 1]);
        }
    }
}

template <int EPI, int CG, int MC, int NW>
__global__ void __launch_bounds__(THREADS, 1)
    gemm_i8_kernel(const __grid_constant__ CUtensorMap tmap_a,
                   const __grid_constant__ CUtensorMap tmap_b,
                   const __grid_constant__ CUtensorMap tmap_p,
                   const __grid_constant__ CUtensorMap tmap_y, const Params p) {
    constexpr bool TS = EPI == EPI_F16 && CG == 2;
    using C = Cfg<CG, MC, TS, NW>;
    constexpr int TBN = C::TBN;
    constexpr int WOC = wo_cap_of(NW);
    constexpr int COLS_PER_WARP = TBN / (EPI_WARPS / 4);
    constexpr size_t SMEM_WO = smem_wo_of(NW);
    constexpr size_t SMEM_COLS = smem_cols_of(NW);
    constexpr int STAGES = C::STAGES;
    constexpr int B_BYTES = C::B_BYTES;
    constexpr size_t SMEM_OPERANDS = C::SMEM_OPERANDS;
    constexpr size_t SMEM_STAGE_OUT = TS ? SMEM_STG : 0;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-byte alignment for SWIZZLE_128B, by offsetting within the shared
    // array (pointer arithmetic keeps the shared address space -> LDS, not LD)
    uint8_t* smem = smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u);
    uint8_t* smem_a = smem;
    uint8_t* smem_b = smem + static_cast<size_t>(STAGES) * A_BYTES;
    uint8_t* smem_stg = smem + SMEM_OPERANDS;  // TS: per-warp output staging tiles
    float* smem_wo = reinterpret_cast<float*>(smem + SMEM_OPERANDS + SMEM_STAGE_OUT);
    double* smem_col = reinterpret_cast<double*>(smem + SMEM_OPERANDS + SMEM_STAGE_OUT + SMEM_WO);
    Barriers* bars = reinterpret_cast<Barriers*>(smem + SMEM_OPERANDS + SMEM_STAGE_OUT + SMEM_WO + SMEM_COLS);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    if (threadIdx.x == 0) gstamp(p.dbg, 0);
    const uint32_t cl_rank = C::CLUSTER > 1 ? cluster_ctarank() : 0u;
    const uint32_t crank = cl_rank % CG;            // rank within the CTA pair
    const uint32_t pair = cl_rank / CG;             // which pair of the cluster
    const uint32_t leader_rank = pair * CG;         // cluster rank of this pair's MMA leader
    const bool leader = crank == 0;
    const int cluster_id = static_cast<int>(blockIdx.x) / C::CLUSTER;
    const int n_clusters = static_cast<int>(gridDim.x) / C::CLUSTER;

    if (threadIdx.x == 0) {
        tma_prefetch_desc(&tmap_a);
        tma_prefetch_desc(&tmap_b);
        if (p.patch_count != nullptr) tma_prefetch_desc(&tmap_p);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&bars->full[s], 1);
            mbar_init(&bars->empty[s], MC);  // freed by every pair's MMA (multicast B)
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&bars->tmem_full[a], 1);
            // one arrive per epilogue warp of every CTA of the pair
            mbar_init(&bars->tmem_empty[a], CG * EPI_WARPS);
        }
        fence_mbarrier_init();
    }
    if (warp == 2) {
        if constexpr (CG == 2) tmem_alloc_pair<TMEM_COLS>(&bars->tmem_slot);
        else tmem_alloc<TMEM_COLS>(&bars->tmem_slot);
    }
    tc_fence_before();
    __syncthreads();
    if constexpr (C::CLUSTER > 1) cluster_sync_all();  // peer barriers initialised + TMEM allocated
    tc_fence_after();
    const uint32_t tmem_base = bars->tmem_slot;
    pdl_wait();  // setup above overlaps the predecessor's tail (programmatic dependent launch)
    pdl_trigger();
    // the live tile count reads the patch counter written by the prologue:
    // only after the dependency wait
    const TileSpace ts = tile_space(p, TBN);
    if (threadIdx.x == 0) gstamp(p.dbg, 1);

    if (warp == 0) {
        // ===================== TMA producer =====================
        if (lane == 0) {
            const uint64_t pol = l2_policy_evict_normal();
            // the group's A panels stay in L2 while the B panels stream past them
            const uint64_t pol_a = (p.l2_pol & 1) ? l2_policy_evict_last() : pol;
            const uint64_t pol_b = (p.l2_pol & 2) ? l2_policy_evict_first() : pol;
            int stage = 0;
            uint32_t phase = 0;
            long long w_empty = 0;
            for (int u = cluster_id; u < ts.total * p.ksplit; u += n_clusters) {
                const int t = u / p.ksplit, sl = u % p.ksplit;
                const int kb0 = sl * p.num_kb / p.ksplit, kb1 = (sl + 1) * p.num_kb / p.ksplit;
                int m_blk, n_blk;
                const bool is_patch = tile_coords(p, ts, t, m_blk, n_blk);
                const CUtensorMap* map_b = is_patch ? &tmap_p : &tmap_b;
                const int a_row = m_blk * C::TILE_M + static_cast<int>(pair) * (BM * CG) +
                                  static_cast<int>(crank) * BM;
                // N-half h of the tile: rows n_blk*TBN + h*BN + crank*(BN/CG) (+ this pair's share)
                const int b_row = n_blk * TBN + static_cast<int>(crank) * (BN / CG) +
                                  static_cast<int>(pair) * (C::B_LOAD_ROWS / NW);
                // this CTA's B piece is multicast to the CTAs of equal crank in every pair
                uint16_t b_mask = 0;
#pragma unroll
                for (int q = 0; q < MC; ++q) b_mask |= static_cast<uint16_t>(1u << (q * CG + crank));
                if (u == cluster_id) gstamp(p.dbg, 2);
                for (int kb = kb0; kb < kb1; ++kb) {
                    if ((kDev && p.dbg != nullptr)) {
                        const long long c0 = clock64();
                        mbar_wait(&bars->empty[stage], phase ^ 1u);
                        w_empty += clock64() - c0;
                    }
                    mbar_wait(&bars->empty[stage], phase ^ 1u);
                    if constexpr (CG == 2) {
                        // the pair leader's full barrier counts every byte landing in the pair
                        if (leader) mbar_arrive_expect_tx(&bars->full[stage], CG * C::STAGE_BYTES);
                        tma_load_2d_pair(&tmap_a, &bars->full[stage], smem_a + stage * A_BYTES,
                                         kb * BK, a_row, pol_a);
                        uint8_t* bdst = smem_b + stage * B_BYTES + pair * (C::B_LOAD_ROWS * BK);
                        if constexpr (MC > 1)
                            tma_load_2d_pair_mc(map_b, &bars->full[stage], bdst, kb * BK, b_row,
                                                b_mask, pol_b);
                        else
#pragma unroll
                            for (int h = 0; h < NW; ++h)  // the tile's N-halves, 16 KB each
                                tma_load_2d_pair(map_b, &bars->full[stage], bdst + h * (BN / CG) * BK, kb * BK,
                                                 b_row + h * BN, pol_b);
                    } else {
                        mbar_arrive_expect_tx(&bars->full[stage], C::STAGE_BYTES);
                        tma_load_2d(&tmap_a, &bars->full[stage], smem_a + stage * A_BYTES, kb * BK,
                                    a_row, pol_a);
                        tma_load_2d(map_b, &bars->full[stage], smem_b + stage * B_BYTES, kb * BK,
                                    b_row, pol_b);
                    }
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
            }
            if ((kDev && p.dbg != nullptr)) p.dbg[blockIdx.x * 16 + 14] = static_cast<unsigned long long>(w_empty);
        }
    } else if (warp == 1 && leader) {
        // ===================== MMA issuer (leader CTA) =====================
        constexpr uint32_t idesc = idesc_i8(BM * CG, BN);
        const uint64_t a_desc0 = smem_desc_k_sw128(smem_addr(smem_a));
        const uint64_t b_desc0 = smem_desc_k_sw128(smem_addr(smem_b));
        int stage = 0;
        uint32_t phase = 0;
        int it = 0;
        long long w_full = 0, w_acc = 0;
        for (int u = cluster_id; u < ts.total * p.ksplit; u += n_clusters, ++it) {
            const int sl = u % p.ksplit;
            const int kb0 = sl * p.num_kb / p.ksplit, kb1 = (sl + 1) * p.num_kb / p.ksplit;
            // NW == 1: two 256-column accumulators alternate; NW == 2: one 512-column
            const int acc = NW == 1 ? (it & 1) : 0;
            const uint32_t acc_phase = NW == 1 ? ((it >> 1) & 1) : (it & 1);
            if ((kDev && p.dbg != nullptr)) {
                const long long c0 = clock64();
                mbar_wait(&bars->tmem_empty[acc], acc_phase ^ 1u);
                w_acc += clock64() - c0;
            }
            mbar_wait(&bars->tmem_empty[acc], acc_phase ^ 1u);
            tc_fence_after();
            const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * BN);
            for (int kb = kb0; kb < kb1; ++kb) {
                if ((kDev && p.dbg != nullptr)) {
                    const long long c0 = clock64();
                    mbar_wait(&bars->full[stage], phase);
                    w_full += clock64() - c0;
                }
                mbar_wait(&bars->full[stage], phase);
                tc_fence_after();
                if (lane == 0 && it == 0 && kb == kb0) gstamp(p.dbg, 3);
                if (lane == 0) {
                    // descriptors advance by +2 per 32-byte K step (the address field
                    // is in 16-byte units): no per-MMA descriptor arithmetic
                    const uint64_t a_d = a_desc0 + static_cast<uint64_t>(stage * (A_BYTES >> 4));
                    const uint64_t b_d = b_desc0 + static_cast<uint64_t>(stage * (B_BYTES >> 4));
#pragma unroll
                    for (int k = 0; k < BK / UMMA_K; ++k) {
                        const uint64_t ad = a_d + 2 * k;
                        const uint32_t accum = (kb != kb0 || k != 0) ? 1u : 0u;
#pragma unroll
                        for (int h = 0; h < NW; ++h) {  // N-half h: B rows h*BN/CG.., TMEM columns h*BN..
                            const uint64_t bd = b_d + static_cast<uint64_t>(h * ((BN / CG * BK) >> 4)) + 2 * k;
                            if constexpr (CG == 2) mma_i8_pair(d_tmem + h * BN, ad, bd, idesc, accum);
                            else mma_i8(d_tmem + h * BN, ad, bd, idesc, accum);
                        }
                    }
                    // frees the smem slot (in both CTAs of a pair) when the MMAs finish
                    // (with MC > 1 the slot also holds B pieces written by the other
                    // pairs' producers, so every CTA of the cluster is told)
                    if constexpr (CG == 2)
                        mma_commit_pair(&bars->empty[stage],
                                        static_cast<uint16_t>((1u << C::CLUSTER) - 1u));
                    else mma_commit(&bars->empty[stage]);
                }
                __syncwarp();
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1u;
                }
            }
            if (lane == 0 && it == 0) gstamp(p.dbg, 4);
            if (lane == 0) {  // accumulator ready (both CTAs' epilogues)
                if constexpr (CG == 2)
                    mma_commit_pair(&bars->tmem_full[acc], static_cast<uint16_t>(0x3u << leader_rank));
                else mma_commit(&bars->tmem_full[acc]);
            }
            __syncwarp();
        }
        if ((kDev && p.dbg != nullptr) && lane == 0) {
            p.dbg[blockIdx.x * 16 + 12] = static_cast<unsigned long long>(w_full);
            p.dbg[blockIdx.x * 16 + 13] = static_cast<unsigned long long>(w_acc);
        }
    } else if (warp >= EPI_WARP0) {
        // ===================== epilogue =====================
        const int quad = warp & 3;                       // TMEM lanes 32*quad .. +31
        const int half = (warp - EPI_WARP0) >> 2;        // which half of the BN columns
        const int et = threadIdx.x - EPI_WARP0 * 32;     // 0 .. EPI_THREADS-1
        int n_out = 0;
        if constexpr (EPI != EPI_I32) n_out = p.o_count ? *p.o_count : 0;
        const bool wo_fast = n_out <= WOC && p.wo != nullptr && n_out <= p.wo_cap;
        const bool xo_fast = n_out <= WOC && p.xo != nullptr && n_out <= p.o_cap;
        const bool stage_wo = n_out > 0 && n_out <= WOC;
        // staged outlier rows are padded with zeros to a class of 4 / 6 / 8 / 16 so the
        // FMA loop is straight-line code (per-outlier guards made the compiler
        // shuffle the 32 accumulators between registers at every join)
        const int n_cls = n_out <= 4 ? 4 : (n_out <= 6 ? 6 : (n_out <= 8 ? 8 : WOC));
        uint32_t stg_cnt = 0;  // TS: output boxes issued by this warp
        __shared__ int split_last;
        long long w_tf = 0;
        int it = 0;
        for (int u = cluster_id; u < ts.total * p.ksplit; u += n_clusters, ++it) {
            const int t = u / p.ksplit;
            int m_blk, n_blk;
            const bool is_patch = tile_coords(p, ts, t, m_blk, n_blk);
            const int acc = NW == 1 ? (it & 1) : 0;
            const uint32_t acc_phase = NW == 1 ? ((it >> 1) & 1) : (it & 1);
            const int64_t n_live = is_patch ? ts.patch_n : p.N;
            const float* camax = is_patch ? p.patch_amax : p.col_amax;
            const int32_t* cmap = p.patch_idx;
            const int64_t row = static_cast<int64_t>(m_blk) * C::TILE_M + pair * (BM * CG) +
                                crank * BM + quad * 32 + lane;
            const int64_t col0 = static_cast<int64_t>(n_blk) * TBN;
            const bool row_ok = row < p.M;
            const bool mapped = is_patch;

            float xo_r[WO_CAP];
            float rowf = 0.0f;
            double sx = 1.0;
            if constexpr (EPI != EPI_I32) {
                // ---- stage per-tile column factors and outlier W rows in smem
                named_bar_sync(1, EPI_THREADS);  // previous tile's readers are done
                for (int j = et; j < TBN; j += EPI_THREADS) {
                    const int64_t c = col0 + j;
                    const float aw = c < n_live ? amax_or_127(camax[c]) : 127.0f;
                    if constexpr (EPI == EPI_F32_EXACT)
                        smem_col[j] = 127.0 / static_cast<double>(aw);
                    else
                        reinterpret_cast<float*>(smem_col)[j] = aw * (1.0f / 16129.0f);
                }
                if (stage_wo) {
                    if (wo_fast && !mapped && col0 + TBN <= n_live && (p.ldwo % 8) == 0) {
                        // 16-byte vector loads of the compact outlier rows
                        for (int i = et; i < n_cls * (TBN / 8); i += EPI_THREADS) {
                            const int o = i / (TBN / 8), v = i % (TBN / 8);
                            const uint4 q = o < n_out ? *reinterpret_cast<const uint4*>(
                                p.wo + static_cast<int64_t>(o) * p.ldwo + col0 + v * 8) : make_uint4(0, 0, 0, 0);
                            const __half2* h2 = reinterpret_cast<const __half2*>(&q);
                            float4* dst = reinterpret_cast<float4*>(smem_wo + o * TBN + v * 8);
                            const float2 f0 = __half22float2(h2[0]), f1 = __half22float2(h2[1]);
                            const float2 f2 = __half22float2(h2[2]), f3 = __half22float2(h2[3]);
                            dst[0] = make_float4(f0.x, f0.y, f1.x, f1.y);
                            dst[1] = make_float4(f2.x, f2.y, f3.x, f3.y);
                        }
                    } else {
                        for (int i = et; i < n_cls * TBN; i += EPI_THREADS) {
                            const int o = i / TBN, j = i % TBN;
                            const int64_t c = col0 + j;
                            float v = 0.0f;
                            if (c < n_live && o < n_out) {
                                const int64_t gc = mapped ? cmap[c] : c;
                                v = wo_fast ? __half2float(p.wo[static_cast<int64_t>(o) * p.ldwo + gc])
                                            : __half2float(p.w[static_cast<int64_t>(p.o_idx[o]) * p.ldw + gc]);
                            }
                            smem_wo[o * TBN + j] = v;
                        }
                    }
                }
                named_bar_sync(1, EPI_THREADS);
                const float ax = row_ok ? amax_or_127(p.row_amax[row]) : 127.0f;
                rowf = ax;
                sx = 127.0 / static_cast<double>(ax);
                if (stage_wo) {
#pragma unroll
                    for (int o = 0; o < WOC; ++o) {
                        float v = 0.0f;
                        if (o < n_out && row_ok)
                            v = xo_fast ? __half2float(p.xo[row * p.o_cap + o])
                                        : __half2float(p.x[row * p.ldx + p.o_idx[o]]);
                        xo_r[o] = v;
                    }
                }
            }

            if (warp == EPI_WARP0 && lane == 0 && it == 0) gstamp(p.dbg, 8);
            if ((kDev && p.dbg != nullptr)) {
                const long long c0 = clock64();
                mbar_wait(&bars->tmem_full[acc], acc_phase);
                w_tf += clock64() - c0;
            }
            mbar_wait(&bars->tmem_full[acc], acc_phase);
            tc_fence_after();
            if (warp == EPI_WARP0 && lane == 0 && it == 0) gstamp(p.dbg, 5);
            const uint32_t t_row = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) +
                                   static_cast<uint32_t>(acc * BN);
            // one 32-column chunk of this thread's row: dequant + outlier term + store
            auto emit = [&](int ch, uint32_t (&r)[32]) {
                const int64_t cbase = col0 + ch * 32;
                if (cbase >= n_live) return;  // warp-uniform
                // columns owned by a patch tile are skipped by the main tile (same launch)
                const uint32_t pm = (!mapped && p.patch_mask != nullptr) ? p.patch_mask[cbase >> 5] : 0u;
                // TS: whole 32 x 32 box through smem + TMA (rows >= M, cols >= N clipped by TMA)
                const bool tma_chunk = TS && !mapped && pm == 0u && p.tma_y;
                if (!tma_chunk && !row_ok) return;
                const bool full_chunk = !mapped && pm == 0u && p.vec_store && cbase + 32 <= n_live;
                if constexpr (EPI == EPI_I32) {
                    int32_t* yr = reinterpret_cast<int32_t*>(p.y) + row * p.ldy;
                    if (full_chunk) {
#pragma unroll
                        for (int u = 0; u < 8; ++u)
                            *reinterpret_cast<uint4*>(yr + cbase + 4 * u) =
                                make_uint4(r[4 * u], r[4 * u + 1], r[4 * u + 2], r[4 * u + 3]);
                    } else {
                        for (int j = 0; j < 32; ++j) {
                            const int64_t c = cbase + j;
                            if (c < n_live && !((pm >> j) & 1u)) yr[mapped ? cmap[c] : c] = static_cast<int32_t>(r[j]);
                        }
                    }
                } else {
                    float v[32];
                    if constexpr (EPI == EPI_F32_EXACT) {
                        // f32( f64(C) / (sx*sw) ) then f32( f64(.) + ordered f64 outlier sum )
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            const double d = __dmul_rn(sx, smem_col[ch * 32 + j]);
                            const double q =
                                __ddiv_rn(static_cast<double>(static_cast<int32_t>(r[j])), d);
                            v[j] = __double2float_rn(q);
                        }
                        if (n_out > 0 && stage_wo) {
                            // the staged fp16 values (exact in f32 and f64): x[row, O] in
                            // registers, W[O, tile] in shared memory, same ascending order
                            const float* wrow = smem_wo + ch * 32;
                            for (int j = 0; j < 32; ++j) {
                                if (cbase + j >= n_live) break;
                                double hacc = 0.0;
                                for (int o = 0; o < n_out; ++o)
                                    hacc = __dadd_rn(hacc, __dmul_rn(static_cast<double>(xo_r[o]),
                                                                     static_cast<double>(wrow[o * TBN + j])));
                                v[j] = __double2float_rn(__dadd_rn(static_cast<double>(v[j]), hacc));
                            }
                        } else if (n_out > 0) {
                            for (int j = 0; j < 32; ++j) {
                                const int64_t c = cbase + j;
                                if (c >= n_live) break;
                                const int64_t gc = mapped ? cmap[c] : c;
                                double hacc = 0.0;
                                for (int o = 0; o < n_out; ++o) {
                                    const int64_t k = p.o_idx[o];
                                    const double xv = __half2float(p.x[row * p.ldx + k]);
                                    const double wv = __half2float(p.w[k * p.ldw + gc]);
                                    hacc = __dadd_rn(hacc, __dmul_rn(xv, wv));
                                }
                                v[j] = __double2float_rn(__dadd_rn(static_cast<double>(v[j]), hacc));
                            }
                        }
                    } else {
                        // dequant + outlier FMAs on packed f32x2 (sm_100 FMUL2 / FFMA2)
                        const float4* cf4 = reinterpret_cast<const float4*>(
                            reinterpret_cast<const float*>(smem_col) + ch * 32);
                        float2* v2 = reinterpret_cast<float2*>(v);
                        const float2 rf2 = make_float2(rowf, rowf);
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            const float4 f = cf4[u];
                            const float2 c01 = make_float2(static_cast<float>(static_cast<int32_t>(r[4 * u + 0])),
                                                           static_cast<float>(static_cast<int32_t>(r[4 * u + 1])));
                            const float2 c23 = make_float2(static_cast<float>(static_cast<int32_t>(r[4 * u + 2])),
                                                           static_cast<float>(static_cast<int32_t>(r[4 * u + 3])));
                            v2[2 * u] = __fmul2_rn(__fmul2_rn(c01, rf2), make_float2(f.x, f.y));
                            v2[2 * u + 1] = __fmul2_rn(__fmul2_rn(c23, rf2), make_float2(f.z, f.w));
                        }
                        if (n_out > 0 && !(kDev && (p.dbg_epi & 1))) {
                            if (stage_wo) {
                                const float* wrow = smem_wo + ch * 32;
                                if (n_cls == 4) outlier_fma<4, TBN>(v2, xo_r, wrow);
                                else if (n_cls == 6) outlier_fma<6, TBN>(v2, xo_r, wrow);
                                else if (n_cls == 8) outlier_fma<8, TBN>(v2, xo_r, wrow);
                                else outlier_fma<WOC, TBN>(v2, xo_r, wrow);
                            } else {
                                for (int o = 0; o < n_out; ++o) {
                                    const int64_t k = p.o_idx[o];
                                    const float xv = __half2float(p.x[row * p.ldx + k]);
                                    for (int j = 0; j < 32; ++j) {
                                        const int64_t c = cbase + j;
                                        float wv = 0.0f;
                                        if (c < n_live)
                                            wv = __half2float(p.w[k * p.ldw + (mapped ? cmap[c] : c)]);
                                        v[j] = fmaf(xv, wv, v[j]);
                                    }
                                }
                            }
                        }
                    }
                    if constexpr (EPI == EPI_F16) {
                        if (p.n_peer > 0 && row_ok) {  // fused all-gather: the same values to every peer
                            uint4 pkv[4];
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                uint32_t pk[4];
#pragma unroll
                                for (int e = 0; e < 4; ++e) {
                                    __half2 h2 = __floats2half2_rn(v[8 * u + 2 * e], v[8 * u + 2 * e + 1]);
                                    pk[e] = *reinterpret_cast<uint32_t*>(&h2);
                                }
                                pkv[u] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                            }
                            for (int q = 0; q < p.n_peer; ++q) {
                                __half* yq = reinterpret_cast<__half*>(p.y_peer[q]) + row * p.peer_ldy + p.peer_col;
                                if (full_chunk && p.peer_vec) {
#pragma unroll
                                    for (int u = 0; u < 4; ++u) *reinterpret_cast<uint4*>(yq + cbase + 8 * u) = pkv[u];
                                } else {
                                    for (int j = 0; j < 32; ++j) {
                                        const int64_t c = cbase + j;
                                        if (c < n_live && !((pm >> j) & 1u))
                                            yq[mapped ? cmap[c] : c] = __float2half_rn(v[j]);
                                    }
                                }
                            }
                        }
                    }
                    if (kDev && (p.dbg_epi & 2)) {
                        if (v[0] == 1234.5f) reinterpret_cast<float*>(p.y)[0] = v[1];  // keep v live
                    } else if (tma_chunk) {
                        // stage this row's 32 outputs (64 B) in the warp's tile, then one
                        // elected lane stores the 32 x 32 box; two tiles alternate so
                        // the next chunk's writes overlap the previous store
                        const int ew = warp - EPI_WARP0;
                        uint8_t* tile = smem_stg + (ew * 2 + (stg_cnt & 1)) * STG_BYTES;
                        if (stg_cnt >= 2) {
                            if (lane == 0) tma_store_wait_read<1>();
                            __syncwarp();
                        }
                        uint4* dst = reinterpret_cast<uint4*>(tile + lane * 64);
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            uint32_t pk[4];
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                __half2 h2 = __floats2half2_rn(v[8 * u + 2 * e], v[8 * u + 2 * e + 1]);
                                pk[e] = *reinterpret_cast<uint32_t*>(&h2);
                            }
                            dst[u ^ ((lane >> 1) & 3)] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                        }
                        fence_proxy_async_smem();
                        __syncwarp();
                        if (lane == 0) {
                            tma_store_2d(&tmap_y, tile, static_cast<int32_t>(cbase),
                                         static_cast<int32_t>(row - lane));
                            tma_store_commit();
                        }
                        ++stg_cnt;
                    } else if constexpr (EPI == EPI_F16) {
                        __half* yr = reinterpret_cast<__half*>(p.y) + row * p.ldy;
                        if (full_chunk) {
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                uint32_t pk[4];
#pragma unroll
                                for (int e = 0; e < 4; ++e) {
                                    __half2 h2 = __floats2half2_rn(v[8 * u + 2 * e], v[8 * u + 2 * e + 1]);
                                    pk[e] = *reinterpret_cast<uint32_t*>(&h2);
                                }
                                *reinterpret_cast<uint4*>(yr + cbase + 8 * u) =
                                    make_uint4(pk[0], pk[1], pk[2], pk[3]);
                            }
                        } else {
                            for (int j = 0; j < 32; ++j) {
                                const int64_t c = cbase + j;
                                if (c < n_live && !((pm >> j) & 1u)) yr[mapped ? cmap[c] : c] = __float2half_rn(v[j]);
                            }
                        }
                    } else {
                        float* yr = reinterpret_cast<float*>(p.y) + row * p.ldy;
                        if (full_chunk) {
#pragma unroll
                            for (int u = 0; u < 8; ++u)
                                *reinterpret_cast<float4*>(yr + cbase + 4 * u) =
                                    make_float4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]);
                        } else {
                            for (int j = 0; j < 32; ++j) {
                                const int64_t c = cbase + j;
                                if (c < n_live && !((pm >> j) & 1u)) yr[mapped ? cmap[c] : c] = v[j];
                            }
                        }
                    }
                }
                        };
            const bool split = CG == 1 && p.ksplit > 1;
            // split-K: c32 column of this tile's first column (patch tiles after the main ones)
            const int64_t c32_col = (is_patch ? static_cast<int64_t>(ts.n_tiles) * BN : 0) +
                                    static_cast<int64_t>(n_blk) * BN;
#pragma unroll 1
            for (int cc = 0; cc < COLS_PER_WARP / 32; ++cc) {
                const int ch = half * (COLS_PER_WARP / 32) + cc;
                uint32_t r[32];
                tmem_ld_32x32b_x32(t_row + ch * 32, r);
                tmem_ld_wait();
                if (!split) {
                    emit(ch, r);
                } else if (row_ok) {  // add this K-range's partial sums (fire-and-forget reds)
                    int32_t* cr = p.c32 + (c32_col + ch * 32) * p.c32_rows + row;
#pragma unroll
                    for (int j = 0; j < 32; ++j) red_add_s32(cr + j * p.c32_rows, static_cast<int32_t>(r[j]));
                }
            }
            if (warp == EPI_WARP0 && lane == 0 && it == 0) gstamp(p.dbg, 6);
            // accumulator drained: hand TMEM back to the MMA warp
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if constexpr (CG == 2) mbar_arrive_remote(&bars->tmem_empty[acc], leader_rank);
                else mbar_arrive(&bars->tmem_empty[acc]);
            }
            if constexpr (CG == 1) {
                if (split) {  // the tile's last K-range to arrive runs the epilogue on the sums
                    // every thread's reductions are ordered before thread 0's acq_rel
                    // count by the barrier (cumulativity), and the last arriver's loads
                    // after it by the second barrier: no per-thread GPU-scope fence
                    named_bar_sync(2, EPI_THREADS);
                    if (et == 0 && it == 0) gstamp(p.dbg, 9);
                    if (et == 0) {
                        int old;
                        asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;"
                                     : "=r"(old)
                                     : "l"(p.c32_cnt + t)
                                     : "memory");
                        split_last = old == p.ksplit - 1;
                    }
                    named_bar_sync(2, EPI_THREADS);
                    if (et == 0 && it == 0) gstamp(p.dbg, 10);
                    if (split_last) {
#pragma unroll 1
                        for (int cc = 0; cc < COLS_PER_WARP / 32; ++cc) {
                            const int ch = half * (COLS_PER_WARP / 32) + cc;
                            uint32_t r[32];
                            int32_t* cr = p.c32 + (c32_col + ch * 32) * p.c32_rows + (row_ok ? row : 0);
#pragma unroll
                            for (int j = 0; j < 32; ++j)
                                r[j] = row_ok ? static_cast<uint32_t>(__ldcg(cr + j * p.c32_rows)) : 0u;
                            // leave the scratch zeroed for the next GEMM over it
                            if (row_ok) {
#pragma unroll
                                for (int j = 0; j < 32; ++j) __stcg(cr + j * p.c32_rows, 0);
                            }
                            emit(ch, r);
                        }
                        named_bar_sync(2, EPI_THREADS);
                        if (et == 0) {
                            p.c32_cnt[t] = 0;  // and the tile's arrival counter
                            gstamp(p.dbg, 11);
                        }
                    }
                }
            }
        }
        if (TS && lane == 0) tma_store_wait<0>();  // staged outputs fully written
        if ((kDev && p.dbg != nullptr) && warp == EPI_WARP0 && lane == 0)
            p.dbg[blockIdx.x * 16 + 15] = static_cast<unsigned long long>(w_tf);
    }

    __syncthreads();
    if (threadIdx.x == 0) gstamp(p.dbg, 7);
    if constexpr (C::CLUSTER > 1) cluster_sync_all();  // all CTAs done with TMEM and barriers
    if (warp == 2) {
        tc_fence_after();
        if constexpr (CG == 2) tmem_dealloc_pair<TMEM_COLS>(tmem_base);
        else tmem_dealloc<TMEM_COLS>(tmem_base);
    }
}

// ------------------------------------------------------------------ host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(ptr);
    });
    return fn;
}

// int8 K-major operand [rows x K] with row pitch ld bytes; box = box_rows x 128 B.
bool make_tmap_i8(CUtensorMap* map, const int8_t* base, int64_t rows, int64_t K, int64_t ld,
                         int box_rows) {
    EncodeTiledFn enc = get_encode_fn();
    if (!enc) return false;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(rows)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld)};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(BK), static_cast<cuuint32_t>(box_rows)};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<int8_t*>(base), dims,
                     strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// fp16 output Y [rows x cols], row pitch ld elements; box = 32 x 32, the
// staging tile's 16-byte chunks XOR-swizzled by (row >> 1) & 3 (SWIZZLE_64B)
static bool make_tmap_f16_out(CUtensorMap* map, void* base, int64_t rows, int64_t cols, int64_t ld) {
    EncodeTiledFn enc = get_encode_fn();
    if (!enc) return false;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * 2)};
    cuuint32_t box[2] = {32, 32};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, base, dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                     CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

template <int EPI, int CG, int MC, int NW>
static cudaError_t launch_epi(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tp,
                              const CUtensorMap& ty, const Params& p, int64_t max_tiles,
                              cudaStream_t st) {
    static std::once_flag once;
    static cudaError_t attr_err = cudaSuccess;
    static int max_clusters = 0;
    constexpr size_t smem = smem_total<CG, MC, EPI == EPI_F16 && CG == 2, NW>();
    static_assert(smem <= 227 * 1024, "shared memory");
    constexpr int CL = CG * MC;
    cudaLaunchConfig_t cfg{};
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    std::call_once(once, [&] {
        attr_err = cudaFuncSetAttribute(gemm_i8_kernel<EPI, CG, MC, NW>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(smem));
        // how many clusters of this shape the GPC layout can co-schedule
        cudaLaunchConfig_t q = cfg;
        q.gridDim = dim3(static_cast<unsigned>(num_sms() / CL * CL));
        int n = 0;
        if (attr_err == cudaSuccess &&
            cudaOccupancyMaxActiveClusters(&n, gemm_i8_kernel<EPI, CG, MC, NW>, &q) == cudaSuccess && n > 0)
            max_clusters = n;
        else
            max_clusters = num_sms() / CL;
        cudaGetLastError();
    });
    if (attr_err != cudaSuccess) return attr_err;
    const int64_t units = max_tiles * p.ksplit;
    int64_t clusters = units < max_clusters ? units : max_clusters;
    // tests only: I8MM_GEMM_MAX_CLUSTERS=c caps the persistent grid so that
    // small shapes run many tiles per CTA (pair): accumulator double-buffering,
    // per-tile restaging and the grouped raster at production depth
    if (const char* e = getenv("I8MM_GEMM_MAX_CLUSTERS")) {
        const int cap = atoi(e);
        if (cap > 0 && clusters > cap) clusters = cap;
    }
    cfg.gridDim = dim3(static_cast<unsigned>(clusters * CL));
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, gemm_i8_kernel<EPI, CG, MC, NW>, ta, tb, tp, ty, p);
    count_launch();
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

template <int EPI>
static cudaError_t launch_cg(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tp,
                             const CUtensorMap& ty, const Params& p, int64_t max_tiles, int cg,
                             int mc, int nw, cudaStream_t st) {
    if (cg == 2 && mc == 2) return launch_epi<EPI, 2, 2, 1>(ta, tb, tp, ty, p, max_tiles, st);
    if (cg == 2 && nw == 2) return launch_epi<EPI, 2, 1, 2>(ta, tb, tp, ty, p, max_tiles, st);
    if (cg == 2) return launch_epi<EPI, 2, 1, 1>(ta, tb, tp, ty, p, max_tiles, st);
    return launch_epi<EPI, 1, 1, 1>(ta, tb, tp, ty, p, max_tiles, st);
}

}  // namespace gemm

bool make_tmap_i8_rows(CUtensorMap* map, const int8_t* base, int64_t rows, int64_t K, int64_t ld,
                       int box_rows) {
    return gemm::make_tmap_i8(map, base, rows, K, ld, box_rows);
}

// fp16 [rows x cols] (row pitch ld elements, 16-byte aligned), box = 128 columns
// x box_rows rows, no swizzle (rows land 256 bytes apart); OOB elements read 0
bool make_tmap_f16_rows(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int64_t ld,
                        int box_rows) {
    gemm::EncodeTiledFn enc = gemm::get_encode_fn();
    if (!enc) return false;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * 2)};
    cuuint32_t box[2] = {128, static_cast<cuuint32_t>(box_rows)};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// Kernel-variant overrides for tests / A-B measurements:
//   I8MM_FORCE_CG1=1 pins the 1-CTA kernel; I8MM_GEMM_MC=2 enables the
//   B-multicast cluster of two CTA pairs (M >= 2048).
static int env_int(const char* name) {
    const char* e = getenv(name);
    return (e && e[0]) ? atoi(e) : 0;
}
static int g_cg_override = -1, g_mc_override = -1;
static int gemm_cg_override() {
    if (g_cg_override < 0) g_cg_override = env_int("I8MM_FORCE_CG1") == 1 ? 1 : 0;
    return g_cg_override;
}
static int gemm_mc_override() {
    if (g_mc_override < 0) g_mc_override = env_int("I8MM_GEMM_MC");
    return g_mc_override;
}
// 512-wide pair tiles: env I8MM_GEMM_WIDE = 1 forces, 2 forbids; default by shape
static bool gemm_wide_mode(int64_t M, int64_t N, int64_t K) {
    const int e = env_int("I8MM_GEMM_WIDE");
    if (e == 1) return true;
    if (e == 2) return false;
    // its epilogue cannot overlap the next tile's MMAs (one 512-column accumulator),
    // so it pays only when the K loop is long (measured, scripts/gemm_wide_ab.sh:
    // cfg5 fc2 K = 49152 +15 %, cfg5 fc1 K = 12288 -4 %, cfg4 fc1 K = 9216 -8 %)
    return M >= 2048 && N >= 2 * gemm::BN && K >= 32768;
}

void set_gemm_variant(int cg, int mc) {
    g_cg_override = cg;
    g_mc_override = mc;
}

int64_t gemm_split_tiles(int64_t N, bool patches) {
    const int64_t nt = (N + gemm::BN - 1) / gemm::BN;
    return patches ? 2 * nt : nt;
}
int64_t gemm_split_cols(int64_t N, bool patches) { return gemm_split_tiles(N, patches) * gemm::BN; }

// K-split of the single-m-tile GEMM: units ~ one per SM, each keeping >= 16
// K-blocks (2 KB of K), and only for K >= 8192 where the per-unit costs
// (partial-sum reds, the last unit's read-back, zeroing the scratch) pay:
// measured OPT-13B fc2 (K = 20480) M = 32..128: 96-102 -> 61-72 us; qkvo
// (K = 5120) lost 4-6 us, so it is not split. 1 = no split.
int gemm_split_factor(int64_t M, int64_t N, int64_t K) {
    static int off = -1;
    if (off < 0) {
        const char* e = getenv("I8MM_NO_SPLITK");
        off = (e && e[0] == '1') ? 1 : 0;
    }
    static int force = -1;  // I8MM_SPLITK_FORCE=S: A/B measurements only
    if (force < 0) {
        const char* e = getenv("I8MM_SPLITK_FORCE");
        force = (e && e[0]) ? atoi(e) : 0;
    }
    if (force >= 2 && M > 0 && M <= gemm::BM) return force;
    if (off || M <= 0 || M > gemm::BM || K < 8192) return 1;
    const int64_t num_kb = (K + gemm::BK - 1) / gemm::BK;
    const int64_t main_tiles = (N + gemm::BN - 1) / gemm::BN;
    int64_t sk = num_sms() / (main_tiles > 0 ? main_tiles : 1);
    if (sk > num_kb / 16) sk = num_kb / 16;
    if (sk > 16) sk = 16;
    return sk >= 2 ? static_cast<int>(sk) : 1;
}

// m-tiles per raster group (see launch_gemm_one)
static int raster_group_m(int64_t N, int64_t K, int cg, int mc, int tbn) {
    using namespace gemm;
    const int gm_env = env_int("I8MM_GROUP_M");
    if (gm_env > 0) return gm_env;
    const int64_t n_tiles = (N + tbn - 1) / tbn;
    const int64_t wave = num_sms() / (cg * mc);
    if (n_tiles * 2 <= wave) return 1;
    const int64_t panel = static_cast<int64_t>(BM) * cg * mc * (K > 0 ? K : 1);
    const int64_t g = (32LL << 20) / panel;
    int gm = 1;
    while (gm * 2 <= g && gm < 32) gm *= 2;
    return gm;
}

static cudaError_t launch_gemm_one(const GemmArgs& a, int epi, cudaStream_t st);

// Row chunks (measured, profiles/r2/gemm_chunk_ab.txt): a persistent launch over
// many raster groups lets its clusters drift apart by several tiles, so the
// tiles in flight span more than one group and the L2 stops holding the group's
// panels: cfg5 fc1 read 18.5 GB of DRAM for 0.8 GB of operands. One launch per
// chunk of whole groups (>= 8 waves of tiles, so the last wave's idle SMs stay a
// small share) resets the drift: 6.75 GB, and the power-capped SM clock rises
// 1.29 -> 1.48 GHz (+8-12 % on the bench line). I8MM_GEMM_CHUNK_WAVES=0 disables.
cudaError_t launch_gemm_sm100(const GemmArgs& a, int epi, cudaStream_t st) {
    using namespace gemm;
    if (a.M <= 0 || a.N <= 0) return cudaSuccess;
    const char* cw_env = getenv("I8MM_GEMM_CHUNK_WAVES");  // read per call (tests set it)
    const int chunk_waves = (cw_env && cw_env[0]) ? atoi(cw_env) : 8;
    if (chunk_waves > 0 && a.M > BM && a.c32 == nullptr) {
        const int cg = gemm_cg_override() != 1 ? 2 : 1;
        const int mc = (cg == 2 && a.M >= 2048 && gemm_mc_override() == 2) ? 2 : 1;
        const int nw = (cg == 2 && mc == 1 && gemm_wide_mode(a.M, a.N, a.K)) ? 2 : 1;
        const int tbn = BN * nw;
        const int gm = raster_group_m(a.N, a.K, cg, mc, tbn);
        const int64_t group_rows = static_cast<int64_t>(gm) * BM * cg * mc;
        const int64_t n_tiles = (a.N + tbn - 1) / tbn;
        const int64_t wave = num_sms() / (cg * mc);
        const int64_t groups_per_chunk = (chunk_waves * wave + gm * n_tiles - 1) / (gm * n_tiles);
        const int64_t chunk = group_rows * (groups_per_chunk > 0 ? groups_per_chunk : 1);
        if (gm > 1 && a.M > chunk + group_rows / 2) {
            const int elt = epi == EPI_F16 ? 2 : 4;
            for (int64_t r0 = 0; r0 < a.M; r0 += chunk) {
                // a short tail joins the previous chunk
                const int64_t rows = (a.M - r0 < chunk + group_rows / 2) ? a.M - r0 : chunk;
                GemmArgs c = a;
                c.a = a.a + r0 * a.lda;
                c.M = rows;
                c.y = static_cast<char*>(a.y) + r0 * a.ldy * elt;
                if (a.row_amax) c.row_amax = a.row_amax + r0;
                if (a.x) c.x = a.x + r0 * a.ldx;
                if (a.xo) c.xo = a.xo + r0 * a.o_cap;
                for (int q = 0; q < a.n_peer; ++q)
                    c.y_peer[q] = static_cast<char*>(a.y_peer[q]) + r0 * a.peer_ldy * 2;
                if (cudaError_t e = launch_gemm_one(c, epi, st)) return e;
                if (rows != chunk) break;
            }
            return cudaSuccess;
        }
    }
    return launch_gemm_one(a, epi, st);
}

static cudaError_t launch_gemm_one(const GemmArgs& a, int epi, cudaStream_t st) {
    using namespace gemm;
    if ((a.lda % 16) || (a.ldb % 16) || (reinterpret_cast<uintptr_t>(a.a) & 15) ||
        (reinterpret_cast<uintptr_t>(a.b) & 15))
        return cudaErrorInvalidValue;
    // CTA pairs (cta_group::2, 256-row tiles) unless M fits one 128-row tile.
    // The 4-CTA cluster that multicasts WqT between two pairs (MC=2) halves the
    // B-operand L2 reads but only 132 SMs can host 4-CTA clusters; measured
    // (profiles/) it does not beat plain pairs, so it is opt-in (I8MM_GEMM_MC=2).
    const int cg = (a.M > BM && gemm_cg_override() != 1) ? 2 : 1;
    const int mc = (cg == 2 && a.M >= 2048 && gemm_mc_override() == 2) ? 2 : 1;
    // 256 x 512 pair tiles (two N=256 MMAs share each A panel: 0.75x the L2 -> SM
    // bytes of 256 x 256, the ceiling of this GEMM at full clock) when the
    // layer is big enough in N and K for one accumulator without epilogue overlap
    const int nw = (cg == 2 && mc == 1 && gemm_wide_mode(a.M, a.N, a.K)) ? 2 : 1;
    const int tbn = BN * nw;
    CUtensorMap ta, tb;
    const int64_t kdim = a.K > 0 ? a.K : 16;
    if (!make_tmap_i8(&ta, a.a, a.M, kdim, a.lda, BM)) return cudaErrorInvalidValue;
    if (!make_tmap_i8(&tb, a.b, a.N, kdim, a.ldb, BN / cg / mc)) return cudaErrorInvalidValue;
    CUtensorMap tp = tb;
    if (a.patch_count != nullptr &&
        !make_tmap_i8(&tp, a.b_patch, a.N, kdim, a.ldb, BN / cg / mc))
        return cudaErrorInvalidValue;
    Params p{};
    p.M = a.M;
    p.N = a.N;
    p.K = a.K;
    p.num_kb = static_cast<int>((a.K + BK - 1) / BK);
    if (p.num_kb == 0) p.num_kb = 1;  // K == 0: one zero-filled block -> C = 0
    p.m_tiles = static_cast<int>((a.M + BM * cg * mc - 1) / (BM * cg * mc));
    // upper bound on tiles (patches at most double the N-tiles); the kernel
    // computes the live count on the device
    const int64_t max_tiles = static_cast<int64_t>(p.m_tiles) * ((a.N + tbn - 1) / tbn) *
                              (a.patch_count != nullptr ? 2 : 1);
    p.y = a.y;
    p.ldy = a.ldy;
    p.row_amax = a.row_amax;
    p.col_amax = a.col_amax;
    p.x = a.x;
    p.ldx = a.ldx;
    p.w = a.w;
    p.ldw = a.ldw;
    p.xo = a.xo;
    p.o_cap = a.o_cap;
    p.o_idx = a.o_idx;
    p.o_count = a.o_count;
    p.wo = a.wo;
    p.ldwo = a.ldwo;
    p.wo_cap = a.wo ? a.wo_cap : 0;
    p.patch_count = a.patch_count;
    p.patch_idx = a.patch_idx;
    p.patch_amax = a.patch_amax;
    p.patch_mask = a.patch_mask;
    const int elt = (epi == EPI_F16) ? 2 : 4;
    p.vec_store = ((a.ldy * elt) % 16 == 0) && ((reinterpret_cast<uintptr_t>(a.y) & 15) == 0);
    p.dbg_epi = env_int("I8MM_DBG_EPI");
    p.dbg = debug_timeline();
    p.n_peer = 0;
    if (epi == EPI_F16 && a.n_peer > 0) {
        if (a.n_peer > kMaxPeers) return cudaErrorInvalidValue;
        p.n_peer = a.n_peer;
        for (int q = 0; q < a.n_peer; ++q) p.y_peer[q] = a.y_peer[q];
        p.peer_ldy = a.peer_ldy;
        p.peer_col = a.peer_col;
        bool vec = (a.peer_ldy % 8 == 0) && (a.peer_col % 8 == 0);
        for (int q = 0; q < a.n_peer; ++q) vec = vec && (reinterpret_cast<uintptr_t>(a.y_peer[q]) & 15u) == 0;
        p.peer_vec = vec ? 1 : 0;
    }
    // split-K when one m-tile's N-tiles would leave most SMs idle (M <= 128)
    p.ksplit = 1;
    if (cg == 1 && a.c32 != nullptr && p.m_tiles == 1) {
        const int sk = gemm_split_factor(a.M, a.N, a.K);
        if (sk >= 2) {
            p.ksplit = static_cast<int>(sk);
            p.c32 = a.c32;
            p.c32_rows = a.c32_rows;
            p.c32_cnt = a.c32_cnt;
        }
    }
    {
        // Raster (measured, scripts/ab_raster.sh): when one wave of concurrent
        // tiles covers >= 2 full rows of N-tiles, B panels are reused within the
        // wave -> row-major (group 1); otherwise group GROUP_M m-tiles so their
        // A panels (GROUP_M x TILE_M x K bytes) stay within ~32 MB of L2 while
        // the B panels stream past them.
        p.group_m = raster_group_m(a.N, a.K, cg, mc, tbn);
        const int pol_env = env_int("I8MM_GEMM_L2POL");
        // bit 0: A panels evict_last, bit 1: B panels evict_first (measured: B panels
        // are reused by the group's m-tiles, evict_first on them costs ~10 %)
        p.l2_pol = pol_env > 0 ? pol_env : 0;
    }
    CUtensorMap ty = ta;
    p.tma_y = 0;
    if (epi == EPI_F16 && p.vec_store && env_int("I8MM_NO_TMA_STORE") != 1)
        p.tma_y = make_tmap_f16_out(&ty, a.y, a.M, a.N, a.ldy) ? 1 : 0;
    switch (epi) {
        case EPI_I32: return launch_cg<EPI_I32>(ta, tb, tp, ty, p, max_tiles, cg, mc, nw, st);
        case EPI_F16: return launch_cg<EPI_F16>(ta, tb, tp, ty, p, max_tiles, cg, mc, nw, st);
        case EPI_F32: return launch_cg<EPI_F32>(ta, tb, tp, ty, p, max_tiles, cg, mc, nw, st);
        case EPI_F32_EXACT: return launch_cg<EPI_F32_EXACT>(ta, tb, tp, ty, p, max_tiles, cg, mc, nw, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace i8mm
