// K4: int8 x int8 -> int32 GEMM on the 5th-gen tensor cores (tcgen05, sm_100a)
// with the LLM.int8() epilogue fused in: vector-wise dequantization by the
// outer product of row/column absmax (gemm.py:120-147, row x col branch) plus
// the high-precision outlier term sum_{o in O} X[:,o] W[o,:] (gemm.py:238,
// 244-247), written straight to the output tile.
//
// Structure (one CTA per SM, persistent, warp-specialised, 256 threads):
//   warp 0      TMA producer   : A (Xq, 128x128 B) + B (WqT, 256x128 B) per
//                                stage into a 4-deep SWIZZLE_128B smem ring
//   warp 1      MMA issuer     : tcgen05.mma.cta_group::1.kind::i8, M=128,
//                                N=256, K=32, accumulating in TMEM
//   warp 2      TMEM allocator : 512 columns = two 128x256 int32 accumulators
//   warps 4..7  epilogue       : tcgen05.ld -> dequant + outlier FMAs ->
//                                global stores, overlapping the next tile's
//                                mainloop (double-buffered TMEM)
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>

#include "kernels.cuh"
#include "sm100_ptx.cuh"

namespace i8mm {

namespace gemm {
constexpr int BM = 128;
constexpr int BN = 256;
constexpr int BK = 128;  // bytes == int8 elements: one SWIZZLE_128B atom row
constexpr int UMMA_K = 32;
constexpr int STAGES = 4;
constexpr int A_BYTES = BM * BK;
constexpr int B_BYTES = BN * BK;
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int WO_CAP = 16;  // outlier rows of W staged in smem per tile
constexpr int THREADS = 256;
constexpr int EPI_WARP0 = 4;
constexpr uint32_t TMEM_COLS = 2 * BN;
constexpr int GROUP_M = 16;

struct __align__(8) Barriers {
    uint64_t full[STAGES];
    uint64_t empty[STAGES];
    uint64_t tmem_full[2];
    uint64_t tmem_empty[2];
    uint32_t tmem_slot;
};

constexpr size_t SMEM_OPERANDS = static_cast<size_t>(STAGES) * STAGE_BYTES;
constexpr size_t SMEM_WO = static_cast<size_t>(WO_CAP) * BN * sizeof(float);
constexpr size_t SMEM_COLS = static_cast<size_t>(BN) * sizeof(double);
constexpr size_t SMEM_TOTAL = 1024 /*align slack*/ + SMEM_OPERANDS + SMEM_WO + SMEM_COLS +
                              sizeof(Barriers) + 64;

struct Params {
    int64_t M, N, K;
    int num_kb;
    int m_tiles, n_tiles, total_tiles;
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
    int vec_store;  // 1: y rows 16-byte aligned and N % (16/elt) == 0
};

__device__ __forceinline__ void tile_coords(const Params& p, int t, int& m_blk, int& n_blk) {
    // grouped raster: GROUP_M m-tiles share each B panel while it is hot in L2
    const int per_group = GROUP_M * p.n_tiles;
    const int g = t / per_group;
    const int first_m = g * GROUP_M;
    const int gm = min(GROUP_M, p.m_tiles - first_m);
    const int local = t - g * per_group;
    m_blk = first_m + local % gm;
    n_blk = local / gm;
}

__device__ __forceinline__ float amax_or_127(float a) { return a == 0.0f ? 127.0f : a; }

template <int EPI>
__global__ void __launch_bounds__(THREADS, 1)
    gemm_i8_kernel(const __grid_constant__ CUtensorMap tmap_a,
                   const __grid_constant__ CUtensorMap tmap_b, const Params p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    uint8_t* smem_a = smem;
    uint8_t* smem_b = smem + static_cast<size_t>(STAGES) * A_BYTES;
    float* smem_wo = reinterpret_cast<float*>(smem + SMEM_OPERANDS);
    double* smem_col = reinterpret_cast<double*>(smem + SMEM_OPERANDS + SMEM_WO);
    Barriers* bars = reinterpret_cast<Barriers*>(smem + SMEM_OPERANDS + SMEM_WO + SMEM_COLS);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        tma_prefetch_desc(&tmap_a);
        tma_prefetch_desc(&tmap_b);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&bars->full[s], 1);
            mbar_init(&bars->empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&bars->tmem_full[a], 1);
            mbar_init(&bars->tmem_empty[a], 4);  // one arrive per epilogue warp
        }
        fence_mbarrier_init();
    }
    if (warp == 2) tmem_alloc<TMEM_COLS>(&bars->tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = bars->tmem_slot;

    if (warp == 0) {
        // ===================== TMA producer =====================
        if (lane == 0) {
            const uint64_t pol = l2_policy_evict_normal();
            int stage = 0;
            uint32_t phase = 0;
            for (int t = blockIdx.x; t < p.total_tiles; t += gridDim.x) {
                int m_blk, n_blk;
                tile_coords(p, t, m_blk, n_blk);
                for (int kb = 0; kb < p.num_kb; ++kb) {
                    mbar_wait(&bars->empty[stage], phase ^ 1u);
                    mbar_arrive_expect_tx(&bars->full[stage], STAGE_BYTES);
                    tma_load_2d(&tmap_a, &bars->full[stage], smem_a + stage * A_BYTES, kb * BK,
                                m_blk * BM, pol);
                    tma_load_2d(&tmap_b, &bars->full[stage], smem_b + stage * B_BYTES, kb * BK,
                                n_blk * BN, pol);
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer =====================
        constexpr uint32_t idesc = idesc_i8(BM, BN);
        int stage = 0;
        uint32_t phase = 0;
        int it = 0;
        for (int t = blockIdx.x; t < p.total_tiles; t += gridDim.x, ++it) {
            const int acc = it & 1;
            const uint32_t acc_phase = (it >> 1) & 1;
            mbar_wait(&bars->tmem_empty[acc], acc_phase ^ 1u);
            tc_fence_after();
            const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * BN);
            for (int kb = 0; kb < p.num_kb; ++kb) {
                mbar_wait(&bars->full[stage], phase);
                tc_fence_after();
                if (lane == 0) {
                    const uint32_t a0 = smem_addr(smem_a + stage * A_BYTES);
                    const uint32_t b0 = smem_addr(smem_b + stage * B_BYTES);
#pragma unroll
                    for (int k = 0; k < BK / UMMA_K; ++k) {
                        const uint64_t ad = smem_desc_k_sw128(a0 + k * UMMA_K);
                        const uint64_t bd = smem_desc_k_sw128(b0 + k * UMMA_K);
                        mma_i8(d_tmem, ad, bd, idesc, (kb | k) != 0 ? 1u : 0u);
                    }
                    mma_commit(&bars->empty[stage]);  // frees the smem slot when MMAs finish
                }
                __syncwarp();
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1u;
                }
            }
            if (lane == 0) mma_commit(&bars->tmem_full[acc]);  // accumulator ready
            __syncwarp();
        }
    } else if (warp >= EPI_WARP0) {
        // ===================== epilogue =====================
        const int ew = warp - EPI_WARP0;  // == warp % 4: TMEM lanes 32*ew .. 32*ew+31
        const int et = threadIdx.x - EPI_WARP0 * 32;  // 0..127
        int n_out = 0;
        if constexpr (EPI != EPI_I32) n_out = p.o_count ? *p.o_count : 0;
        const bool fast_o = n_out <= WO_CAP && n_out <= p.o_cap && p.xo != nullptr;
        int it = 0;
        for (int t = blockIdx.x; t < p.total_tiles; t += gridDim.x, ++it) {
            int m_blk, n_blk;
            tile_coords(p, t, m_blk, n_blk);
            const int acc = it & 1;
            const uint32_t acc_phase = (it >> 1) & 1;
            const int64_t row = static_cast<int64_t>(m_blk) * BM + ew * 32 + lane;
            const int64_t col0 = static_cast<int64_t>(n_blk) * BN;
            const bool row_ok = row < p.M;

            float xo_r[WO_CAP];
            float rowf = 0.0f;
            double sx = 1.0;
            if constexpr (EPI != EPI_I32) {
                // stage per-tile column factors and outlier W rows in smem
                named_bar_sync(1, 128);  // previous tile's readers are done
                for (int j = et; j < BN; j += 128) {
                    const int64_t c = col0 + j;
                    const float aw = c < p.N ? amax_or_127(p.col_amax[c]) : 127.0f;
                    if constexpr (EPI == EPI_F32_EXACT)
                        smem_col[j] = 127.0 / static_cast<double>(aw);
                    else
                        reinterpret_cast<float*>(smem_col)[j] = aw * (1.0f / 16129.0f);
                }
                if (fast_o) {
                    for (int i = et; i < n_out * BN; i += 128) {
                        const int o = i / BN, j = i - (i / BN) * BN;
                        const int64_t c = col0 + j;
                        smem_wo[i] =
                            c < p.N ? __half2float(p.w[static_cast<int64_t>(p.o_idx[o]) * p.ldw + c])
                                    : 0.0f;
                    }
                }
                named_bar_sync(1, 128);
                const float ax = row_ok ? amax_or_127(p.row_amax[row]) : 127.0f;
                rowf = ax;
                sx = 127.0 / static_cast<double>(ax);
                if (fast_o) {
#pragma unroll
                    for (int o = 0; o < WO_CAP; ++o)
                        xo_r[o] = (o < n_out && row_ok) ? __half2float(p.xo[row * p.o_cap + o]) : 0.0f;
                }
            }

            mbar_wait(&bars->tmem_full[acc], acc_phase);
            tc_fence_after();
            const uint32_t t_row = tmem_base + (static_cast<uint32_t>(ew * 32) << 16) +
                                   static_cast<uint32_t>(acc * BN);
#pragma unroll 1
            for (int ch = 0; ch < BN / 32; ++ch) {
                uint32_t r[32];
                tmem_ld_32x32b_x32(t_row + ch * 32, r);
                tmem_ld_wait();
                const int64_t cbase = col0 + ch * 32;
                if (!row_ok) continue;
                if constexpr (EPI == EPI_I32) {
                    int32_t* yr = reinterpret_cast<int32_t*>(p.y) + row * p.ldy;
                    if (p.vec_store && cbase + 32 <= p.N) {
#pragma unroll
                        for (int u = 0; u < 8; ++u)
                            *reinterpret_cast<uint4*>(yr + cbase + 4 * u) =
                                make_uint4(r[4 * u], r[4 * u + 1], r[4 * u + 2], r[4 * u + 3]);
                    } else {
                        for (int j = 0; j < 32; ++j)
                            if (cbase + j < p.N) yr[cbase + j] = static_cast<int32_t>(r[j]);
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
                        if (n_out > 0) {
                            for (int j = 0; j < 32; ++j) {
                                const int64_t c = cbase + j;
                                if (c >= p.N) break;
                                double hacc = 0.0;
                                for (int o = 0; o < n_out; ++o) {
                                    const int64_t k = p.o_idx[o];
                                    const double xv = __half2float(p.x[row * p.ldx + k]);
                                    const double wv = __half2float(p.w[k * p.ldw + c]);
                                    hacc = __dadd_rn(hacc, __dmul_rn(xv, wv));
                                }
                                v[j] = __double2float_rn(__dadd_rn(static_cast<double>(v[j]), hacc));
                            }
                        }
                    } else {
                        const float* cf = reinterpret_cast<const float*>(smem_col) + ch * 32;
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            v[j] = static_cast<float>(static_cast<int32_t>(r[j])) * rowf * cf[j];
                        if (n_out > 0) {
                            if (fast_o) {
#pragma unroll
                                for (int o = 0; o < WO_CAP; ++o) {
                                    if (o < n_out) {
                                        const float xv = xo_r[o];
                                        const float* wr = smem_wo + o * BN + ch * 32;
#pragma unroll
                                        for (int j = 0; j < 32; ++j) v[j] = fmaf(xv, wr[j], v[j]);
                                    }
                                }
                            } else {
                                for (int o = 0; o < n_out; ++o) {
                                    const int64_t k = p.o_idx[o];
                                    const float xv = __half2float(p.x[row * p.ldx + k]);
                                    for (int j = 0; j < 32; ++j) {
                                        const int64_t c = cbase + j;
                                        const float wv = c < p.N ? __half2float(p.w[k * p.ldw + c]) : 0.0f;
                                        v[j] = fmaf(xv, wv, v[j]);
                                    }
                                }
                            }
                        }
                    }
                    if constexpr (EPI == EPI_F16) {
                        __half* yr = reinterpret_cast<__half*>(p.y) + row * p.ldy;
                        if (p.vec_store && cbase + 32 <= p.N) {
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
                            for (int j = 0; j < 32; ++j)
                                if (cbase + j < p.N) yr[cbase + j] = __float2half_rn(v[j]);
                        }
                    } else {
                        float* yr = reinterpret_cast<float*>(p.y) + row * p.ldy;
                        if (p.vec_store && cbase + 32 <= p.N) {
#pragma unroll
                            for (int u = 0; u < 8; ++u)
                                *reinterpret_cast<float4*>(yr + cbase + 4 * u) =
                                    make_float4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]);
                        } else {
                            for (int j = 0; j < 32; ++j)
                                if (cbase + j < p.N) yr[cbase + j] = v[j];
                        }
                    }
                }
            }
            // accumulator drained: hand TMEM back to the MMA warp
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bars->tmem_empty[acc]);
        }
    }

    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc<TMEM_COLS>(tmem_base);
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
static bool make_tmap_i8(CUtensorMap* map, const int8_t* base, int64_t rows, int64_t K, int64_t ld,
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

template <int EPI>
static cudaError_t launch_epi(const CUtensorMap& ta, const CUtensorMap& tb, const Params& p,
                              int grid, cudaStream_t st) {
    static std::once_flag once;
    static cudaError_t attr_err = cudaSuccess;
    std::call_once(once, [] {
        attr_err = cudaFuncSetAttribute(gemm_i8_kernel<EPI>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(SMEM_TOTAL));
    });
    if (attr_err != cudaSuccess) return attr_err;
    gemm_i8_kernel<EPI><<<grid, THREADS, SMEM_TOTAL, st>>>(ta, tb, p);
    count_launch();
    return cudaGetLastError();
}

}  // namespace gemm

cudaError_t launch_gemm_sm100(const GemmArgs& a, int epi, cudaStream_t st) {
    using namespace gemm;
    if (a.M <= 0 || a.N <= 0) return cudaSuccess;
    if ((a.lda % 16) || (a.ldb % 16) || (reinterpret_cast<uintptr_t>(a.a) & 15) ||
        (reinterpret_cast<uintptr_t>(a.b) & 15))
        return cudaErrorInvalidValue;
    CUtensorMap ta, tb;
    const int64_t kdim = a.K > 0 ? a.K : 16;
    if (!make_tmap_i8(&ta, a.a, a.M, kdim, a.lda, BM)) return cudaErrorInvalidValue;
    if (!make_tmap_i8(&tb, a.b, a.N, kdim, a.ldb, BN)) return cudaErrorInvalidValue;
    Params p{};
    p.M = a.M;
    p.N = a.N;
    p.K = a.K;
    p.num_kb = static_cast<int>((a.K + BK - 1) / BK);
    if (p.num_kb == 0) p.num_kb = 1;  // K == 0: one zero-filled block -> C = 0
    p.m_tiles = static_cast<int>((a.M + BM - 1) / BM);
    p.n_tiles = static_cast<int>((a.N + BN - 1) / BN);
    p.total_tiles = p.m_tiles * p.n_tiles;
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
    const int elt = (epi == EPI_F16) ? 2 : 4;
    p.vec_store = ((a.ldy * elt) % 16 == 0) && ((reinterpret_cast<uintptr_t>(a.y) & 15) == 0);
    const int grid = static_cast<int>(p.total_tiles < num_sms() ? p.total_tiles : num_sms());
    switch (epi) {
        case EPI_I32: return launch_epi<EPI_I32>(ta, tb, p, grid, st);
        case EPI_F16: return launch_epi<EPI_F16>(ta, tb, p, grid, st);
        case EPI_F32: return launch_epi<EPI_F32>(ta, tb, p, grid, st);
        case EPI_F32_EXACT: return launch_epi<EPI_F32_EXACT>(ta, tb, p, grid, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace i8mm
