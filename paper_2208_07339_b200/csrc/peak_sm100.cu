// Measured INT8 tensor-core ceiling of this B200: a kernel that
// does nothing but issue tcgen05.mma.kind::i8 from shared memory, one CTA (or
// CTA pair) per SM, so the roofline's denominator is this box's achievable
// dense int8 rate at its clocks and power cap, not the datasheet's 4.5 POPS.
//
// Operands are pseudo-random bytes (the tensor pipe's power draw depends on
// the data; zero operands would overstate the rate under a power cap). The
// issuing thread never waits inside the loop: the MMA queue back-pressures it.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/llmint8.h"
#include "kernels.cuh"
#include "sm100_ptx.cuh"

namespace i8mm {
namespace peak {

constexpr int STAGES = 2;       // distinct K-blocks cycled through
constexpr int A_BYTES = 128 * 128;  // 128 rows x 128 B (K = 128 int8), SWIZZLE_128B
constexpr int TMEM_COLS = 256;

template <int CG>
constexpr int b_bytes() { return (256 / CG) * 128; }
template <int CG>
constexpr size_t smem_bytes() { return 1024 + STAGES * (A_BYTES + b_bytes<CG>()); }

template <int CG>
__global__ void __launch_bounds__(128, 1) mma_peak_kernel(int iters) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sa = base;
    uint8_t* sb = base + STAGES * A_BYTES;
    __shared__ __align__(8) uint64_t done_bar;
    __shared__ uint32_t tmem_slot;
    const uint32_t rank = CG == 2 ? cluster_ctarank() : 0;
    const bool leader = rank == 0;
    // operands: a hash of the byte index (any int8 pattern is a valid operand)
    uint32_t* w32 = reinterpret_cast<uint32_t*>(base);
    const int words = STAGES * (A_BYTES + b_bytes<CG>()) / 4;
    for (int i = threadIdx.x; i < words; i += blockDim.x) {
        uint32_t h = static_cast<uint32_t>(i) * 2654435761u + blockIdx.x * 40503u + 0x9e3779b9u;
        h ^= h >> 15;
        h *= 2246822519u;
        h ^= h >> 13;
        w32[i] = h & 0x7f7f7f7fu;  // keep every byte in [0, 127] (no -128 code)
    }
    fence_proxy_async_smem();
    if (threadIdx.x == 0) {
        mbar_init(&done_bar, 1);
        fence_mbarrier_init();
    }
    __syncthreads();
    if constexpr (CG == 2) cluster_sync_all();
    if (threadIdx.x < 32) {
        if constexpr (CG == 2) tmem_alloc_pair<TMEM_COLS>(&tmem_slot);
        else tmem_alloc<TMEM_COLS>(&tmem_slot);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_slot;
    if (leader && threadIdx.x == 0) {
        constexpr uint32_t idesc = idesc_i8(128 * CG, 256);
        const uint32_t a0 = smem_addr(sa), b0 = smem_addr(sb);
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int s = 0; s < STAGES; ++s) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint64_t ad = smem_desc_k_sw128(a0 + s * A_BYTES + k * 32);
                    const uint64_t bd = smem_desc_k_sw128(b0 + s * b_bytes<CG>() + k * 32);
                    const uint32_t acc = (it | s | k) ? 1u : 0u;
                    if constexpr (CG == 2) mma_i8_pair(tmem, ad, bd, idesc, acc);
                    else mma_i8(tmem, ad, bd, idesc, acc);
                }
            }
        }
        if constexpr (CG == 2) mma_commit_pair(&done_bar, 0x3);
        else mma_commit(&done_bar);
    }
    mbar_wait(&done_bar, 0);
    tc_fence_after();
    __syncthreads();
    if constexpr (CG == 2) cluster_sync_all();
    if (threadIdx.x < 32) {
        if constexpr (CG == 2) tmem_dealloc_pair<TMEM_COLS>(tmem);
        else tmem_dealloc<TMEM_COLS>(tmem);
    }
}

template <int CG>
static cudaError_t launch(int iters, cudaStream_t st) {
    constexpr size_t smem = smem_bytes<CG>();
    cudaError_t e = cudaFuncSetAttribute(mma_peak_kernel<CG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(num_sms() / CG * CG));
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CG;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, mma_peak_kernel<CG>, iters);
    count_launch();
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

// Dev micro-benchmark: issue cost of small swap-AB MMAs (decode shape, M = 128
// weight rows, N = n_tok token rows, K = 32), cycling n_acc accumulators, one
// commit every `per_commit` MMAs (the decode kernel's per-unit stage release).
__global__ void __launch_bounds__(128, 1) mma_small_kernel(int iters, int n_tok, int n_acc, int per_commit,
                                                           unsigned long long* cycles) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sa = base;
    uint8_t* sb = base + STAGES * A_BYTES;
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tmem_slot;
    uint32_t* w32 = reinterpret_cast<uint32_t*>(base);
    for (int i = threadIdx.x; i < STAGES * (A_BYTES + 256 * 128) / 4; i += blockDim.x) w32[i] = 0x01010101u * (i & 7);
    fence_proxy_async_smem();
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_mbarrier_init();
    }
    __syncthreads();
    if (threadIdx.x < 32) tmem_alloc<512>(&tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_slot;
    if (threadIdx.x == 0) {
        const uint32_t idesc = idesc_i8(128, static_cast<uint32_t>(n_tok));
        const uint64_t ad0 = smem_desc_k_sw128(smem_addr(sa)), bd0 = smem_desc_k_sw128(smem_addr(sb));
        if (per_commit == 0) {  // lean: precomputed descriptors (+2 per 32 B), accumulator by mask
            for (int it = 0; it < iters; ++it) {
                const uint64_t ad = ad0 + static_cast<uint64_t>((it & 1) * (A_BYTES >> 4));
                const uint64_t bd = bd0 + static_cast<uint64_t>((it & 1) * (2048 >> 4));
                const uint32_t d = tmem + static_cast<uint32_t>(((it * 4) & (n_acc - 1)) * n_tok);
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    mma_i8(d + static_cast<uint32_t>(k * n_tok), ad + 2 * k, bd + 2 * k, idesc, it > 0 ? 1u : 0u);
                mma_commit(&bar);
            }
        } else {
            const uint32_t a0 = smem_addr(sa), b0 = smem_addr(sb);
            int j = 0, c = 0;
            for (int it = 0; it < iters; ++it) {
                for (int k = 0; k < 4; ++k, ++j) {
                    const uint64_t ad = smem_desc_k_sw128(a0 + (it & 1) * A_BYTES + k * 32);
                    const uint64_t bd = smem_desc_k_sw128(b0 + (it & 1) * 2048 + k * 32);
                    mma_i8(tmem + static_cast<uint32_t>((j % n_acc) * n_tok), ad, bd, idesc, j >= n_acc ? 1u : 0u);
                    if (++c == per_commit) {
                        c = 0;
                        mma_commit(&bar);
                    }
                }
            }
        }
        mma_commit(&bar);
        if (blockIdx.x == 0) cycles[0] = static_cast<unsigned long long>(iters);  // wall time is taken on the host
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

}  // namespace peak
}  // namespace i8mm

extern "C" int i8mm_debug_mma_small(int iters, int n_tok, int n_acc, int per_commit, unsigned long long* cycles,
                                    void* stream) {
    using namespace i8mm::peak;
    const size_t smem = 1024 + STAGES * (A_BYTES + 256 * 128);
    cudaFuncSetAttribute(mma_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    mma_small_kernel<<<i8mm::num_sms(), 128, smem, static_cast<cudaStream_t>(stream)>>>(iters, n_tok, n_acc,
                                                                                         per_commit, cycles);
    return cudaGetLastError() == cudaSuccess ? I8MM_OK : I8MM_ERR_CUDA;
}

extern "C" int i8mm_peak_mma_launch(int cg, int iters, void* stream) {
    if ((cg != 1 && cg != 2) || iters <= 0) return I8MM_ERR_ARGUMENT;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const cudaError_t e = cg == 2 ? i8mm::peak::launch<2>(iters, st) : i8mm::peak::launch<1>(iters, st);
    return e == cudaSuccess ? I8MM_OK : I8MM_ERR_CUDA;
}

extern "C" double i8mm_peak_mma_ops(int cg, int iters) {
    if (cg != 1 && cg != 2) return 0.0;
    const double units = static_cast<double>(i8mm::num_sms() / cg);  // CTAs or CTA pairs
    const double per_mma = 2.0 * (128.0 * cg) * 256.0 * 32.0;
    return units * per_mma * 4.0 * i8mm::peak::STAGES * static_cast<double>(iters);
}
