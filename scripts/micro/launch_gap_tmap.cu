// Launch gap between consecutive graph-captured, PDL-chained cluster kernels whose
// TMA descriptor is (a) a __grid_constant__ kernel parameter or (b) a 128-byte
// CUtensorMap in global memory written once before the graph (dev micro).
//   ./launch_gap_tmap [grid] [smem_kb]
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned long long gt() {
    unsigned long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    return g;
}
__device__ __forceinline__ void tma_load(const void* map, uint64_t* bar, void* dst, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            sa(dst)),
        "l"(map), "r"(sa(bar)), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void body(const void* map, unsigned long long* t, int which, int mode) {
    extern __shared__ __align__(1024) char sm[];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) atomicMin(&t[2 * which], gt());
    if (threadIdx.x == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (mode & 1) {
        asm volatile("griddepcontrol.wait;" ::: "memory");
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
        if (threadIdx.x == 0) atomicMax(&t[32 + which], gt());
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(16384) : "memory");
        tma_load(map, &bar, sm, 0, (blockIdx.x % 64) * 128);
        uint32_t ok = 0;
        while (!ok)
            asm volatile(
                "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                : "=r"(ok)
                : "r"(sa(&bar))
                : "memory");
    }
    __syncthreads();
    const unsigned long long g0 = gt();
    while (gt() - g0 < 10000) {
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (threadIdx.x == 0) atomicMax(&t[2 * which + 1], gt());
}
__global__ void k_param(const __grid_constant__ CUtensorMap tm, unsigned long long* t, int which, int mode) {
    body(&tm, t, which, mode);
}
__global__ void k_global(const CUtensorMap* tm, unsigned long long* t, int which, int mode) {
    body(tm, t, which, mode);
}
struct Big { unsigned long long v[150]; };
__global__ void k_big(const __grid_constant__ CUtensorMap tm, const Big b, unsigned long long* t, int which, int mode) {
    if (b.v[threadIdx.x & 127] == 12345ull) t[40] = 1;
    body(&tm, t, which, mode);
}

typedef CUresult (*encode_fn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
    const int grid = argc > 1 ? atoi(argv[1]) : 120, smem_kb = argc > 2 ? atoi(argv[2]) : 200;
    void* w;
    cudaMalloc(&w, 8192 * 128);
    encode_fn enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    CUtensorMap tm;
    cuuint64_t dims[2] = {128, 8192}, strides[1] = {128};
    cuuint32_t box[2] = {128, 128}, es[2] = {1, 1};
    if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, w, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != 0) {
        printf("encode failed\n");
        return 1;
    }
    CUtensorMap* dtm;
    cudaMalloc(&dtm, sizeof(CUtensorMap));
    cudaMemcpy(dtm, &tm, sizeof(tm), cudaMemcpyHostToDevice);
    unsigned long long* t;
    cudaMalloc(&t, 64 * 8);
    for (auto f : {(const void*)k_param, (const void*)k_global, (const void*)k_big})
        if (cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_kb * 1024) != cudaSuccess) {
            printf("attr failed\n");
            return 1;
        }
    Big big{};
    for (int variant = 0; variant < 3; ++variant)
        for (int mode = 0; mode < 2; ++mode) {
            cudaStream_t st;
            cudaStreamCreate(&st);
            cudaGraph_t g;
            cudaGraphExec_t ge;
            unsigned long long init[16];
            for (int i = 0; i < 16; ++i) init[i] = (i % 2 == 0) ? ~0ull : 0ull;
            cudaMemset(t + 32, 0, 8 * 8);
            cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
            for (int wi = 0; wi < 6; ++wi) {
                cudaLaunchConfig_t cfg{};
                cfg.gridDim = dim3(grid);
                cfg.blockDim = dim3(256);
                cfg.dynamicSmemBytes = smem_kb * 1024;
                cfg.stream = st;
                cudaLaunchAttribute at[2];
                at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = 8;
                at[0].val.clusterDim.y = 1;
                at[0].val.clusterDim.z = 1;
                at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                at[1].val.programmaticStreamSerializationAllowed = 1;
                cfg.attrs = at;
                cfg.numAttrs = mode ? 2 : 1;
                if (variant == 0)
                    cudaLaunchKernelEx(&cfg, k_param, tm, t, wi, mode);
                else if (variant == 1)
                    cudaLaunchKernelEx(&cfg, k_global, (const CUtensorMap*)dtm, t, wi, mode);
                else
                    cudaLaunchKernelEx(&cfg, k_big, tm, big, t, wi, mode);
            }
            cudaStreamEndCapture(st, &g);
            if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) {
                printf("instantiate failed\n");
                return 1;
            }
            for (int r = 0; r < 3; ++r) {
                cudaMemcpy(t, init, sizeof(init), cudaMemcpyHostToDevice);
                cudaGraphLaunch(ge, st);
                cudaStreamSynchronize(st);
            }
            unsigned long long h[16];
            cudaMemcpy(h, t, sizeof(h), cudaMemcpyDeviceToHost);
            printf("%s pdl %d: gaps us:", variant == 1 ? "global tmap" : variant == 2 ? "param+1.2KB" : "param tmap ", mode);
            for (int wi = 1; wi < 6; ++wi) printf(" %.2f", (double)((long long)h[2 * wi] - (long long)h[2 * wi - 1]) / 1e3);
            if (mode) {
                unsigned long long h2[8];
                cudaMemcpy(h2, t + 32, sizeof(h2), cudaMemcpyDeviceToHost);
                printf("  | wait released after prev end (max over CTAs) us:");
                for (int wi = 1; wi < 6; ++wi) printf(" %.2f", (double)((long long)h2[wi] - (long long)h[2 * wi - 1]) / 1e3);
            }
            printf("  err=%s\n", cudaGetErrorString(cudaGetLastError()));
        }
}
