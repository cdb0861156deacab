// Microbenchmark (dev tool): cost of one grid-wide barrier on B200 with one
// CTA per SM (cooperative launch): cooperative_groups grid.sync() vs a
// counter/generation barrier (words on separate 128-byte lines).
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
namespace cg = cooperative_groups;

struct alignas(128) Line { unsigned v; unsigned pad[31]; };

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

template <int MODE>
__global__ void bench(Line* st, int iters, unsigned long long* out) {
    cg::grid_group grid = cg::this_grid();
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (MODE == 0) {
            grid.sync();
        } else {
            __syncthreads();
            if (threadIdx.x == 0) {
                const unsigned g = ld_acq(&st[1].v);
                unsigned old;
                if (MODE == 1) {
                    __threadfence();
                    old = atomicAdd(&st[0].v, 1u);
                } else {
                    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(&st[0].v) : "memory");
                }
                if (old == gridDim.x - 1) {
                    st[0].v = 0;
                    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(&st[1].v), "r"(g + 1) : "memory");
                } else {
                    while (ld_acq(&st[1].v) == g) {
                        if (MODE == 3) __nanosleep(32);
                    }
                }
            }
            __syncthreads();
        }
    }
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) *out = t1 - t0;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    Line* st;
    cudaMalloc(&st, sizeof(Line) * 4);
    cudaMemset(st, 0, sizeof(Line) * 4);
    unsigned long long* out;
    cudaMalloc(&out, 8);
    int iters = 200;
    const char* names[4] = {"cg grid.sync", "fence+atomicAdd / release gen", "atom.acq_rel / release gen", "acq_rel + nanosleep"};
    for (int mode = 0; mode < 4; ++mode) {
        for (int threads : {256, 512}) {
            void* args[] = {&st, &iters, &out};
            void* fn = mode == 0 ? (void*)bench<0> : mode == 1 ? (void*)bench<1> : mode == 2 ? (void*)bench<2> : (void*)bench<3>;
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaLaunchCooperativeKernel(fn, sms, threads, args, 0, 0);  // warm
            cudaEventRecord(a);
            cudaLaunchCooperativeKernel(fn, sms, threads, args, 0, 0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            cudaError_t e = cudaGetLastError();
            printf("%-34s threads=%d: %.2f us per barrier (%s)\n", names[mode], threads, ms * 1e3 / iters,
                   cudaGetErrorString(e));
        }
    }
    return 0;
}
