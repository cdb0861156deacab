// Does __syncthreads() still wait for every warp after griddepcontrol.launch_dependents
// (PREEXIT)? Warp 0 spins ~10 us before the barrier; the other warps stamp the time
// they leave it. mode bit 0: trigger before the barrier, bit 1: launch with the PDL
// attribute, bit 2: 2-CTA cluster, bit 3: named barrier (bar.sync 1, 256) instead.
#include <cuda_runtime.h>

#include <cstdio>

__device__ __forceinline__ unsigned long long gt() {
    unsigned long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    return g;
}
__global__ void k(unsigned long long* out, int mode) {
    if (mode & 1) {
        asm volatile("griddepcontrol.wait;" ::: "memory");
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    }
    const unsigned long long t0 = gt();
    if ((mode & 16) ? threadIdx.x == 0 : threadIdx.x < 32) {  // bit 4: lane 0 alone spins
        while (gt() - t0 < 10000) {
        }
    }
    if (mode & 8)
        asm volatile("bar.sync 1, 256;" ::: "memory");
    else
        __syncthreads();
    if (threadIdx.x == 64) out[blockIdx.x] = gt() - t0;
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 64 * 8);
    for (int mode : {0, 3, 16, 19, 23, 27}) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(8);
        cfg.blockDim = dim3(256);
        cudaLaunchAttribute at[2];
        int na = 0;
        if (mode & 2) {
            at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[na].val.programmaticStreamSerializationAllowed = 1;
            ++na;
        }
        if (mode & 4) {
            at[na].id = cudaLaunchAttributeClusterDimension;
            at[na].val.clusterDim.x = 2;
            at[na].val.clusterDim.y = 1;
            at[na].val.clusterDim.z = 1;
            ++na;
        }
        cfg.attrs = at;
        cfg.numAttrs = na;
        cudaLaunchKernelEx(&cfg, k, d, mode);
        cudaDeviceSynchronize();
        unsigned long long h[8];
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        printf("mode %2d (trigger %d pdl %d cluster %d named %d lane0-only %d): warp 2 left the barrier after", mode, mode & 1,
               (mode >> 1) & 1, (mode >> 2) & 1, (mode >> 3) & 1, (mode >> 4) & 1);
        for (int i = 0; i < 8; ++i) printf(" %.1f", h[i] / 1e3);
        printf(" us  (%s)\n", cudaGetErrorString(cudaGetLastError()));
    }
}
