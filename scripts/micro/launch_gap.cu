#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(unsigned long long* t, int which, int mode) {
  extern __shared__ __align__(1024) char sm[];
  __shared__ uint32_t slot;
  if (threadIdx.x == 0) { unsigned long long g; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g)); atomicMin(&t[2*which], g); }
  if (mode & 1) { asm volatile("griddepcontrol.wait;" ::: "memory"); asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
  if ((mode & 2) && threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(sa(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (mode & 4) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  unsigned long long g0; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  while (true) { unsigned long long g; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g)); if (g - g0 > 10000) break; }
  sm[threadIdx.x] = 1;
  __syncthreads();
  if ((mode & 2) && threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(slot) : "memory");
  if (mode & 4) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (threadIdx.x == 0) { unsigned long long g; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g)); atomicMax(&t[2*which+1], g); }
}
int main(int argc, char** argv) {
  const int grid = argc > 1 ? atoi(argv[1]) : 120, smem_kb = argc > 2 ? atoi(argv[2]) : 200;
  unsigned long long* t; cudaMalloc(&t, 64*8);
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_kb*1024) != cudaSuccess) { printf("attr failed\n"); return 1; }
  for (int mode = 0; mode < 8; ++mode) {
    cudaStream_t st; cudaStreamCreate(&st);
    cudaGraph_t g; cudaGraphExec_t ge;
    unsigned long long init[16]; for (int i = 0; i < 16; ++i) init[i] = (i % 2 == 0) ? ~0ull : 0ull;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
    for (int w = 0; w < 6; ++w) {
      cudaLaunchConfig_t cfg{}; cfg.gridDim = dim3(grid); cfg.blockDim = dim3(256); cfg.dynamicSmemBytes = smem_kb*1024; cfg.stream = st;
      cudaLaunchAttribute at[2];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization; at[0].val.programmaticStreamSerializationAllowed = 1;
      at[1].id = cudaLaunchAttributeClusterDimension; at[1].val.clusterDim.x = 8; at[1].val.clusterDim.y = 1; at[1].val.clusterDim.z = 1;
      cfg.attrs = at; cfg.numAttrs = 2;
      cudaLaunchKernelEx(&cfg, k, t, w, mode);
    }
    cudaStreamEndCapture(st, &g);
    if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) { printf("instantiate failed: %s\n", cudaGetErrorString(cudaGetLastError())); return 1; }
    for (int r = 0; r < 3; ++r) { cudaMemcpy(t, init, sizeof(init), cudaMemcpyHostToDevice); cudaGraphLaunch(ge, st); cudaStreamSynchronize(st); }
    unsigned long long h[16]; cudaMemcpy(h, t, sizeof(h), cudaMemcpyDeviceToHost);
    printf("mode %d (pdl %d tmem %d clsync %d): gaps us:", mode, mode&1, (mode>>1)&1, (mode>>2)&1);
    for (int w = 1; w < 6; ++w) printf(" %.2f", (double)((long long)h[2*w] - (long long)h[2*w-1]) / 1e3);
    printf("  err=%s\n", cudaGetErrorString(cudaGetLastError()));
  }
}
