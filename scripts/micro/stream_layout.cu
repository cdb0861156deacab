// Microbenchmark (dev tool): HBM read bandwidth of a 128-row x 128-byte block
// walk over a K-major int8 weight (rows ldq bytes apart) vs the same blocks
// stored contiguously (16 KB each). One CTA per SM, 8 warps, 16-byte loads.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void walk(const uint4* __restrict__ w, int64_t ntiles, int64_t nkb, int64_t ldq, int tiled,
                     unsigned long long* sink) {
    const int64_t total = ntiles * nkb;
    const int64_t G = gridDim.x;
    const int64_t u0 = total * blockIdx.x / G, u1 = total * (blockIdx.x + 1) / G;
    uint32_t acc = 0;
    for (int64_t u = u0; u < u1; ++u) {
        const int64_t t = u / nkb, kb = u % nkb;
        // 128 rows x 8 uint4 = 1024 uint4 per block, 256 threads -> 4 each
        uint4 v[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int e = threadIdx.x + i * 256;
            const int r = e >> 3, c = e & 7;
            const int64_t off = tiled ? ((u * 128 + r) * 128 + c * 16) : ((t * 128 + r) * ldq + kb * 128 + c * 16);
            v[i] = __ldcs(reinterpret_cast<const uint4*>(reinterpret_cast<const char*>(w) + off));
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) acc ^= v[i].x ^ v[i].y ^ v[i].z ^ v[i].w;
    }
    if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

int main() {
    const int64_t shapes[3][2] = {{5120, 5120}, {5120, 20480}, {20480, 5120}};  // K, N
    unsigned long long* sink;
    cudaMalloc(&sink, 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (auto& s : shapes) {
        const int64_t K = s[0], N = s[1], ldq = K, nt = N / 128, nkb = K / 128;
        const size_t bytes = static_cast<size_t>(N) * K;
        void* w;
        cudaMalloc(&w, bytes);
        cudaMemset(w, 1, bytes);
        void* fl;
        cudaMalloc(&fl, 256 << 20);
        for (int tiled = 0; tiled < 2; ++tiled) {
            for (int blocks_per_sm = 1; blocks_per_sm <= 4; blocks_per_sm *= 2) {
                cudaEvent_t a, b;
                cudaEventCreate(&a);
                cudaEventCreate(&b);
                float best = 1e9;
                for (int it = 0; it < 10; ++it) {
                    cudaMemsetAsync(fl, it, 256 << 20);
                    cudaEventRecord(a);
                    walk<<<sms * blocks_per_sm, 256>>>(reinterpret_cast<const uint4*>(w), nt, nkb, ldq, tiled, sink);
                    cudaEventRecord(b);
                    cudaEventSynchronize(b);
                    float ms;
                    cudaEventElapsedTime(&ms, a, b);
                    if (ms < best) best = ms;
                }
                printf("K=%lld N=%lld %s blocks/SM=%d: %.1f us  %.0f GB/s\n", (long long)K, (long long)N,
                       tiled ? "tiled " : "strided", blocks_per_sm, best * 1e3, bytes / (best * 1e-3) / 1e9);
            }
        }
        cudaFree(w);
        cudaFree(fl);
    }
    return 0;
}
