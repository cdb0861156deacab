// Which L2 partition (die) serves each SM (dev micro): one CTA per SM times an
// L2-hit load of each of NL lines (4 KB apart) with clock64, after a warm-up
// read by the same SM. Lines homed in the SM's own die's L2 answer faster; the
// latency matrix [smid][line] is written to lat.bin for scripts/l2_die.py.
//   ./l2_die [lines]
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

__global__ void probe(const uint32_t* __restrict__ buf, int nl, int stride_words, uint32_t* lat, int* smid_of) {
    extern __shared__ uint8_t pad[];  // forces one CTA per SM
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    if (threadIdx.x != 0) return;
    smid_of[blockIdx.x] = static_cast<int>(smid);
    pad[0] = 0;
    uint32_t sink = 0;
    for (int i = 0; i < nl; ++i) {
        const uint32_t* p = buf + static_cast<int64_t>(i) * stride_words;
        uint32_t v;
        asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");  // warm (L2)
        sink += v;
        uint32_t best = 0xFFFFFFFFu;
        for (int r = 0; r < 4; ++r) {
            // 8 dependent loads of the same line (its word is 0: the next address is
            // p + value), timed together
            long long t0, t1;
            uint32_t off = sink & 0u;
            asm volatile("mov.u64 %0, %%clock64;" : "=l"(t0)::"memory");
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p + off) : "memory");
                off = v;
            }
            asm volatile("add.u32 %0, %0, 0;" : "+r"(off)::"memory");
            asm volatile("mov.u64 %0, %%clock64;" : "=l"(t1) : "r"(off) : "memory");
            sink += off;
            const uint32_t d = static_cast<uint32_t>(t1 - t0) / 8u;
            best = d < best ? d : best;
        }
        lat[static_cast<int64_t>(smid) * nl + i] = best;
    }
    if (sink == 0x12345678u) lat[0] = sink;
}

int main(int argc, char** argv) {
    const int nl = argc > 1 ? atoi(argv[1]) : 128;
    const int stride_words = 1024;  // 4 KB
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t* buf;
    cudaMalloc(&buf, static_cast<size_t>(nl) * stride_words * 4);
    cudaMemset(buf, 0, static_cast<size_t>(nl) * stride_words * 4);
    uint32_t* lat;
    int* smid_of;
    cudaMalloc(&lat, static_cast<size_t>(256) * nl * 4);
    cudaMemset(lat, 0, static_cast<size_t>(256) * nl * 4);
    cudaMalloc(&smid_of, 256 * 4);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    // one CTA at a time per launch would serialise; all SMs at once is fine: the
    // loads are single-thread and far apart in time from other SMs' traffic
    probe<<<sms, 32, 200 * 1024>>>(buf, nl, stride_words, lat, smid_of);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(e));
        return 1;
    }
    uint32_t* h = static_cast<uint32_t*>(malloc(static_cast<size_t>(256) * nl * 4));
    cudaMemcpy(h, lat, static_cast<size_t>(256) * nl * 4, cudaMemcpyDeviceToHost);
    FILE* f = fopen(argc > 2 ? argv[2] : "gpurun_out/lat.bin", "wb");
    fwrite(&nl, 4, 1, f);
    fwrite(&sms, 4, 1, f);
    fwrite(h, 4, static_cast<size_t>(256) * nl, f);
    fclose(f);
    printf("ok sms=%d lines=%d\n", sms, nl);
    return 0;
}
