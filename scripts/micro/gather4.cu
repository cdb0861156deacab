// Dev micro-test: semantics of TMA tile::gather4 (sm_100a) with SWIZZLE_128B.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -o gather4 gather4.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cuda.h>
#include <cuda_runtime.h>

__global__ void k(const __grid_constant__ CUtensorMap m, int c0, int r0, int r1, int r2, int r3, uint8_t* out, int off) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar;
    uint8_t* buf = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
    uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(buf + off));
    uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(&bar));
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
        asm volatile("fence.mbarrier_init.release.cluster;");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(512));
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
            :: "r"(d), "l"(reinterpret_cast<uint64_t>(&m)), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(b) : "memory");
        uint32_t ok = 0;
        while (!ok) {
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                         : "=r"(ok) : "r"(b) : "memory");
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 512; i += blockDim.x) out[i] = buf[off + i];
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const int R = 64, C = 256;
    uint8_t h[R * C];
    for (int r = 0; r < R; ++r)
        for (int c = 0; c < C; ++c) h[r * C + c] = static_cast<uint8_t>((r * 3 + c / 16) & 0xFF);
    uint8_t *dq, *dout;
    cudaMalloc(&dq, R * C);
    cudaMalloc(&dout, 512);
    cudaMemcpy(dq, h, R * C, cudaMemcpyHostToDevice);
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    EncFn enc = reinterpret_cast<EncFn>(fp);
    const int rows_idx[4] = {5, 17, 2, 40};
    for (int off : {0, 512}) for (int bh : {1}) {
        CUtensorMap m;
        cuuint64_t dims[2] = {static_cast<cuuint64_t>(C), static_cast<cuuint64_t>(R)};
        cuuint64_t strides[1] = {static_cast<cuuint64_t>(C)};
        cuuint32_t box[2] = {128, static_cast<cuuint32_t>(bh)};
        cuuint32_t es[2] = {1, 1};
        CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, dq, dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) { printf("box h=%d: encode failed %d\n", bh, (int)r); continue; }
        cudaMemset(dout, 0xEE, 512);
        k<<<1, 128, 4096>>>(m, 128, rows_idx[0], rows_idx[1], rows_idx[2], rows_idx[3], dout, off);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("box h=%d: kernel error %s\n", bh, cudaGetErrorString(e)); cudaGetLastError(); return 1; }
        uint8_t o[512];
        cudaMemcpy(o, dout, 512, cudaMemcpyDeviceToHost);
        int bad_plain = 0, bad_swz = 0;
        for (int i = 0; i < 4; ++i)
            for (int cch = 0; cch < 8; ++cch) {
                const uint8_t want = static_cast<uint8_t>((rows_idx[i] * 3 + (128 + cch * 16) / 16) & 0xFF);
                if (o[i * 128 + cch * 16] != want) ++bad_plain;
                if (o[i * 128 + ((cch ^ (i + off / 128)) * 16)] != want) ++bad_swz;
            }
        printf("off=%d box h=%d: mismatches plain=%d swizzle128(row i)=%d  first bytes: %d %d %d %d\n", off, bh, bad_plain, bad_swz,
               o[0], o[16], o[128], o[144]);
    }
    return 0;
}
