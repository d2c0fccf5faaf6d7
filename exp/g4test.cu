// tile::gather4 probe: which boxDim[1] does cuTensorMapEncodeTiled accept for a
// 2-D gather4 load, and does the load land as 4 packed rows?
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *, const cuuint64_t *,
                             const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
__global__ void k(const __grid_constant__ CUtensorMap tm, double *out, int C, int r0, int r1, int r2, int r3) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm);
    double *buf = reinterpret_cast<double *>(sm + 128);
    uint32_t b = (uint32_t)__cvta_generic_to_shared(bar), d = (uint32_t)__cvta_generic_to_shared(buf);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
        asm volatile("fence.mbarrier_init.release.cluster;");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(4 * C * 8));
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                     ::"r"(d), "l"(&tm), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(b) : "memory");
        uint32_t ok = 0;
        while (!ok) asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p;}" : "=r"(ok) : "r"(b));
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 4 * C; i += blockDim.x) out[i] = buf[i];
}
int main() {
    EncodeFn enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
    if (!enc) { printf("no encode\n"); return 1; }
    const int C = 52, R = 1000;
    std::vector<double> h((size_t)C * R);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (double)i;
    double *dg, *dout;
    cudaMalloc(&dg, h.size() * 8);
    cudaMalloc(&dout, 4 * C * 8);
    cudaMemcpy(dg, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 + 4 * C * 8);
    for (cuuint32_t bx1 : {1u, 4u}) {
        CUtensorMap tm;
        cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)R};
        cuuint64_t strides[1] = {(cuuint64_t)C * 8};
        cuuint32_t box[2] = {(cuuint32_t)C, bx1}, es[2] = {1, 1};
        CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, dg, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        printf("box {%d,%u}: encode %d\n", C, bx1, (int)r);
        if (r != CUDA_SUCCESS) continue;
        cudaMemset(dout, 0, 4 * C * 8);
        k<<<1, 128, 128 + 4 * C * 8>>>(tm, dout, C, 7, 3, 999, 500);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<double> o(4 * C);
        cudaMemcpy(o.data(), dout, o.size() * 8, cudaMemcpyDeviceToHost);
        int rows[4] = {7, 3, 999, 500}, bad = 0;
        for (int rr = 0; rr < 4; ++rr)
            for (int c = 0; c < C; ++c) bad += o[rr * C + c] != (double)(rows[rr] * C + c);
        printf("  run %s, mismatches %d (o[0]=%g o[52]=%g)\n", cudaGetErrorString(e), bad, o[0], o[C]);
        if (e != cudaSuccess) return 0;
    }
    return 0;
}
