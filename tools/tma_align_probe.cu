// tma_align_probe.cu -- does a TMA tensor load accept a shared-memory destination
// that is 16-byte but not 128-byte aligned?  argv[1] = destination offset in bytes.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tma_align_probe tools/tma_align_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ unsigned smem_u32(const void* p) { return unsigned(__cvta_generic_to_shared(p)); }

__global__ void probe(const __grid_constant__ CUtensorMap m, int c0, int c1, int c2, unsigned tx, double* out,
                      int n, unsigned* status, int off) {
    extern __shared__ __align__(128) unsigned char sm[];
    double* buf = reinterpret_cast<double*>(sm + off);
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(sm + 8192 * 8);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(1) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(tx)
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(buf)),
            "l"(reinterpret_cast<unsigned long long>(&m)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
            : "memory");
    }
    unsigned ok = 0;
    for (unsigned spin = 0; spin < (1u << 22) && !ok; ++spin) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(0)
            : "memory");
    }
    if (threadIdx.x == 0) *status = ok ? 1u : 2u;
    if (!ok) return;
    for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = buf[i];
}

int main(int argc, char** argv) {
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    EncodeFn enc = reinterpret_cast<EncodeFn>(fp);
    printf("encode fn %p q=%d\n", fp, int(q));
    const int nz = 40, nzp = 40, ny = 12, planes = 6;
    std::vector<double> h(size_t(planes) * ny * nzp);
    for (size_t i = 0; i < h.size(); ++i) h[i] = double(i) + 1;
    double *d, *out;
    unsigned* st;
    cudaMalloc(&d, h.size() * 8);
    cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaMalloc(&out, 8192 * 8);
    cudaMallocManaged(&st, 4);
    CUtensorMap m;
    const cuuint64_t dims[3] = {cuuint64_t(nz), cuuint64_t(ny), cuuint64_t(planes)};
    const cuuint64_t strides[2] = {cuuint64_t(nzp) * 8, cuuint64_t(nzp) * ny * 8};
    const int BW = 34, HY = 10;
    const cuuint32_t box[3] = {BW, HY, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode result %d\n", int(r));
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192 * 8 + 64);
    int cases[][3] = {{0, 0, 0}, {-2, -1, 2}, {-2, -2, 5}, {10, 5, 3}, {20, 8, 1}, {-1, 0, 0}};
    const int which = 1;
    const int off = argc > 1 ? atoi(argv[1]) : 0;
    printf("dst offset %d bytes\n", off);
    for (int ci = which; ci <= which; ++ci) {
        auto& c = cases[ci];
        *st = 0;
        probe<<<1, 128, 8192 * 8 + 64>>>(m, c[0], c[1], c[2], BW * HY * 8, out, BW * HY, st, off);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<double> o(BW * HY);
        cudaMemcpy(o.data(), out, o.size() * 8, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int a = 0; a < HY; ++a)
            for (int b = 0; b < BW; ++b) {
                int z = c[0] + b, y = c[1] + a, x = c[2];
                double want = (z >= 0 && z < nz && y >= 0 && y < ny) ? h[(size_t(x) * ny + y) * nzp + z] : 0.0;
                if (o[a * BW + b] != want) ++bad;
            }
        printf("case (%d,%d,%d): err=%s status=%u mismatches=%d\n", c[0], c[1], c[2], cudaGetErrorString(e), *st,
               bad);
    }
    return 0;
}
