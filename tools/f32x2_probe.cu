// Probe (run under gpurun): do the packed fp32 operations (fma/mul/add .rn.f32x2,
// FFMA2/FMUL2/FADD2 on sm_100a) give the same bits as the scalar .rn.f32 ones?
#include <cstdio>
#include <cstdint>
#include <cstring>
__global__ void k(const float* a, const float* b, const float* c, unsigned* bad, int n) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (2 * t + 1 >= n) return;
    float a0 = a[2 * t], a1 = a[2 * t + 1], b0 = b[2 * t], b1 = b[2 * t + 1], c0 = c[2 * t], c1 = c[2 * t + 1];
    float2 f = __ffma2_rn(make_float2(a0, a1), make_float2(b0, b1), make_float2(c0, c1));
    float2 m = __fmul2_rn(make_float2(a0, a1), make_float2(b0, b1));
    float2 s = __fadd2_rn(make_float2(a0, a1), make_float2(c0, c1));
    if (f.x != __fmaf_rn(a0, b0, c0) || f.y != __fmaf_rn(a1, b1, c1)) atomicAdd(&bad[0], 1u);
    if (m.x != __fmul_rn(a0, b0) || m.y != __fmul_rn(a1, b1)) atomicAdd(&bad[1], 1u);
    if (s.x != __fadd_rn(a0, c0) || s.y != __fadd_rn(a1, c1)) atomicAdd(&bad[2], 1u);
}
int main() {
    const int n = 1 << 24;
    float *a, *b, *c; unsigned* bad;
    cudaMallocManaged(&a, n * 4); cudaMallocManaged(&b, n * 4); cudaMallocManaged(&c, n * 4); cudaMallocManaged(&bad, 12);
    uint32_t s = 12345;
    auto rnd = [&]() { s = s * 1664525u + 1013904223u; return (s >> 8) * (1.0f / 16777216.0f); };
    for (int i = 0; i < n; ++i) { a[i] = 0.9f + 0.2f * rnd(); b[i] = 0.01f + 0.05f * rnd(); c[i] = (rnd() - 0.5f) * 0.1f; }
    memset(bad, 0, 12);
    k<<<n / 2 / 256, 256>>>(a, b, c, bad, n);
    cudaDeviceSynchronize();
    printf("mismatches over %d pairs: fma %u  mul %u  add %u\n", n / 2, bad[0], bad[1], bad[2]);
    return 0;
}
