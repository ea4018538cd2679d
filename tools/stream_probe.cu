// Ceiling probe for the VTI step's DRAM access mix (not part of the library):
// 7 float streams read, 2 written, N floats each, plain float4 grid-stride
// loops. Prints TB/s for several launch shapes; compare with the step kernel's
// ncu DRAM rate. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/sp tools/stream_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void mix(const float4 *__restrict__ a, const float4 *__restrict__ b, const float4 *__restrict__ c,
                    const float4 *__restrict__ d, const float4 *__restrict__ e, const float4 *__restrict__ f,
                    const float4 *__restrict__ g, float4 *__restrict__ o1, float4 *__restrict__ o2, size_t n4)
{
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
        float4 x = a[i], y = b[i], z = c[i], w = d[i], u = e[i], v = f[i], t = g[i];
        o1[i] = make_float4(x.x + y.x + z.x + w.x, x.y + y.y + z.y + w.y, x.z + y.z + z.z + w.z, x.w + y.w + z.w + w.w);
        o2[i] = make_float4(u.x + v.x + t.x, u.y + v.y + t.y, u.z + v.z + t.z, u.w + v.w + t.w);
    }
}

int main(int argc, char **argv)
{
    // points per stream: 512^3 (C2) by default, or argv[1] (e.g. 4294967296 for C4's 2048^2 x 1024)
    const size_t n = argc > 1 ? (size_t)atoll(argv[1]) : 512ull * 512 * 512, n4 = n / 4;
    printf("points per stream: %zu (%.1f GB over 9 streams)\n", n, 36.0 * n / 1e9);
    float4 *p[9];
    for (int i = 0; i < 9; ++i) {
        cudaMalloc(&p[i], n * 4);
        cudaMemset(p[i], 0, n * 4);
    }
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t t0, t1;
    cudaEventCreate(&t0);
    cudaEventCreate(&t1);
    const int shapes[][2] = {{1, 256}, {2, 256}, {4, 256}, {8, 256}, {2, 512}, {4, 512}, {1, 1024}, {2, 1024}};
    for (auto &sh : shapes) {
        const int grid = sms * sh[0], block = sh[1];
        for (int w = 0; w < 3; ++w) mix<<<grid, block>>>(p[0], p[1], p[2], p[3], p[4], p[5], p[6], p[7], p[8], n4);
        cudaEventRecord(t0);
        const int reps = n > (1ull << 30) ? 3 : 20;
        for (int r = 0; r < reps; ++r) mix<<<grid, block>>>(p[0], p[1], p[2], p[3], p[4], p[5], p[6], p[7], p[8], n4);
        cudaEventRecord(t1);
        cudaEventSynchronize(t1);
        float ms;
        cudaEventElapsedTime(&ms, t0, t1);
        const double tbs = 36.0 * n * reps / (ms * 1e-3) / 1e12;
        printf("grid %4d x %4d: %.3f ms/iter, %.3f TB/s (36 B/pt), %.1f Gpts/s\n", grid, block, ms / reps, tbs,
               n * reps / (ms * 1e-3) / 1e9);
    }
    return 0;
}
