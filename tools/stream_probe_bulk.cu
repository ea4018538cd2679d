// Ceiling probe, part 2 (not part of the library): does the way the VTI step's
// DRAM mix is moved change its ceiling? 7 float streams read, 2 written,
// N floats each, three forms:
//   ldg : plain float4 loads and stores (as tools/stream_probe.cu)
//   tma : 1-D cp.async.bulk loads into a 3-stage shared-memory ring (mbarriers), float4 stores
//   tma+bst : the same loads, results staged in shared memory and written with
//             cp.async.bulk shared -> global (bulk-group completion)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/spb tools/stream_probe_bulk.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int CH = 2048;   // floats per stream per chunk (8 KB)
constexpr int ST = 3;      // ring stages
constexpr int NT = 256;    // threads

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t c)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t *b, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t ph)
{
    asm volatile(
        "{\n .reg .pred P;\n W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n @!P bra W;\n}\n" ::"r"(sa(b)),
        "r"(ph)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *b)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(dst)),
                 "l"(src), "r"(bytes), "r"(sa(b))
                 : "memory");
}
__device__ __forceinline__ void bulk_s2g(void *dst, const void *src, uint32_t bytes)
{
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(sa(src)), "r"(bytes)
                 : "memory");
}

__global__ void mix_ldg(const float4 *__restrict__ a, const float4 *__restrict__ b, const float4 *__restrict__ c,
                        const float4 *__restrict__ d, const float4 *__restrict__ e, const float4 *__restrict__ f,
                        const float4 *__restrict__ g, float4 *__restrict__ o1, float4 *__restrict__ o2, size_t n4)
{
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
        float4 x = a[i], y = b[i], z = c[i], w = d[i], u = e[i], v = f[i], t = g[i];
        o1[i] = make_float4(x.x + y.x + z.x + w.x, x.y + y.y + z.y + w.y, x.z + y.z + z.z + w.z, x.w + y.w + z.w + w.w);
        o2[i] = make_float4(u.x + v.x + t.x, u.y + v.y + t.y, u.z + v.z + t.z, u.w + v.w + t.w);
    }
}

struct Streams {
    const float *in[7];
    float *out[2];
};

template <bool BST>
__global__ void __launch_bounds__(NT, 1) mix_tma(const __grid_constant__ Streams S, size_t n)
{
    extern __shared__ __align__(128) uint8_t smem[];
    float *ring = reinterpret_cast<float *>(smem);                   // [ST][7][CH]
    float *outb = ring + ST * 7 * CH;                                // [2][2][CH]
    uint64_t *full = reinterpret_cast<uint64_t *>(outb + 4 * CH);   // [ST]
    const size_t nch = n / CH;
    if (threadIdx.x == 0) {
        for (int s = 0; s < ST; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](size_t ch, int s) {
        mbar_expect(&full[s], 7 * CH * 4);
        for (int k = 0; k < 7; ++k) bulk_g2s(ring + (s * 7 + k) * CH, S.in[k] + ch * CH, CH * 4, &full[s]);
    };
    if (threadIdx.x == 0)
        for (int s = 0; s < ST; ++s)
            if (blockIdx.x + (size_t)s * gridDim.x < nch) issue(blockIdx.x + (size_t)s * gridDim.x, s);
    uint32_t phase = 0;
    int s = 0, t = 0;
    for (size_t ch = blockIdx.x; ch < nch; ch += gridDim.x, ++t) {
        mbar_wait(&full[s], phase);
        const float4 *r = reinterpret_cast<const float4 *>(ring + s * 7 * CH);
        float *ob = outb + (t & 1) * 2 * CH;
        if (BST && t >= 2 && threadIdx.x == 0)   // the store issued from this buffer two chunks ago has read it
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        if (BST) __syncthreads();
        for (int i = threadIdx.x; i < CH / 4; i += NT) {
            const float4 x = r[i], y = r[CH / 4 + i], z = r[2 * CH / 4 + i], w = r[3 * CH / 4 + i];
            const float4 u = r[4 * CH / 4 + i], v = r[5 * CH / 4 + i], q = r[6 * CH / 4 + i];
            const float4 A = make_float4(x.x + y.x + z.x + w.x, x.y + y.y + z.y + w.y, x.z + y.z + z.z + w.z,
                                         x.w + y.w + z.w + w.w);
            const float4 B = make_float4(u.x + v.x + q.x, u.y + v.y + q.y, u.z + v.z + q.z, u.w + v.w + q.w);
            if (BST) {
                reinterpret_cast<float4 *>(ob)[i] = A;
                reinterpret_cast<float4 *>(ob + CH)[i] = B;
            } else {
                reinterpret_cast<float4 *>(S.out[0] + ch * CH)[i] = A;
                reinterpret_cast<float4 *>(S.out[1] + ch * CH)[i] = B;
            }
        }
        if (BST) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();   // stage s consumed (and, BST, the out tile written)
        if (threadIdx.x == 0) {
            if (BST) {
                bulk_s2g(S.out[0] + ch * CH, ob, CH * 4);
                bulk_s2g(S.out[1] + ch * CH, ob + CH, CH * 4);
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            const size_t nxt = ch + (size_t)ST * gridDim.x;
            if (nxt < nch) issue(nxt, s);
        }
        if (++s == ST) {
            s = 0;
            phase ^= 1;
        }
    }
    if (BST && threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char **argv)
{
    const size_t n = argc > 1 ? (size_t)atoll(argv[1]) : 512ull * 512 * 512;
    printf("points per stream: %zu (%.1f GB over 9 streams)\n", n, 36.0 * n / 1e9);
    float *p[9];
    for (int i = 0; i < 9; ++i) {
        cudaMalloc(&p[i], n * 4);
        cudaMemset(p[i], 0, n * 4);
    }
    Streams S;
    for (int k = 0; k < 7; ++k) S.in[k] = p[k];
    S.out[0] = p[7];
    S.out[1] = p[8];
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int smem = (ST * 7 * CH + 4 * CH) * 4 + ST * 8;
    cudaFuncSetAttribute(mix_tma<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(mix_tma<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t t0, t1;
    cudaEventCreate(&t0);
    cudaEventCreate(&t1);
    const int reps = 20;
    auto time = [&](const char *name, int grid, auto launch) {
        for (int w = 0; w < 3; ++w) launch();
        cudaEventRecord(t0);
        for (int r = 0; r < reps; ++r) launch();
        cudaEventRecord(t1);
        cudaEventSynchronize(t1);
        float ms;
        cudaEventElapsedTime(&ms, t0, t1);
        cudaError_t e = cudaGetLastError();
        printf("%-8s grid %4d: %.3f ms/iter, %.3f TB/s (36 B/pt), %.1f Gpts/s %s\n", name, grid, ms / reps,
               36.0 * n * reps / (ms * 1e-3) / 1e12, n * reps / (ms * 1e-3) / 1e9,
               e == cudaSuccess ? "" : cudaGetErrorString(e));
    };
    for (int g : {2 * sms, 4 * sms})
        time("ldg", g, [&] {
            mix_ldg<<<g, 256>>>((float4 *)p[0], (float4 *)p[1], (float4 *)p[2], (float4 *)p[3], (float4 *)p[4],
                                (float4 *)p[5], (float4 *)p[6], (float4 *)p[7], (float4 *)p[8], n / 4);
        });
    for (int g : {110, 128, sms})
        time("tma", g, [&] { mix_tma<false><<<g, NT, smem>>>(S, n); });
    for (int g : {110, 128, sms})
        time("tma+bst", g, [&] { mix_tma<true><<<g, NT, smem>>>(S, n); });
    return 0;
}
