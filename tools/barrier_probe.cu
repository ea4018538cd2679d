// barrier_probe.cu -- latency of in-kernel step synchronisation on B200 (measurement tool for the
// small-grid multi-step kernel): a cooperative grid of G CTAs runs N rounds of
//   (a) a grid barrier: every CTA arrives on one counter (atomicAdd after __syncthreads), thread
//       0 polls it with ld.acquire.gpu until it reaches G * (round + 1);
//   (b) neighbour flags: CTA b publishes round r (st.release.gpu) and waits for CTAs b-1 and b+1
//       (the shape of the multi-step kernel's partner waits, with 2 partners instead of 26);
//   (c) the same as (a) with relaxed polling and one acquire fence.
// Prints microseconds per round. nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bp barrier_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void grid_barrier(unsigned int *ctr, int rounds, int relaxed)
{
    for (int r = 0; r < rounds; ++r) {
        __syncthreads();
        if (threadIdx.x == 0) {
            atomicAdd(ctr, 1u);
            const unsigned int want = gridDim.x * (unsigned int)(r + 1);
            unsigned int v;
            if (relaxed) {
                do {
                    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
                } while (v < want);
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
            } else {
                do {
                    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
                } while (v < want);
            }
        }
        __syncthreads();
    }
}

__global__ void neighbour_flags(unsigned int *flags, int rounds)
{
    const int b = blockIdx.x, G = gridDim.x;
    for (int r = 0; r < rounds; ++r) {
        __syncthreads();
        if (threadIdx.x == 0)
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags + b), "r"((unsigned int)r + 1) : "memory");
        if (threadIdx.x == 1 || threadIdx.x == 2) {
            const int nb = threadIdx.x == 1 ? (b + G - 1) % G : (b + 1) % G;
            unsigned int v;
            do {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + nb) : "memory");
            } while (v < (unsigned int)r + 1);
        }
        __syncthreads();
    }
}

int main(int argc, char **argv)
{
    const int G = argc > 1 ? atoi(argv[1]) : 148, rounds = argc > 2 ? atoi(argv[2]) : 2000;
    unsigned int *buf;
    cudaMalloc(&buf, 4096 * sizeof(unsigned int));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int mode = 0; mode < 3; ++mode) {
        cudaMemset(buf, 0, 4096 * sizeof(unsigned int));
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3(G);
        lc.blockDim = dim3(256);
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeCooperative;
        at[0].val.cooperative = 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        int relaxed = mode == 2;
        void *args_b[] = {&buf, (void *)&rounds, &relaxed};
        void *args_n[] = {&buf, (void *)&rounds};
        cudaEventRecord(a);
        cudaError_t e = mode == 1 ? cudaLaunchKernelExC(&lc, (const void *)neighbour_flags, args_n)
                                  : cudaLaunchKernelExC(&lc, (const void *)grid_barrier, args_b);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        printf("%s G=%d rounds=%d: %.3f us per round (%s)\n",
               mode == 0 ? "grid barrier (acquire poll)" : mode == 1 ? "neighbour flags (2 partners)"
                                                                     : "grid barrier (relaxed poll)",
               G, rounds, 1e3 * ms / rounds, cudaGetErrorString(e));
    }
    return 0;
}
