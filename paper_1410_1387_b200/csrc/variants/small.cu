// Small-grid step kernels (vti_small.cuh), fp32, 16-row tiles: the tile height the
// runtime picks for grids of at most 4 M points, for the radius pairs whose default
// mapping has 4 x points per thread.
#include "../vti_entry.cuh"
#include "../vti_small.cuh"

template <typename T, int R, int RZ, int TY>
static SmallEntry small_entry()
{
    using namespace vti;
    return SmallEntry{(int)sizeof(T), R, RZ, TY, (const void *)vti_small_kernel<T, R, RZ, TY>,
                      (const void *)vti_small_kernel<T, R, RZ, TY, true>,
                      (const void *)vti_small_multi_kernel<T, R, RZ, TY>,
                      (const void *)vti_small_multi_kernel<T, R, RZ, TY, true>,
                      (const void *)vti_small_direct_kernel<T, R, RZ, TY>,
                      (const void *)vti_small_direct_kernel<T, R, RZ, TY, true>, SmallDCfg<T, R, RZ, TY>::SMEM,
                      SmallCfg<T, R, RZ, TY>::SMEM, SmallCfg<T, R, RZ, TY>::THREADS};
}

SmallTable vti_small_kernels()
{
    // fp32 only: an fp64 item (128 KB of shared memory, 1 CTA per SM) measured slower than the
    // persistent fp64 kernel on C1 (32.5 vs 39.4 Gpoints/s)
    // fp32 only: fp64 items (the direct form at 184-246 registers, one CTA per SM) measured
    // slower than the persistent fp64 kernel on C1 fp64 in round 2 too: 37.6 (direct) and 35.6
    // (TMA-staged) vs 40.5 Gpoints/s
    static const SmallEntry t[] = {small_entry<float, 4, 4, 16>(), small_entry<float, 8, 4, 16>(),
                                   small_entry<float, 6, 6, 16>()};
    // 32-row small-grid tiles (128 items on C1, one CTA per SM) measured slower in round 2:
    // one-step 74.5 vs 77.8-78.1 Gpoints/s, multi-step 47 vs 34 (both below the default)
    return SmallTable{t, (int)(sizeof t / sizeof t[0])};
}
