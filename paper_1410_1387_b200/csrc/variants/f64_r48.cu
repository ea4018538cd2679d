// fp64 (4,4) and (8,4) variants. Default first per pair: two x
// points per thread (one double2) halve the q-queue registers, so 15 consumer
// warps + a producer warp fit 128 registers (C2 fp64 88.8 -> 95.8, C3 71.9 -> 93.2
// Gpoints/s against the 4-point, 8-warp mapping). The 4-point variants use 14- or
// 16-row tiles so three stages fit in shared memory.
#include "../vti_entry.cuh"
VTI_TABLE(vti_variants_f64_r48,
          (entry_io<double, 4, 4, 15, 1, 1, 3, 1, 2>()), (entry<double, 4, 4, 16, 1, 0, 3, 1, 2>()),
          (entry<double, 4, 4, 16, 1, 1, 3, 1, 2>()),
          (entry<double, 4, 4, 16, 1, 1, 3, 1>()), (entry<double, 4, 4, 16, 1, 0, 3, 1>()),
          (entry<double, 4, 4, 14, 1, 1, 3, 1>()),
          (entry_io<double, 8, 4, 15, 1, 1, 3, 1, 2>()), (entry<double, 8, 4, 16, 1, 0, 3, 1, 2>()),
          (entry<double, 8, 4, 16, 1, 1, 3, 1, 2>()),
          (entry<double, 8, 4, 16, 1, 1, 3, 1>()), (entry<double, 8, 4, 16, 1, 0, 3, 1>()),
          (entry<double, 8, 4, 14, 1, 1, 3, 1>()))
