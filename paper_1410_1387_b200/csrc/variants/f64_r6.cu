// fp64 (6,6) variants. Default: two x points per thread, TY = 15 + producer warp
// (16 warps, 128 registers; C5 fp64 86.9 -> 93.9 Gpoints/s against the 4-point
// TY = 14 mapping, which runs 8 warps at 244 registers).
#include "../vti_entry.cuh"
VTI_TABLE(vti_variants_f64_r6,
          (entry_io<double, 6, 6, 15, 1, 1, 3, 1, 2>()), (entry<double, 6, 6, 16, 1, 0, 3, 1, 2>()),
          (entry<double, 6, 6, 14, 1, 1, 3, 1>()), (entry<double, 6, 6, 16, 1, 0, 3, 1>()),
          (entry<double, 6, 6, 16, 1, 1, 3, 1>()))
