// fp32 (12,8) step-kernel variants (the paper's radii). Default first:
// two x points (float2) x two rows per thread, so the two rows share their 2R+2
// y-neighbour loads -- 14 % fewer shared-memory bytes, the bound at R_xy = 12
// (N1 168.6 -> 188.7 Gpoints/s against one row of four points per thread).
#include "../vti_entry.cuh"
VTI_TABLE(vti_variants_f32_r12,
          (entry_io<float, 12, 8, 30, 2, 1, 3, 1, 2>()),
          (entry<float, 12, 8, 30, 1, 1, 3, 1>()), (entry<float, 12, 8, 32, 1, 1, 3, 1>()),
          (entry<float, 12, 8, 32, 1, 0, 3, 1>()), (entry<float, 12, 8, 16, 1, 0, 2, 2>()))
