// fp64 (6,6) variants: TY = 14 + producer warp = 8 warps -> up to 255 registers.
#include "../vti_entry.cuh"
VTI_TABLE(vti_variants_f64_r6,
          (entry<double, 6, 6, 14, 1, 1, 3, 1>()), (entry<double, 6, 6, 16, 1, 0, 3, 1>()),
          (entry<double, 6, 6, 16, 1, 1, 3, 1>()))
