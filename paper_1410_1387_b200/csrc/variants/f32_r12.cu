// fp32 (12,8) step-kernel variants (the paper's radii). Default first.
#include "../vti_entry.cuh"
VTI_TABLE(vti_variants_f32_r12,
          (entry<float, 12, 8, 30, 1, 1, 3, 1>()), (entry<float, 12, 8, 32, 1, 1, 3, 1>()),
          (entry<float, 12, 8, 32, 1, 0, 3, 1>()), (entry<float, 12, 8, 16, 1, 0, 2, 2>()))
