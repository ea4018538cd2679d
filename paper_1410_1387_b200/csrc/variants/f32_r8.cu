// fp32 (8,4) step-kernel variants (BASELINE C3). Default first.
#include "../vti_entry.cuh"
VTI_TABLE(vti_variants_f32_r8,
          (entry_io<float, 8, 4, 32, 1, 1, 3, 1>()), (entry<float, 8, 4, 32, 1, 0, 3, 1>()),
          (entry<float, 8, 4, 30, 1, 1, 3, 1>()), (entry<float, 8, 4, 16, 1, 1, 3, 2>()),
          (entry<float, 8, 4, 32, 2, 1, 3, 1, 2>()))
