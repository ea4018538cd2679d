// fp32 (6,6) step-kernel variants (BASELINE C5). Default first: TY = 30 with the
// producer warp is 16 warps -> 128 registers for the 13-deep queue, no spills.
#include "../vti_entry.cuh"
VTI_TABLE(vti_variants_f32_r6,
          (entry_io<float, 6, 6, 30, 1, 1, 3, 1>()), (entry<float, 6, 6, 32, 1, 0, 3, 1>()),
          (entry<float, 6, 6, 32, 1, 1, 3, 1>()), (entry<float, 6, 6, 16, 1, 0, 3, 2>()),
          (entry<float, 6, 6, 30, 2, 1, 3, 1, 2>()))
