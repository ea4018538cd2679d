// fp32 (4,4) step-kernel variants (BASELINE C1, C2, C4). Default first.
// RPT = 2 (8 warps, up to 255 registers) halves the y-neighbour shared-memory
// reads but measured slower (C2 187 vs 193 Gpoints/s): an autotune candidate.
#include "../vti_entry.cuh"
VTI_TABLE(vti_variants_f32_r4,
          (entry_io<float, 4, 4, 32, 1, 1, 3, 1>()), (entry<float, 4, 4, 32, 1, 0, 3, 1>()),
          (entry<float, 4, 4, 30, 1, 1, 3, 1>()), (entry<float, 4, 4, 32, 2, 0, 3, 1>()),
          (entry<float, 4, 4, 16, 1, 1, 3, 2>()),
          (entry<float, 4, 4, 32, 2, 1, 3, 1, 2>()))
