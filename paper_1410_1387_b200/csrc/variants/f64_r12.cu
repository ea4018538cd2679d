// fp64 (12,8) variants.
#include "../vti_entry.cuh"
VTI_TABLE(vti_variants_f64_r12,
          (entry<double, 12, 8, 14, 1, 1, 3, 1>()), (entry<double, 12, 8, 16, 1, 1, 2, 1>()),
          (entry<double, 12, 8, 16, 1, 0, 2, 1>()))
