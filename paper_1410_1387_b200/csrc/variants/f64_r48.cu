// fp64 (4,4) and (8,4) variants: 16- or 14-row tiles so three
// stages fit in shared memory. Default first per pair.
#include "../vti_entry.cuh"
VTI_TABLE(vti_variants_f64_r48,
          (entry<double, 4, 4, 16, 1, 1, 3, 1>()), (entry<double, 4, 4, 16, 1, 0, 3, 1>()),
          (entry<double, 4, 4, 14, 1, 1, 3, 1>()),
          (entry<double, 8, 4, 16, 1, 1, 3, 1>()), (entry<double, 8, 4, 16, 1, 0, 3, 1>()),
          (entry<double, 8, 4, 14, 1, 1, 3, 1>()))
