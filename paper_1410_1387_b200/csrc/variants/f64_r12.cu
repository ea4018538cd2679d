// fp64 (12,8) variants. Default: two x points per thread, TY = 15 + producer
// warp (N1 fp64 28.7 -> 52.4 Gpoints/s against the 4-point TY = 14 mapping).
#include "../vti_entry.cuh"
VTI_TABLE(vti_variants_f64_r12,
          (entry<double, 12, 8, 15, 1, 1, 3, 1, 2>()), (entry<double, 12, 8, 16, 1, 0, 2, 1, 2>()),
          (entry<double, 12, 8, 14, 1, 1, 3, 1>()), (entry<double, 12, 8, 16, 1, 1, 2, 1>()),
          (entry<double, 12, 8, 16, 1, 0, 2, 1>()))
