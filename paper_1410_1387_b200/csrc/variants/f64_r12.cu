// fp64 (12,8) variants. Default: two x points per thread (one double2), TY = 10 +
// producer warp = 11 warps at 168 registers without spills (N1 fp64 28.7 with the
// 4-point TY = 14 mapping -> 52.4 with TY = 15 at 128 registers (644 B of spills)
// -> 75.9 Gpoints/s).
#include "../vti_entry.cuh"
VTI_TABLE(vti_variants_f64_r12,
          (entry<double, 12, 8, 10, 1, 1, 3, 1, 2>()), (entry<double, 12, 8, 8, 1, 1, 3, 1, 2>()),
          (entry<double, 12, 8, 15, 1, 1, 3, 1, 2>()), (entry<double, 12, 8, 16, 1, 0, 2, 1, 2>()),
          (entry<double, 12, 8, 14, 1, 1, 3, 1>()), (entry<double, 12, 8, 16, 1, 1, 2, 1>()),
          (entry<double, 12, 8, 16, 1, 0, 2, 1>()))
