// fp64 (12,8) variants. Default: two x points per thread (one double2), TY = 8 +
// producer warp = 9 warps, 4-deep TMA ring (N1 fp64 28.7 with the 4-point TY = 14
// mapping -> 52.4 with TY = 15 at 128 registers (644 B of spills) -> 75.9 Gpoints/s
// with TY = 10 and 3 stages -> +4.9 % with TY = 8 and 4 stages: 68.4 -> 71.8 on the
// same box, twice each, 1000 steps; TY = 6 x 5 stages 66.3, TY = 12 55.7, TY = 10
// x 4 stages 69.7). One double per thread (PX = 1, 17 warps at 96 registers) measured
// slower in round 2: 65-66 (TY = 8, 3 or 4 stages), 63-64 (TY = 6 / 4) vs 77-78; two CTAs per
// SM (MINB = 2) spill into L1, which is the shared-memory bound's own pipe: 43 (TY = 8, 2 stages,
// 256 B of spills) and 53 (TY = 6, 120 B) Gpoints/s.
#include "../vti_entry.cuh"
VTI_TABLE(vti_variants_f64_r12,
          (entry_io<double, 12, 8, 8, 1, 1, 4, 1, 2>()), (entry<double, 12, 8, 10, 1, 1, 3, 1, 2>()),
          (entry<double, 12, 8, 15, 1, 1, 3, 1, 2>()), (entry<double, 12, 8, 16, 1, 0, 2, 1, 2>()),
          (entry<double, 12, 8, 14, 1, 1, 3, 1>()), (entry<double, 12, 8, 16, 1, 1, 2, 1>()),
          (entry<double, 12, 8, 16, 1, 0, 2, 1>()))
