// vti_variants.h -- the table of compiled step-kernel variants.
//
// Each translation unit under csrc/variants/ instantiates a few
// vti_step_kernel<T, R, RZ, TY, RPT, WP, STAGES, MINB> variants and exports
// them as a VariantTable, so the instantiations compile in parallel. The
// runtime scans the tables in vti_variant_tables() order; the first entry that
// matches (precision, r_xy, r_z) is the default for that pair.
#pragma once

struct KernelEntry {
    int esize, r, rz, ty, rpt, wp, stages, minb, stage_bytes;
    int px;                // points per thread along x (4, or 2 for the fp64 double2 mapping)
    const void *fn;        // host stub of the instantiation (cudaLaunchKernelExC with a StepParams<T> argument)
    const void *fn_peer;   // the same with the fused peer-halo stores (edge launches of peer-connected slabs)
    const void *fn_io;     // with the N4 point sets (injection / receivers), or NULL (default variants only)
    const void *fn_peer_io;
    int zrow;
    int threads;
};

struct VariantTable {
    const KernelEntry *e;
    int n;
};

VariantTable vti_variants_f32_r4();    // (4,4)
VariantTable vti_variants_f32_r8();    // (8,4)
VariantTable vti_variants_f32_r6();    // (6,6)
VariantTable vti_variants_f32_r12();   // (12,8)
VariantTable vti_variants_f64_r48();   // (4,4), (8,4)
VariantTable vti_variants_f64_r6();    // (6,6)
VariantTable vti_variants_f64_r12();   // (12,8)

// Small-grid kernels (vti_small.cuh): one CTA per (tile, plane), all loads of the item at once.
struct SmallEntry {
    int esize, r, rz, ty;
    const void *fn;
    const void *fn_io;     // with the N4 point sets
    const void *fn_multi;  // multi-step cooperative kernel (vti_small_multi_kernel), and its IO form
    const void *fn_multi_io;
    const void *fn_direct; // direct-load form (vti_small_direct_kernel), and its IO form
    const void *fn_direct_io;
    int smem_direct;
    int smem, threads;
};
struct SmallTable {
    const SmallEntry *e;
    int n;
};
SmallTable vti_small_kernels();
