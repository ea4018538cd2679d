// vti_entry.cuh -- build a KernelEntry from one vti_step_kernel instantiation.
#pragma once

#include "vti_kernel.cuh"
#include "vti_variants.h"

template <typename T, int R, int RZ, int TY, int RPT, int WP, int S, int B, int PX = 4>
static KernelEntry entry()
{
    using namespace vti;
    return KernelEntry{(int)sizeof(T), R, RZ, TY, RPT, WP, S, B, Cfg<T, R, RZ, TY>::STAGE, PX,
                       (const void *)vti_step_kernel<T, R, RZ, TY, RPT, WP, S, B, false, PX>,
                       (const void *)vti_step_kernel<T, R, RZ, TY, RPT, WP, S, B, true, PX>, nullptr, nullptr,
                       Cfg<T, R, RZ, TY>::ZROW, nthreads(TY, RPT, WP, PX)};
}

// The same plus the N4 point-set (IO) instantiations: the default variant of each table.
template <typename T, int R, int RZ, int TY, int RPT, int WP, int S, int B, int PX = 4>
static KernelEntry entry_io()
{
    using namespace vti;
    KernelEntry e = entry<T, R, RZ, TY, RPT, WP, S, B, PX>();
    e.fn_io = (const void *)vti_step_kernel<T, R, RZ, TY, RPT, WP, S, B, false, PX, true>;
    e.fn_peer_io = (const void *)vti_step_kernel<T, R, RZ, TY, RPT, WP, S, B, true, PX, true>;
    return e;
}

#define VTI_TABLE(name, ...)                                     \
    VariantTable name()                                          \
    {                                                            \
        static const KernelEntry t[] = {__VA_ARGS__};            \
        return VariantTable{t, (int)(sizeof t / sizeof t[0])};   \
    }
