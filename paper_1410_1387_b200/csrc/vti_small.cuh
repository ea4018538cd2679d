// vti_small.cuh -- the step kernel for small, latency-bound grids (fp32, single slab).
//
// The persistent kernel of vti_kernel.cuh marches a register queue of q along z,
// so a work item of one plane still walks 2 R_z priming loads and one full load
// through its 3-stage ring, one round trip after another. That latency is most
// of a step on grids like BASELINE C1 (64^3: 0.26 M points, ~4.6 us per step).
// Here one CTA computes one (64 x TY tile, plane k) item with one round trip of
// loads, all in flight at once. Three forms, same arithmetic (the scalar
// canonical order of the main kernel, reading c12, so results are
// bitwise identical):
//  * vti_small_direct_kernel (the default): TMA stages only what threads share,
//    the halo'd p^n plane tile and the w^z + gz row; every thread loads its own
//    q^n column k - R_z .. k + R_z (zero outside 0..nz-1: the zero exterior in
//    z), p^{n-1}, q^{n-1} and model straight into registers;
//  * vti_small_kernel (VTI_SMALL_DIRECT=0): one elected thread issues every
//    load as TMA on one mbarrier, the q column as one 3-D box;
//  * vti_small_multi_kernel (VTI_MULTI=1): a whole vti_step call in one
//    cooperative launch, per-item epoch counters between steps (slower).
#pragma once

#include "vti_kernel.cuh"

namespace vti {

template <typename T>
struct SmallParams {
    StepParams<T> P;
    CUtensorMap tm_qcol;   // q^n interior view, box {TX, TY, 2 R_z + 1}
    // interior views (row 0, plane 0; strides P.ys, P.zs) for the direct-load kernel
    const T *q_cur, *p_m, *q_m, *vx, *vn, *vz;
};

template <typename T, int R, int RZ, int TY>
struct SmallCfg {
    using C = Cfg<T, R, RZ, TY>;
    static constexpr int NQ = C::NQ;
    static constexpr int OFF_P = 0;
    static constexpr int OFF_Q = align128(C::P_BYTES);               // [NQ][TY][TX]
    static constexpr int OFF_PM = OFF_Q + NQ * C::S_BYTES;
    static constexpr int OFF_QM = OFF_PM + C::S_BYTES;
    static constexpr int OFF_VX = OFF_QM + C::S_BYTES;
    static constexpr int OFF_VN = OFF_VX + C::S_BYTES;
    static constexpr int OFF_VZ = OFF_VN + C::S_BYTES;
    static constexpr int OFF_ZR = OFF_VZ + C::S_BYTES;
    static constexpr int OFF_BAR = align128(OFF_ZR + C::ZROW * C::ES);
    static constexpr int SMEM = OFF_BAR + 16;
    static constexpr uint32_t TX_BYTES = C::P_BYTES + (NQ + 5) * C::S_BYTES + C::ZROW * C::ES;
    static constexpr int THREADS = TY * (TX / 4);   // 16 threads x 4 points per tile row
};

// One tile-plane item's update. prow0 = the halo'd p^n tile in shared memory (row 0 = tile
// row -R, x window starting RA points left of the tile), zr = the plane's w^z row + gz; qv =
// this thread's q^n column k - R_z .. k + R_z, pm4 / qm4 its u^{n-1}, vx4 / vn4 / vz4 its model
// (4 points each). Returns u^{n+1} in pn / qn and this thread's u^n centre values in pc / qc
// (the next step's u^{n-1} in the multi-step kernel). s = s(t^n); inj_row / rec_row: the N4
// trace rows of this step (IO only).
template <typename T, int R, int RZ, int TY, bool IO, int PX = 4>
__device__ __forceinline__ void small_update(const StepParams<T> &P, const T *ptile, const T *zr, int y0, int k,
                                             int tg, int tx, int xg, int yl, const Vec<T, PX> &g4, T gyv, T s,
                                             long long inj_row, long long rec_row, const Vec<T, PX> &pm4,
                                             const Vec<T, PX> &qm4, const Vec<T, PX> (&qv)[2 * RZ + 1],
                                             const Vec<T, PX> &vx4, const Vec<T, PX> &vn4, const Vec<T, PX> &vz4,
                                             T (&pn)[1][PX], T (&qn)[1][PX], T (&pc)[PX], T (&qc)[PX])
{
    using C = Cfg<T, R, RZ, TY>;
    constexpr int NQ = C::NQ;
    constexpr int RA = C::RA;
    static_assert(RA % PX == 0, "x apron must be whole vectors");
    const T *prow = ptile + (tg + R) * C::PW + PX * tx;   // smem row of this tile row
    const T *pbase = ptile + tg * C::PW + PX * tx;
    auto wx = [&](int i) { return ldv<PX>(prow + PX * (i / PX))[i % PX]; };
    T L[PX];
#pragma unroll
    for (int c = 0; c < PX; ++c) {
        pc[c] = wx(RA + c);
        L[c] = P.cxy[0] * pc[c];
    }
#pragma unroll
    for (int l = 1; l <= R; ++l) {
        const Vec<T, PX> yp = ldv<PX>(pbase + (R + l) * C::PW + RA);
        const Vec<T, PX> ym = ldv<PX>(pbase + (R - l) * C::PW + RA);
#pragma unroll
        for (int c = 0; c < PX; ++c) {
            const T xpair = wx(RA + c + l) + wx(RA + c - l);
            const T ypair = yp[c] + ym[c];
            L[c] = fma_rn(P.cxy[l], xpair + ypair, L[c]);
        }
    }
    const T gz = zr[NQ];
    const bool src_here = P.src_mask != 0 && P.src_j == yl && P.src_k == k && P.src_i >= xg && P.src_i < xg + PX;
    bool inj_on = false;
    const T *inj_base = nullptr;
    int inj_e = 0, inj_end = 0;
    if constexpr (IO) {
        if (P.inj_off != nullptr && ps_tile_any(P.inj_off, P.nyl, k, y0, TY)) {
            inj_on = inj_row >= 0 && inj_row < P.inj_nt;
            inj_base = P.inj_tr + inj_row * P.inj_cols;
        }
        if (inj_on && yl < P.nyl) ps_row_range(P.inj_off, P.inj_ent, P.nyl, k, yl, xg, inj_e, inj_end);
    }
#pragma unroll
    for (int c = 0; c < PX; ++c) {
        qc[c] = qv[RZ][c];
        // Eq. 5: ascending m, D = w0 q_{k-Rz}; D = fma(w_m, q_{k-Rz+m}, D)
        T D = zr[0] * qv[0][c];
#pragma unroll
        for (int m = 1; m < NQ; ++m) D = fma_rn(zr[m], qv[m][c], D);
        const T vD = vz4[c] * D;
        T Fp = fma_rn(vx4[c], L[c], vD);
        T Fq = fma_rn(vn4[c], L[c], vD);
        if (src_here && c == P.src_i - xg) {
            if (P.src_mask & 1) Fp = Fp + s;
            if (P.src_mask & 2) Fq = Fq + s;
        }
        if constexpr (IO) {
            if (inj_on) {   // N4 injected sample at column xg + c, after the source
                while (inj_e < inj_end && P.inj_ent[inj_e].x < xg + c) ++inj_e;
                if (inj_e < inj_end && P.inj_ent[inj_e].x == xg + c) {
                    const T v = inj_base[P.inj_ent[inj_e].y];
                    if (P.inj_mask & 1) Fp = Fp + v;
                    if (P.inj_mask & 2) Fq = Fq + v;
                }
            }
        }
        const T g = (g4[c] * gyv) * gz;   // (gx gy) gz
        pn[0][c] = g * fma_rn(P.dt2, Fp, fma_rn(-g, pm4[c], T(2) * pc[c]));
        qn[0][c] = g * fma_rn(P.dt2, Fq, fma_rn(-g, qm4[c], T(2) * qv[RZ][c]));
    }
    if constexpr (IO) record_points_row<T, 1, PX>(P, k, y0, TY, yl, xg, rec_row, pn, qn);
}

// The q column and stream operands of a thread from the TMA-staged item in shared memory.
template <typename T, int R, int RZ, int TY>
__device__ __forceinline__ void small_operands_smem(const uint8_t *smem, int tg, int tx, V4<T> (&qv)[2 * RZ + 1],
                                                    V4<T> &vx4, V4<T> &vn4, V4<T> &vz4)
{
    using C = Cfg<T, R, RZ, TY>;
    using SC = SmallCfg<T, R, RZ, TY>;
    const T *st = reinterpret_cast<const T *>(smem);
    const int sidx = tg * TX + 4 * tx;
#pragma unroll
    for (int m = 0; m < 2 * RZ + 1; ++m) qv[m] = lds4(st + SC::OFF_Q / C::ES + sidx + m * TX * TY);
    vx4 = lds4(st + SC::OFF_VX / C::ES + sidx);
    vn4 = lds4(st + SC::OFF_VN / C::ES + sidx);
    vz4 = lds4(st + SC::OFF_VZ / C::ES + sidx);
}

// IO: also the N4 point sets (injection into F, receivers from u^{n+1}; see StepParams).
template <typename T, int R, int RZ, int TY, bool IO = false>
__global__ void __launch_bounds__(SmallCfg<T, R, RZ, TY>::THREADS)
    vti_small_kernel(const __grid_constant__ SmallParams<T> S)
{
    using C = Cfg<T, R, RZ, TY>;
    using SC = SmallCfg<T, R, RZ, TY>;
    constexpr int RA = C::RA;
    const StepParams<T> &P = S.P;
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + SC::OFF_BAR);

    int x0, y0, kb, ke;
    decode_item<TY>(P, blockIdx.x, x0, y0, kb, ke);   // zchunk = 1: plane k = kb
    const int k = kb;
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        // programmatic dependent launch: everything above overlaps the previous step; the
        // previous grid must complete before this item reads u^n / overwrites u^{n-1}
        // (no-op without the launch attribute). Every store below follows these loads.
        asm volatile("griddepcontrol.wait;" ::: "memory");
        mbar_arrive_expect_tx(bar, SC::TX_BYTES);
        tma_load_3d(smem + SC::OFF_P, &P.tm_p, x0 - RA, y0, k, bar);
        tma_load_3d(smem + SC::OFF_Q, &S.tm_qcol, x0, y0, k - RZ, bar);
        tma_load_3d(smem + SC::OFF_PM, &P.tm_pm, x0, y0, k, bar);
        tma_load_3d(smem + SC::OFF_QM, &P.tm_qm, x0, y0, k, bar);
        tma_load_3d(smem + SC::OFF_VX, &P.tm_vx, x0, y0, k, bar);
        tma_load_3d(smem + SC::OFF_VN, &P.tm_vn, x0, y0, k, bar);
        tma_load_3d(smem + SC::OFF_VZ, &P.tm_vz, x0, y0, k, bar);
        bulk_load(smem + SC::OFF_ZR, P.zrow + (size_t)k * C::ZROW, C::ZROW * C::ES, bar);
    }
    // independent of the loads: this thread's columns, damping and output pointers
    const int tx = threadIdx.x & 15, tg = threadIdx.x >> 4;
    const int xg = x0 + 4 * tx, yl = y0 + tg;
    const V4<T> g4 = lds4(P.gx + xg);   // generic load (global)
    const T gyv = (yl < P.nyl) ? P.gy[yl] : T(0);
    const bool store_ok = (yl < P.nyl) && (xg < P.nx);
    const T sv = P.s_table ? P.s_table[P.s_index] : P.s;
    __syncthreads();   // the barrier is initialised before anyone waits on it
    mbar_wait(bar, 0);

    const T *st = reinterpret_cast<const T *>(smem);
    const int sidx = tg * TX + 4 * tx;
    const V4<T> pm4 = lds4(st + SC::OFF_PM / C::ES + sidx);
    const V4<T> qm4 = lds4(st + SC::OFF_QM / C::ES + sidx);
    V4<T> qv[2 * RZ + 1], vx4, vn4, vz4;
    small_operands_smem<T, R, RZ, TY>(smem, tg, tx, qv, vx4, vn4, vz4);
    T pn[1][4], qn[1][4], pc[4], qc[4];
    small_update<T, R, RZ, TY, IO>(P, st + SC::OFF_P / C::ES, st + SC::OFF_ZR / C::ES, y0, k, tg, tx, xg, yl, g4,
                                   gyv, sv, IO ? inj_row_of(P) : 0, IO ? rec_row_of(P) : 0, pm4, qm4, qv, vx4, vn4,
                                   vz4, pn, qn, pc, qc);
    if (store_ok) {
        const long long off = (long long)k * P.zs + (long long)yl * P.ys + xg;
        stv(P.p_out + off, pn[0]);
        stv(P.q_out + off, qn[0]);
    }
}

// ---------------------------------------------------------------- direct-load small-grid kernel
// The same item with only the halo'd p^n tile (the operand other threads share) and the w^z row
// staged by TMA; every thread loads its own q^n column, u^{n-1} and model straight from global
// memory into registers (14 independent 16-byte loads, all in flight at once). Shared memory
// drops from ~64 KB to ~8 KB per item, and the TMA unit moves 24 rows per item instead of 168.
template <typename T, int R, int RZ, int TY>
struct SmallDCfg {
    using C = Cfg<T, R, RZ, TY>;
    static constexpr int OFF_P = 0;
    static constexpr int OFF_ZR = align128(C::P_BYTES);
    static constexpr int OFF_BAR = align128(OFF_ZR + C::ZROW * C::ES);
    static constexpr int SMEM = OFF_BAR + 16;
    static constexpr uint32_t TX_BYTES = C::P_BYTES + C::ZROW * C::ES;
};

template <typename T, int PX> __device__ __forceinline__ Vec<T, PX> vzero()
{
    Vec<T, PX> v;
    if constexpr (std::is_same<T, float>::value && PX == 4) v.v = make_float4(0.f, 0.f, 0.f, 0.f);
    else if constexpr (std::is_same<T, float>::value && PX == 2) v.v = make_float2(0.f, 0.f);
    else if constexpr (PX == 4) v.a = v.b = make_double2(0.0, 0.0);
    else v.a = make_double2(0.0, 0.0);
    return v;
}
template <typename T> __device__ __forceinline__ V4<T> v4_zero();
template <> __device__ __forceinline__ V4<float> v4_zero<float>() { return V4<float>{make_float4(0.f, 0.f, 0.f, 0.f)}; }
template <> __device__ __forceinline__ V4<double> v4_zero<double>()
{
    return V4<double>{make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
}

// PX consecutive x points per thread (TX / PX threads per tile row): fewer points per thread
// shorten each thread's dependent instruction chain, the latency of a small-grid step.
template <typename T, int R, int RZ, int TY, bool IO = false, int PX = 4>
__global__ void __launch_bounds__(TY * (TX / PX))
    vti_small_direct_kernel(const __grid_constant__ SmallParams<T> S)
{
    using C = Cfg<T, R, RZ, TY>;
    using DC = SmallDCfg<T, R, RZ, TY>;
    using VP = Vec<T, PX>;
    constexpr int RA = C::RA;
    constexpr int NQ = C::NQ;
    constexpr int TPR = TX / PX;
    const StepParams<T> &P = S.P;
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + DC::OFF_BAR);

    int x0, y0, kb, ke;
    decode_item<TY>(P, blockIdx.x, x0, y0, kb, ke);   // zchunk = 1: plane k = kb
    const int k = kb;
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    const int tx = threadIdx.x % TPR, tg = threadIdx.x / TPR;
    const int xg = x0 + PX * tx, yl = y0 + tg;
    const VP g4 = ldv<PX>(P.gx + xg);
    const T gyv = (yl < P.nyl) ? P.gy[yl] : T(0);
    const bool store_ok = (yl < P.nyl) && (xg < P.nx);
    const T sv = P.s_table ? P.s_table[P.s_index] : P.s;
    __syncthreads();   // the barrier is initialised before anyone waits on it
    // programmatic dependent launch: every thread reads the previous step's output below
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(bar, DC::TX_BYTES);
        tma_load_3d(smem + DC::OFF_P, &P.tm_p, x0 - RA, y0, k, bar);
        bulk_load(smem + DC::OFF_ZR, P.zrow + (size_t)k * C::ZROW, C::ZROW * C::ES, bar);
    }
    VP qv[NQ], pm4 = vzero<T, PX>(), qm4 = vzero<T, PX>(), vx4 = vzero<T, PX>(), vn4 = vzero<T, PX>(),
               vz4 = vzero<T, PX>();
#pragma unroll
    for (int m = 0; m < NQ; ++m) qv[m] = vzero<T, PX>();
    if (store_ok) {   // this thread's points: q column (zero exterior in z), u^{n-1}, model
        const long long off = (long long)yl * P.ys + xg;
#pragma unroll
        for (int m = 0; m < NQ; ++m) {
            const int kk = k - RZ + m;
            if (kk >= 0 && kk < P.nz) qv[m] = ldv<PX>(S.q_cur + off + (long long)kk * P.zs);
        }
        const long long o = off + (long long)k * P.zs;
        pm4 = ldv<PX>(S.p_m + o);
        qm4 = ldv<PX>(S.q_m + o);
        vx4 = ldv<PX>(S.vx + o);
        vn4 = ldv<PX>(S.vn + o);
        vz4 = ldv<PX>(S.vz + o);
    }
    mbar_wait(bar, 0);
    const T *st = reinterpret_cast<const T *>(smem);
    T pn[1][PX], qn[1][PX], pc[PX], qc[PX];
    small_update<T, R, RZ, TY, IO, PX>(P, st + DC::OFF_P / C::ES, st + DC::OFF_ZR / C::ES, y0, k, tg, tx, xg, yl,
                                       g4, gyv, sv, IO ? inj_row_of(P) : 0, IO ? rec_row_of(P) : 0, pm4, qm4, qv,
                                       vx4, vn4, vz4, pn, qn, pc, qc);
    if (store_ok) {
        const long long off = (long long)k * P.zs + (long long)yl * P.ys + xg;
        stv(P.p_out + off, pn[0]);
        stv(P.q_out + off, qn[0]);
    }
}

// ---------------------------------------------------------------- multi-step small-grid kernel
// Small grids are latency-bound: each step of vti_small_kernel is one dependent launch (PDL +
// CUDA graphs still leave ~3.5 us per step on C1). Here ONE cooperative launch advances
// nsteps steps: every CTA owns one (tile, plane) item for the whole launch, keeps its own u^n
// and u^{n-1} points in registers (the next step's u^{n-1} is this step's centre), keeps the
// model and w^z row in shared memory, and before step s waits only for the items it exchanges
// data with -- tile rows within R_xy, tiles within the x apron, planes within R_z -- to have
// finished step s-1 (per-item epoch counters, release / acquire at gpu scope). That one wait
// covers both hazards: their u^s is written (read after write) and they no longer read the
// u^{s-1} this step overwrites (write after read). Then one TMA round trip brings the halo'd
// p^n tile and the q^n column. Arithmetic: small_update, i.e. bitwise the one-step kernels.
template <typename T>
struct MultiParams {
    StepParams<T> P[2];        // by buffer parity: P[c] reads buffers c (u^n) and writes 1 - c
    CUtensorMap tm_qcol[2];    // q^n column views of buffer c
    unsigned int *done;        // [items] epoch counters (monotone across launches)
    unsigned int epoch0;       // every counter's value at launch
    int nsteps;
    int cur0;                  // parity of step 0
    int dir;                   // +1 / -1 (vti_reverse): the time index moves by dir per step
    const T *s_table;          // [nsteps] s(t^n) of each step
    int mode;                  // synchronisation variant bits (env VTI_MULTI_MODE, measurement switch)
};

template <typename T, int R, int RZ, int TY, bool IO = false>
__global__ void __launch_bounds__(SmallCfg<T, R, RZ, TY>::THREADS)
    vti_small_multi_kernel(const __grid_constant__ MultiParams<T> M)
{
    using C = Cfg<T, R, RZ, TY>;
    using SC = SmallCfg<T, R, RZ, TY>;
    constexpr int RA = C::RA;
    constexpr int NQ = C::NQ;
    constexpr int DTY = (R + TY - 1) / TY;           // tile rows within R_xy
    constexpr int DTX = (RA + TX - 1) / TX;          // tiles within the x apron
    constexpr int NDEP = (2 * DTY + 1) * (2 * DTX + 1) * NQ;
    static_assert(NDEP <= SC::THREADS, "one polling thread per dependency");
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + SC::OFF_BAR);
    const StepParams<T> &P0 = M.P[0];

    const int item = blockIdx.x;
    int x0, y0, kb, ke;
    decode_item<TY>(P0, item, x0, y0, kb, ke);   // items = ntx * nty * nz, plane k = kb
    const int k = kb;
    const int ntx = P0.ntx, nty = P0.ntr0;
    const int itx = item % ntx, ity = (item / ntx) % nty;
    // this thread's dependency (if any): item (itx + dx, ity + dy, k + dz)
    int dep = -1;
    if (threadIdx.x < NDEP) {
        const int t = threadIdx.x;
        const int dz = t % NQ - RZ, dy = (t / NQ) % (2 * DTY + 1) - DTY, dx = t / (NQ * (2 * DTY + 1)) - DTX;
        const int jx = itx + dx, jy = ity + dy, jz = k + dz;
        if ((dx | dy | dz) != 0 && jx >= 0 && jx < ntx && jy >= 0 && jy < nty && jz >= 0 && jz < P0.nz)
            dep = (jz * nty + jy) * ntx + jx;
    }

    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        // once per launch: u^{n-1} of this item, the model and the plane's w^z + gz row
        const StepParams<T> &P = M.P[M.cur0];
        mbar_arrive_expect_tx(bar, 5 * C::S_BYTES + C::ZROW * C::ES);
        tma_load_3d(smem + SC::OFF_PM, &P.tm_pm, x0, y0, k, bar);
        tma_load_3d(smem + SC::OFF_QM, &P.tm_qm, x0, y0, k, bar);
        tma_load_3d(smem + SC::OFF_VX, &P.tm_vx, x0, y0, k, bar);
        tma_load_3d(smem + SC::OFF_VN, &P.tm_vn, x0, y0, k, bar);
        tma_load_3d(smem + SC::OFF_VZ, &P.tm_vz, x0, y0, k, bar);
        bulk_load(smem + SC::OFF_ZR, P0.zrow + (size_t)k * C::ZROW, C::ZROW * C::ES, bar);
    }
    const int tx = threadIdx.x & 15, tg = threadIdx.x >> 4;
    const int xg = x0 + 4 * tx, yl = y0 + tg;
    const V4<T> g4 = lds4(P0.gx + xg);
    const T gyv = (yl < P0.nyl) ? P0.gy[yl] : T(0);
    const bool store_ok = (yl < P0.nyl) && (xg < P0.nx);
    __syncthreads();
    mbar_wait(bar, 0);
    const T *st = reinterpret_cast<const T *>(smem);
    const int sidx = tg * TX + 4 * tx;
    V4<T> pm4 = lds4(st + SC::OFF_PM / C::ES + sidx);
    V4<T> qm4 = lds4(st + SC::OFF_QM / C::ES + sidx);
    uint32_t phase = 1;

    for (int step = 0; step < M.nsteps; ++step) {
        const int c = (M.cur0 + step) & 1;
        const StepParams<T> &P = M.P[c];
        if (step > 0) {
            // the exchange partners finished step - 1
            if (dep >= 0) {
                const unsigned int want = M.epoch0 + (unsigned int)step;
                unsigned int v;
                if (M.mode & 2) {   // relaxed polling, one acquire fence once satisfied
                    for (;;) {
                        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(M.done + dep) : "memory");
                        if ((int)(v - want) >= 0) break;
                        if (M.mode & 4) __nanosleep(32);
                    }
                    asm volatile("fence.acq_rel.gpu;" ::: "memory");
                } else {
                    for (;;) {
                        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(M.done + dep) : "memory");
                        if ((int)(v - want) >= 0) break;
                        if (M.mode & 4) __nanosleep(32);
                    }
                }
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            // generic-proxy stores of other CTAs (made visible by the acquires above) before
            // this thread's async-proxy (TMA) reads
            asm volatile("fence.proxy.async.global;" ::: "memory");
            mbar_arrive_expect_tx(bar, C::P_BYTES + NQ * C::S_BYTES);
            tma_load_3d(smem + SC::OFF_P, &P.tm_p, x0 - RA, y0, k, bar);
            tma_load_3d(smem + SC::OFF_Q, &M.tm_qcol[c], x0, y0, k - RZ, bar);
        }
        const T sv = M.s_table[step];
        mbar_wait(bar, phase);
        phase ^= 1;
        T pn[1][4], qn[1][4], pc[4], qc[4];
        V4<T> qv[2 * RZ + 1], vx4, vn4, vz4;
        small_operands_smem<T, R, RZ, TY>(smem, tg, tx, qv, vx4, vn4, vz4);
        small_update<T, R, RZ, TY, IO>(P, st + SC::OFF_P / C::ES, st + SC::OFF_ZR / C::ES, y0, k, tg, tx, xg, yl,
                                       g4, gyv, sv, IO ? P.inj_row + (long long)step * M.dir : 0,
                                       IO ? P.rec_row + step : 0, pm4, qm4, qv, vx4, vn4, vz4, pn, qn, pc, qc);
        if (store_ok) {
            const long long off = (long long)k * P.zs + (long long)yl * P.ys + xg;
            stv(P.p_out + off, pn[0]);
            stv(P.q_out + off, qn[0]);
        }
        pm4 = v4_of(pc);   // this step's u^n is the next step's u^{n-1}
        qm4 = v4_of(qc);
        __syncthreads();   // every store issued, every shared-memory read of this step done
        if (threadIdx.x == 0) {
            if (M.mode & 8) asm volatile("fence.proxy.async.global;" ::: "memory");
            if (M.mode & 1) __threadfence();
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(M.done + item),
                         "r"(M.epoch0 + (unsigned int)step + 1u)
                         : "memory");
        }
    }
}

}  // namespace vti
