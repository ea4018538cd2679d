// vti_small.cuh -- the step kernel for small, latency-bound grids (fp32, single slab).
//
// The persistent kernel of vti_kernel.cuh marches a register queue of q along z,
// so a work item of one plane still walks 2 R_z priming loads and one full load
// through its 3-stage ring, one round trip after another. That latency is most
// of a step on grids like BASELINE C1 (64^3: 0.26 M points, ~4.6 us per step).
// Here one CTA computes one (64 x TY tile, plane k) item, and a single elected
// thread issues EVERY load of the item at once on one mbarrier: the halo'd p^n
// plane tile, the whole q^n column k - R_z .. k + R_z as one 3-D TMA box
// (planes outside 0..nz-1 are zero-filled, i.e. the paper's zero exterior in z),
// p^{n-1}, q^{n-1}, vx2, vn2, vz2 and the plane's w^z + gz row. One round trip
// per item. The arithmetic is the scalar canonical order of the main kernel
// (reading c12), so results are bitwise identical.
#pragma once

#include "vti_kernel.cuh"

namespace vti {

template <typename T>
struct SmallParams {
    StepParams<T> P;
    CUtensorMap tm_qcol;   // q^n interior view, box {TX, TY, 2 R_z + 1}
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

template <typename T, int R, int RZ, int TY>
__global__ void __launch_bounds__(SmallCfg<T, R, RZ, TY>::THREADS)
    vti_small_kernel(const __grid_constant__ SmallParams<T> S)
{
    using C = Cfg<T, R, RZ, TY>;
    using SC = SmallCfg<T, R, RZ, TY>;
    constexpr int NQ = C::NQ;
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
    const bool src_here = P.src_mask != 0 && P.src_j == yl && P.src_k == k && P.src_i >= xg && P.src_i < xg + 4;
    __syncthreads();   // the barrier is initialised before anyone waits on it
    mbar_wait(bar, 0);

    const T *st = reinterpret_cast<const T *>(smem);
    const int sidx = tg * TX + 4 * tx;
    const T *prow = st + SC::OFF_P / C::ES + (tg + R) * C::PW + 4 * tx;   // smem row of this tile row
    const T *pbase = st + SC::OFF_P / C::ES + tg * C::PW + 4 * tx;
    auto wx = [&](int i) { return lds4(prow + 4 * (i / 4))[i % 4]; };
    T pc[4], L[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        pc[c] = wx(RA + c);
        L[c] = P.cxy[0] * pc[c];
    }
#pragma unroll
    for (int l = 1; l <= R; ++l) {
        const V4<T> yp = lds4(pbase + (R + l) * C::PW + RA);
        const V4<T> ym = lds4(pbase + (R - l) * C::PW + RA);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const T xpair = wx(RA + c + l) + wx(RA + c - l);
            const T ypair = yp[c] + ym[c];
            L[c] = fma_rn(P.cxy[l], xpair + ypair, L[c]);
        }
    }
    const T *zr = st + SC::OFF_ZR / C::ES;
    const T gz = zr[NQ];
    const T *qcol = st + SC::OFF_Q / C::ES + sidx;   // plane m of the column at qcol + m * TX * TY
    const V4<T> pm4 = lds4(st + SC::OFF_PM / C::ES + sidx);
    const V4<T> qm4 = lds4(st + SC::OFF_QM / C::ES + sidx);
    const V4<T> vx4 = lds4(st + SC::OFF_VX / C::ES + sidx);
    const V4<T> vn4 = lds4(st + SC::OFF_VN / C::ES + sidx);
    const V4<T> vz4 = lds4(st + SC::OFF_VZ / C::ES + sidx);
    const V4<T> qc4 = lds4(qcol + RZ * TX * TY);
    T pn[4], qn[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        // Eq. 5: ascending m, D = w0 q_{k-Rz}; D = fma(w_m, q_{k-Rz+m}, D)
        T D = zr[0] * lds4(qcol)[c];
#pragma unroll
        for (int m = 1; m < NQ; ++m) D = fma_rn(zr[m], lds4(qcol + m * TX * TY)[c], D);
        const T vD = vz4[c] * D;
        T Fp = fma_rn(vx4[c], L[c], vD);
        T Fq = fma_rn(vn4[c], L[c], vD);
        if (src_here && c == P.src_i - xg) {
            const T sv = P.s_table ? P.s_table[P.s_index] : P.s;
            if (P.src_mask & 1) Fp = Fp + sv;
            if (P.src_mask & 2) Fq = Fq + sv;
        }
        const T g = (g4[c] * gyv) * gz;   // (gx gy) gz
        pn[c] = g * fma_rn(P.dt2, Fp, fma_rn(-g, pm4[c], T(2) * pc[c]));
        qn[c] = g * fma_rn(P.dt2, Fq, fma_rn(-g, qm4[c], T(2) * qc4[c]));
    }
    if (store_ok) {
        const long long off = (long long)k * P.zs + (long long)yl * P.ys + xg;
        stv(P.p_out + off, pn);
        stv(P.q_out + off, qn);
    }
}

}  // namespace vti
