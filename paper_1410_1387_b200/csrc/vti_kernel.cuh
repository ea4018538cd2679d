// vti_kernel.cuh -- the fused VTI time-step kernel for sm_100a (B200).
//
// One launch = one time step of the reduced elastic VTI propagator
// (Eqs. 1-3) over a set of x-y tiles:
//   L  = cxy0 p + sum_l cxy_l [(p_{i+l}+p_{i-l}) + (p_{j+l}+p_{j-l})]   Eq. 4 / h^2
//   D  = sum_{m=0}^{2Rz} w^z[k][m] q_{k-Rz+m}                            Eq. 5
//   Fp = vx2 L + vz2 D (+ s at the source),  Fq = vn2 L + vz2 D          Eqs. 1-2
//   u^{n+1} = g (2 u^n - g u^{n-1} + dt^2 F),  g = (gx gy) gz            Eq. 3 + Cerjan
// in exactly the operation order of the oracle (reading c12), so
// parity is bitwise. Build with -fmad=false (no FMA contraction beyond the
// explicit __fmaf_rn below) and without --use_fast_math (IEEE subnormals).
//
// Design: 2.5-D blocking after the paper's GPU kernel
// (x-y tile in shared memory + z register rolling), made
// B200-native:
//  * a persistent grid of CTAs pulls work items (a 64 x TY x-y tile, a z-chunk);
//    TY, the producer mode, rows and x points per thread are template
//    parameters (the fp32 (4,4) default: TY = 32, a dedicated producer warp,
//    4 x points per thread);
//  * one producer lane -- the dedicated producer warp (WP = 1) or the CTA's
//    first thread in line (WP = 0) -- drives a STAGES-deep TMA ring: per z
//    plane it issues cp.async.bulk.tensor loads of the halo'd p^n plane tile,
//    the q^n plane Rz ahead, p^{n-1}, q^{n-1}, vx2, vn2, vz2 and a 1-D bulk
//    copy of the plane's w^z row + gz, all completing on one mbarrier; load
//    j + STAGES is issued as soon as every consumer warp has released load j
//    (empty mbarrier), so STAGES - 1 planes are always in flight. Out-of-bounds
//    box elements are zero-filled by TMA, which IS the paper's zero exterior
//    (l.89-90) in x, y and z;
//  * the consumer warps: each thread owns PX consecutive x points (float4,
//    float2 or double2) of RPT rows, keeps a (2Rz+1)-deep register
//    queue of q along z, reads the p cross from shared memory and writes
//    p^{n+1}, q^{n+1} with vector stores in place over p^{n-1}, q^{n-1};
//  * PEER twins also store the slab's boundary rows into the neighbours' halo
//    rows (multi-GPU), IO twins gather receivers / add injected traces (N4).
#pragma once

#include <cuda.h>
#include <stdint.h>

#include <type_traits>

// fp32 arithmetic on packed pairs (FFMA2 / FADD2 / FMUL2, sm_100a); 0 = scalar form (A/B builds)
#ifndef VTI_PACKED_F32
#define VTI_PACKED_F32 1
#endif

namespace vti {

constexpr int TX = 64;               // tile width in x (points)
constexpr int MAX_R = 12;

// Tile height TY, RPT rows per thread (1 or 2), PX consecutive x points per
// thread (4: one float4 / two double2; 2: one double2): TX / PX threads per row
// group, TY * (TX / PX) / (32 RPT) consumer warps, plus one producer warp when WP = 1.
__host__ __device__ constexpr int cons_warps(int ty, int rpt, int px) { return ty * (TX / px) / (32 * rpt); }
__host__ __device__ constexpr int nthreads(int ty, int rpt, int wp, int px)
{
    return (cons_warps(ty, rpt, px) + wp) * 32;
}

__host__ __device__ constexpr int align128(int b) { return (b + 127) / 128 * 128; }

// T = float (the fp32 path of BASELINE.json) or double.
template <typename T, int R, int RZ, int TY>
struct Cfg {
    // x apron rounded up to 4 elements: the TMA box must start on a 16-byte
    // boundary in x (x0 - RA), and every shared-memory read is then a 4-vector.
    static constexpr int RA = (R + 3) / 4 * 4;
    static constexpr int ES = (int)sizeof(T);
    static constexpr int PW = TX + 2 * RA;                // p tile row length (floats)
    static constexpr int PH = TY + 2 * R;                 // p tile rows
    static constexpr int NQ = 2 * RZ + 1;                 // q queue depth
    static constexpr int ZROW = ((NQ + 1 + 3) / 4) * 4;   // w^z row + gz, padded to 4 elements
    static constexpr int P_BYTES = PW * PH * ES;
    static constexpr int S_BYTES = TX * TY * ES;
    static constexpr int OFF_P = 0;
    static constexpr int OFF_Q = align128(P_BYTES);
    static constexpr int OFF_PM = OFF_Q + S_BYTES;
    static constexpr int OFF_QM = OFF_PM + S_BYTES;
    static constexpr int OFF_VX = OFF_QM + S_BYTES;
    static constexpr int OFF_VN = OFF_VX + S_BYTES;
    static constexpr int OFF_VZ = OFF_VN + S_BYTES;
    static constexpr int OFF_ZR = OFF_VZ + S_BYTES;
    static constexpr int STAGE = align128(OFF_ZR + ZROW * ES);
    static constexpr uint32_t FULL_TX = P_BYTES + 6 * S_BYTES + ZROW * ES;
    static constexpr uint32_t PRIME_TX = S_BYTES;
    static_assert(PW % 4 == 0, "p tile rows must be whole 4-vectors");
    static_assert(PW <= 256 && PH <= 256, "TMA box limit");
};

// All arrays share one geometry: nz planes x (nyl + 2R) rows x nxp floats with
// strides ys (row) and zs (plane) in floats; R halo rows on both y sides (only
// p's are ever non-zero). Tensor-map dims are ordered (x, y, z).
template <typename T>
struct StepParams {
    CUtensorMap tm_p;    // p^n  : halo'd view dims {nx, nyl + 2R, nz}, box {TX + 2RA, TY + 2R, 1}
    CUtensorMap tm_q;    // q^n  : interior view dims {nx, nyl, nz}, box {TX, TY, 1}
    CUtensorMap tm_pm;   // p^{n-1}: interior view of the other p buffer
    CUtensorMap tm_qm;   // q^{n-1}
    CUtensorMap tm_vx;   // vx2
    CUtensorMap tm_vn;   // vn2
    CUtensorMap tm_vz;   // vz2
    T *p_out;            // p^{n+1}: interior row 0, plane 0 of the other p buffer
    T *q_out;            // q^{n+1}: interior row 0, plane 0 of the other q buffer
    // Fused halo transport (y-slabs, peer memory): p^{n+1} of local rows [0, R) is also
    // stored at rows [0, R) of peer_lo (rank-1's buffer from its top halo row, plane 0),
    // and of local rows [nyl - R, nyl) at rows [0, R) of peer_hi (rank+1's buffer from
    // its bottom halo row); peer_zs_* are the neighbours' plane strides. NULL = no peer.
    T *peer_lo;
    T *peer_hi;
    long long peer_zs_lo, peer_zs_hi;
    const T *zrow;       // [nz][ZROW]: w^z[k][0..2Rz], gz[k], 0 ...
    const T *gx;         // [ntx * TX] (1 beyond nx)
    const T *gy;         // [nyl] local rows
    T cxy[MAX_R + 1];
    T dt2;
    T s;                 // s(t^n) this step (direct launches)
    const T *s_table;    // CUDA-graph launches: s(t^n) = s_table[s_index], refilled before each replay
    int s_index;
    int src_i, src_j, src_k, src_mask;   // local indices; src_mask = 0: no source here
    int nx, nyl, nz;
    long long ys, zs;                    // row / plane strides (elements)
    int ntx;                             // tiles along x
    int tr0, ntr0, tr1, ntr1;            // tile rows [tr0, tr0+ntr0) then [tr1, tr1+ntr1)
    int zchunk, nzc;                     // planes per chunk, chunks
    int items;                           // ntx * (ntr0 + ntr1) * nzc
    // Round alignment (cooperative launch only): CTAs arrive on *sync_ctr after
    // each non-final round r and wait until it reaches sync_base + (r+1) * grid,
    // so all CTAs start round r+1 together and neighbouring tiles stay within
    // the L2 window of each other's p rows. NULL = no alignment.
    unsigned long long *sync_ctr;
    unsigned long long sync_base;
    // Fused multi-GPU step (PEER kernels only): one launch covers the edge tile rows
    // (tr0.., tr1..; items [0, edge_items)) and then the interior rows [tr2, tr2 + ntr2)
    // (the remaining items). The CTA that completes the last edge item -- the edge_ctr
    // counter reaching edge_target after every edge CTA fenced its stores at system
    // scope -- stores sig_val[i] to *sig[i] with release semantics: the neighbours'
    // ACK and DATA flag words. edge_items = 0: a plain launch (tile rows tr0.., tr1..).
    int tr2, ntr2;
    int edge_items;
    unsigned long long *edge_ctr;
    unsigned long long edge_target;
    unsigned int *sig[4];
    unsigned int sig_val[4];
    // N4 point sets (IO kernels only; NULL = none), SURVEY.md 8(f) N4. Each is a CSR over
    // (plane k, local row yl): entries ent[off[k*nyl + yl] .. off[k*nyl + yl + 1]) = (x, column),
    // sorted by x.
    //  * injection: inj_tr[row * inj_cols + column] is added into F_p (inj_mask bit 1) / F_q
    //    (bit 2) after the Ricker source; row = the time index n - t_first of this step;
    //  * receivers: the u^{n+1} just computed goes to rec_tr[(row * rec_cols + column) * nf + f]
    //    (p before q, nf = fields in rec_mask).
    // Rows: direct launches pass inj_row / rec_row; graph replays read dyn[0] + graph_i * dyn[2]
    // and dyn[1] + graph_i (the header refilled before each replay). Rows outside
    // [0, inj_nt) / [0, rec_cap) are skipped.
    const int *inj_off;
    const int2 *inj_ent;
    const T *inj_tr;
    int inj_cols, inj_mask, inj_nt;
    long long inj_row;
    const int *rec_off;
    const int2 *rec_ent;
    T *rec_tr;
    int rec_cols, rec_mask, rec_cap;
    long long rec_row;
    const long long *dyn;
    int graph_i;
};

// ---------------------------------------------------------------- N4 point-set helpers
template <typename PP>
__device__ __forceinline__ long long inj_row_of(const PP &P)
{
    return P.dyn ? P.dyn[0] + (long long)P.graph_i * P.dyn[2] : P.inj_row;
}
template <typename PP>
__device__ __forceinline__ long long rec_row_of(const PP &P)
{
    return P.dyn ? P.dyn[1] + P.graph_i : P.rec_row;
}

// Does the tile (rows [y0, y0 + ty) of plane k) hold any entry of the set? (CTA-uniform)
__device__ __forceinline__ bool ps_tile_any(const int *off, int nyl, int k, int y0, int ty)
{
    const long long b = (long long)k * nyl;
    return off[b + y0] != off[b + min(y0 + ty, nyl)];
}

// First entry of row (k, yl) with x >= x0, and the row's end.
__device__ __forceinline__ void ps_row_range(const int *off, const int2 *ent, int nyl, int k, int yl, int x0,
                                             int &e, int &e_end)
{
    const long long b = (long long)k * nyl + yl;
    int lo = off[b], hi = off[b + 1];
    e_end = hi;
    while (lo < hi) {   // lower bound of x0
        const int mid = (lo + hi) >> 1;
        if (ent[mid].x < x0) lo = mid + 1;
        else hi = mid;
    }
    e = lo;
}

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
    uint32_t done;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    } while (!done);
}

__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *tm, int c0, int c1, int c2,
                                            uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void bulk_load(void *dst, const void *src, uint32_t bytes, uint64_t *bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long *p)
{
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void named_bar_sync(int id, int nthreads)
{
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap *tm)
{
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tm)) : "memory");
}

// N consecutive elements held in 16-byte vectors: float4 (float, 4), two double2
// (double, 4) or one double2 (double, 2).
template <typename T, int N> struct Vec;
template <> struct Vec<float, 4> {
    float4 v;
    __device__ __forceinline__ float operator[](int c) const { return c == 0 ? v.x : c == 1 ? v.y : c == 2 ? v.z : v.w; }
};
template <> struct Vec<float, 2> {
    float2 v;
    __device__ __forceinline__ float operator[](int c) const { return c == 0 ? v.x : v.y; }
};
template <> struct Vec<double, 4> {
    double2 a, b;
    __device__ __forceinline__ double operator[](int c) const { return c == 0 ? a.x : c == 1 ? a.y : c == 2 ? b.x : b.y; }
};
template <> struct Vec<double, 2> {
    double2 a;
    __device__ __forceinline__ double operator[](int c) const { return c == 0 ? a.x : a.y; }
};
template <typename T> using V4 = Vec<T, 4>;

// loads of N elements (16-byte aligned), shared or global memory (generic addressing)
template <int N> __device__ __forceinline__ Vec<float, N> ldv(const float *p);
template <> __device__ __forceinline__ Vec<float, 4> ldv<4>(const float *p)
{
    return Vec<float, 4>{*reinterpret_cast<const float4 *>(p)};
}
template <> __device__ __forceinline__ Vec<float, 2> ldv<2>(const float *p)
{
    return Vec<float, 2>{*reinterpret_cast<const float2 *>(p)};
}
template <int N> __device__ __forceinline__ Vec<double, N> ldv(const double *p);
template <> __device__ __forceinline__ Vec<double, 4> ldv<4>(const double *p)
{
    return Vec<double, 4>{reinterpret_cast<const double2 *>(p)[0], reinterpret_cast<const double2 *>(p)[1]};
}
template <> __device__ __forceinline__ Vec<double, 2> ldv<2>(const double *p)
{
    return Vec<double, 2>{*reinterpret_cast<const double2 *>(p)};
}
__device__ __forceinline__ V4<float> v4_of(const float (&a)[4]) { return V4<float>{make_float4(a[0], a[1], a[2], a[3])}; }
__device__ __forceinline__ V4<double> v4_of(const double (&a)[4])
{
    return V4<double>{make_double2(a[0], a[1]), make_double2(a[2], a[3])};
}
__device__ __forceinline__ V4<float> lds4(const float *p) { return ldv<4>(p); }
__device__ __forceinline__ V4<double> lds4(const double *p) { return ldv<4>(p); }

__device__ __forceinline__ void stv(float *p, const float (&v)[4])
{
    *reinterpret_cast<float4 *>(p) = make_float4(v[0], v[1], v[2], v[3]);
}
__device__ __forceinline__ void stv(float *p, const float (&v)[2]) { *reinterpret_cast<float2 *>(p) = make_float2(v[0], v[1]); }
__device__ __forceinline__ void stv(double *p, const double (&v)[4])
{
    reinterpret_cast<double2 *>(p)[0] = make_double2(v[0], v[1]);
    reinterpret_cast<double2 *>(p)[1] = make_double2(v[2], v[3]);
}
__device__ __forceinline__ void stv(double *p, const double (&v)[2])
{
    *reinterpret_cast<double2 *>(p) = make_double2(v[0], v[1]);
}
__device__ __forceinline__ float fma_rn(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double fma_rn(double a, double b, double c) { return __fma_rn(a, b, c); }

template <int TY, typename PP>
__device__ __forceinline__ void decode_item(const PP &P, int item, int &x0, int &y0, int &kb, int &ke)
{
    // edge rows (tr0.., tr1..) first; with edge_items > 0 the interior rows (tr2..) follow
    const bool edge = P.edge_items == 0 || item < P.edge_items;
    const int it = edge ? item : item - P.edge_items;
    const int nsel = edge ? P.ntr0 + P.ntr1 : P.ntr2;
    const int tx = it % P.ntx;
    const int rest = it / P.ntx;
    const int t = rest % nsel;
    const int zc = rest / nsel;
    x0 = tx * TX;
    y0 = (edge ? (t < P.ntr0 ? P.tr0 + t : P.tr1 + (t - P.ntr0)) : P.tr2 + t) * TY;   // local row of the tile
    kb = zc * P.zchunk;
    ke = min(P.nz, kb + P.zchunk);
}

// The flat sequence of stage loads of one CTA: for each of its work items,
// 2Rz priming loads (q only) then one full load per plane. Driven by a
// single thread; load j goes to stage j % STAGES.
template <typename T, int R, int RZ, int TY, int STAGES>
struct Producer {
    int item, t, nload, x0, y0, kb, ke;
    int stage;
    uint32_t phase;

    __device__ __forceinline__ void start(const StepParams<T> &P)
    {
        item = blockIdx.x;
        t = 0;
        stage = 0;
        phase = 0;
        if (item < P.items) {
            decode_item<TY>(P, item, x0, y0, kb, ke);
            nload = (ke - kb) + 2 * RZ;
        }
    }

    __device__ __forceinline__ void issue(const StepParams<T> &P, uint8_t *smem, uint64_t *full, uint64_t *empty)
    {
        using C = Cfg<T, R, RZ, TY>;
        constexpr int RA = C::RA;
        if (item >= P.items) return;
        mbar_wait(&empty[stage], phase ^ 1);   // every warp released the previous load of this stage
        uint8_t *st = smem + stage * C::STAGE;
        uint64_t *bar = &full[stage];
        if (t < 2 * RZ) {
            // priming: q^n planes kb-Rz .. kb+Rz-1 (OOB planes -> 0)
            mbar_arrive_expect_tx(bar, C::PRIME_TX);
            tma_load_3d(st + C::OFF_Q, &P.tm_q, x0, y0, kb - RZ + t, bar);
        } else {
            const int k = kb + t - 2 * RZ;
            mbar_arrive_expect_tx(bar, C::FULL_TX);
            // p^n plane with its apron; the y coordinate is the halo'd row index,
            // whose row y0 is local row y0 - R.
            tma_load_3d(st + C::OFF_P, &P.tm_p, x0 - RA, y0, k, bar);
            tma_load_3d(st + C::OFF_Q, &P.tm_q, x0, y0, k + RZ, bar);
            tma_load_3d(st + C::OFF_PM, &P.tm_pm, x0, y0, k, bar);
            tma_load_3d(st + C::OFF_QM, &P.tm_qm, x0, y0, k, bar);
            tma_load_3d(st + C::OFF_VX, &P.tm_vx, x0, y0, k, bar);
            tma_load_3d(st + C::OFF_VN, &P.tm_vn, x0, y0, k, bar);
            tma_load_3d(st + C::OFF_VZ, &P.tm_vz, x0, y0, k, bar);
            bulk_load(st + C::OFF_ZR, P.zrow + (size_t)k * C::ZROW, C::ZROW * C::ES, bar);
        }
        if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
        }
        if (++t == nload) {
            item += gridDim.x;
            t = 0;
            if (item < P.items) {
                decode_item<TY>(P, item, x0, y0, kb, ke);
                nload = (ke - kb) + 2 * RZ;
            }
        }
    }
};

// N4 receivers: this thread's points of u^{n+1} (rows yr .. yr + RPT - 1, columns xg ..
// xg + PX - 1 of plane k) that are receivers go to their trace row (a tile-uniform early out
// keeps planes without receivers free).
template <typename T, int RPT, int PX>
__device__ __forceinline__ void record_points_row(const StepParams<T> &P, int k, int y0, int ty, int yr, int xg,
                                                  long long row, const T (&pn)[RPT][PX], const T (&qn)[RPT][PX])
{
    if (P.rec_off == nullptr || !ps_tile_any(P.rec_off, P.nyl, k, y0, ty)) return;
    if (row < 0 || row >= P.rec_cap) return;
    const int nf = (P.rec_mask & 1) + ((P.rec_mask >> 1) & 1);
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
        const int yl = yr + r;
        if (yl >= P.nyl || xg >= P.nx) continue;
        int e, e_end;
        ps_row_range(P.rec_off, P.rec_ent, P.nyl, k, yl, xg, e, e_end);
        for (; e < e_end; ++e) {
            const int2 en = P.rec_ent[e];
            if (en.x >= xg + PX) break;
            T vp = pn[r][0], vq = qn[r][0];
#pragma unroll
            for (int c = 1; c < PX; ++c)
                if (en.x == xg + c) {
                    vp = pn[r][c];
                    vq = qn[r][c];
                }
            T *o = P.rec_tr + (row * P.rec_cols + en.y) * nf;
            if (P.rec_mask & 1) *o++ = vp;
            if (P.rec_mask & 2) *o = vq;
        }
    }
}

template <typename T, int RPT, int PX>
__device__ __forceinline__ void record_points(const StepParams<T> &P, int k, int y0, int ty, int yr, int xg,
                                              const T (&pn)[RPT][PX], const T (&qn)[RPT][PX])
{
    record_points_row<T, RPT, PX>(P, k, y0, ty, yr, xg, rec_row_of(P), pn, qn);
}

// ---------------------------------------------------------------- the kernel
// WP = 1: a dedicated producer warp issues every load (consumers never stall
//         on the ring); 17 warps per TY=32 CTA cap registers at 96.
// WP = 0: the CTA's first thread issues load j + STAGES right after releasing
//         load j; 16 warps allow 128 registers (needed for the R_z >= 6 queues).
// PEER: also store the boundary rows into the neighbours' halo rows (StepParams::peer_*);
// only the edge launch of a peer-connected slab uses it, so the other launches keep
// the register allocation of the plain kernel.
// IO: also the N4 point sets (trace injection into F, receivers gathered from u^{n+1} in the
// store epilogue; StepParams::inj_* / rec_*). Only the default variant of each radius pair is
// compiled with IO; the runtime selects it while a point set is active.
template <typename T, int R, int RZ, int TY, int RPT, int WP, int STAGES, int MINB, bool PEER, int PX, bool IO = false>
__global__ void __launch_bounds__(nthreads(TY, RPT, WP, PX), MINB)
    vti_step_kernel(const __grid_constant__ StepParams<T> P)
{
    using C = Cfg<T, R, RZ, TY>;
    using VP = Vec<T, PX>;
    constexpr bool PACKED = VTI_PACKED_F32 && std::is_same<T, float>::value;
    constexpr int NCONS_WARPS = cons_warps(TY, RPT, PX);
    constexpr int TPR = TX / PX;   // threads per tile row
    constexpr int NQ = C::NQ;
    constexpr int RA = C::RA;
    static_assert(PX == 4 || PX == 2, "4 or 2 x points per thread");
    static_assert((TY * TPR) % (32 * RPT) == 0, "tile rows must split into whole warps");
    static_assert(RA % PX == 0, "x apron must be whole vectors");
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + STAGES * C::STAGE);
    uint64_t *empty = full + STAGES;

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    const bool leader = (WP == 0) && threadIdx.x == 0;
    Producer<T, R, RZ, TY, STAGES> prod;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NCONS_WARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        prefetch_tmap(&P.tm_p);
        prefetch_tmap(&P.tm_q);
        prefetch_tmap(&P.tm_pm);
        prefetch_tmap(&P.tm_qm);
        prefetch_tmap(&P.tm_vx);
        prefetch_tmap(&P.tm_vn);
        prefetch_tmap(&P.tm_vz);
    }
    __syncthreads();
    if constexpr (WP == 1) {
        if (warp == NCONS_WARPS) {   // dedicated producer warp: one lane walks the whole load sequence
            if (lane == 0) {
                prod.start(P);
                while (prod.item < P.items) prod.issue(P, smem, full, empty);
            }
            return;
        }
    } else {
        if (leader) {
            prod.start(P);
            for (int s = 0; s < STAGES; ++s) prod.issue(P, smem, full, empty);   // fill the ring
        }
    }

    // =============== all warps consume: TPR x (TY / RPT) threads, PX x RPT points each ===============
    const int tx = threadIdx.x % TPR;
    const int tg = threadIdx.x / TPR;   // row group: tile rows tg*RPT .. tg*RPT + RPT - 1
    int stage = 0;
    uint32_t phase = 0;

    const int rounds = (P.items + gridDim.x - 1) / gridDim.x;
    for (int item = blockIdx.x, round = 0; item < P.items; item += gridDim.x, ++round) {
        if (round > 0 && P.sync_ctr) {
            // align with every other CTA before the next round (see StepParams::sync_ctr)
            named_bar_sync(1, NCONS_WARPS * 32);
            if (threadIdx.x == 0) {
                const unsigned long long target = P.sync_base + (unsigned long long)round * gridDim.x;
                while (ld_acquire_u64(P.sync_ctr) < target) __nanosleep(64);
            }
            named_bar_sync(1, NCONS_WARPS * 32);
        }
        int x0, y0, kb, ke;
        decode_item<TY>(P, item, x0, y0, kb, ke);
        const int xg = x0 + PX * tx;   // first of this thread's PX columns
        const VP g4 = ldv<PX>(P.gx + xg);
        T gxy[RPT][PX];
        bool store_ok[RPT], src_col[RPT];
        T *pout[RPT], *qout[RPT];
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
            const int yl = y0 + tg * RPT + r;   // local row
            const T gyv = (yl < P.nyl) ? P.gy[yl] : T(0);
#pragma unroll
            for (int c = 0; c < PX; ++c) gxy[r][c] = g4[c] * gyv;
            store_ok[r] = (yl < P.nyl) && (xg < P.nx);
            src_col[r] = P.src_mask != 0 && P.src_j == yl && P.src_i >= xg && P.src_i < xg + PX;
            pout[r] = P.p_out + (long long)yl * P.ys + xg;
            qout[r] = P.q_out + (long long)yl * P.ys + xg;
        }
        const int src_c = P.src_i - xg;
        const int sidx = tg * RPT * TX + PX * tx;   // element offset of row 0 in a stream tile

        VP q[RPT][NQ];
        // prime the queue with q(kb - Rz .. kb + Rz - 1)
#pragma unroll
        for (int t = 0; t < 2 * RZ; ++t) {
            mbar_wait(&full[stage], phase);
            const T *st = reinterpret_cast<const T *>(smem + stage * C::STAGE);
#pragma unroll
            for (int r = 0; r < RPT; ++r) q[r][t] = ldv<PX>(st + C::OFF_Q / C::ES + sidx + r * TX);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[stage]);
            if (leader) prod.issue(P, smem, full, empty);
            if (++stage == STAGES) {
                stage = 0;
                phase ^= 1;
            }
        }

        for (int kbase = kb; kbase < ke; kbase += NQ) {
#pragma unroll
            for (int u = 0; u < NQ; ++u) {
                const int k = kbase + u;
                if (k < ke) {
                    mbar_wait(&full[stage], phase);
                    const T *st = reinterpret_cast<const T *>(smem + stage * C::STAGE);
#pragma unroll
                    for (int r = 0; r < RPT; ++r)
                        q[r][(u + 2 * RZ) % NQ] = ldv<PX>(st + C::OFF_Q / C::ES + sidx + r * TX);   // q^n(k + Rz)
                    const T *ps = st + C::OFF_P / C::ES;
                    // smem row of tile row tg*RPT - R is tg*RPT; x window starts at x0 + 4tx - RA
                    const T *pbase = ps + tg * RPT * C::PW + PX * tx;
                    const T *zr = st + C::OFF_ZR / C::ES;
                    const T gz = zr[NQ];
                    T pn[RPT][PX], qn[RPT][PX];
                    // N4 injection: this thread's entries of the tile-plane (if any), walked in x order
                    bool inj_on = false;
                    const T *inj_base = nullptr;
                    int inj_e[RPT], inj_end[RPT];
                    if constexpr (IO) {
                        if (P.inj_off != nullptr && ps_tile_any(P.inj_off, P.nyl, k, y0, TY)) {
                            const long long row = inj_row_of(P);
                            inj_on = row >= 0 && row < P.inj_nt;
                            inj_base = P.inj_tr + row * P.inj_cols;
                        }
#pragma unroll
                        for (int r = 0; r < RPT; ++r) {
                            inj_e[r] = inj_end[r] = 0;
                            const int yl = y0 + tg * RPT + r;
                            if (inj_on && yl < P.nyl) ps_row_range(P.inj_off, P.inj_ent, P.nyl, k, yl, xg, inj_e[r], inj_end[r]);
                        }
                    }
                    // adds the injected sample at column x (if any) to f_p / f_q, after the source
                    auto inject = [&](int r, int x, T &f_p, T &f_q) {
                        if constexpr (IO) {
                            if (!inj_on) return;
                            while (inj_e[r] < inj_end[r] && P.inj_ent[inj_e[r]].x < x) ++inj_e[r];
                            if (inj_e[r] < inj_end[r] && P.inj_ent[inj_e[r]].x == x) {
                                const T v = inj_base[P.inj_ent[inj_e[r]].y];
                                if (P.inj_mask & 1) f_p = f_p + v;
                                if (P.inj_mask & 2) f_q = f_q + v;
                            }
                        }
                    };
                    if constexpr (PACKED) {
                        // fp32: the same canonical operation order, lane for lane, on packed pairs
                        // (c0,c1), (c2,c3) -- FADD2 / FMUL2 / FFMA2 round each lane exactly like
                        // the scalar instruction, so results are bitwise those of the scalar form
                        // with half the FP instructions. Scalar weights are broadcast operands.
                        constexpr int NPAIR = PX / 2;
                        float2 L2[RPT][NPAIR], pc2[RPT][NPAIR];
#pragma unroll
                        for (int r = 0; r < RPT; ++r) {
                            const float *prow = pbase + (r + R) * C::PW;
                            // (w[i], w[i+1]) of the x window; i odd straddles two register pairs
                            auto wpair = [&](int i) -> float2 {
                                const Vec<float, PX> a4 = ldv<PX>(prow + PX * (i / PX));
                                if (i % PX != PX - 1) return make_float2(a4[i % PX], a4[i % PX + 1]);
                                return make_float2(a4[PX - 1], ldv<PX>(prow + PX * (i / PX + 1))[0]);
                            };
                            const float2 c0 = make_float2(P.cxy[0], P.cxy[0]);
#pragma unroll
                            for (int hp = 0; hp < NPAIR; ++hp) {
                                pc2[r][hp] = wpair(RA + 2 * hp);
                                L2[r][hp] = __fmul2_rn(c0, pc2[r][hp]);
                            }
#pragma unroll
                            for (int l = 1; l <= R; ++l) {
                                const Vec<float, PX> yp = ldv<PX>(pbase + (r + R + l) * C::PW + RA);
                                const Vec<float, PX> ym = ldv<PX>(pbase + (r + R - l) * C::PW + RA);
                                const float2 cl = make_float2(P.cxy[l], P.cxy[l]);
#pragma unroll
                                for (int hp = 0; hp < NPAIR; ++hp) {
                                    const float2 xpair = __fadd2_rn(wpair(RA + 2 * hp + l), wpair(RA + 2 * hp - l));
                                    const float2 ypair = __fadd2_rn(make_float2(yp[2 * hp], yp[2 * hp + 1]),
                                                                    make_float2(ym[2 * hp], ym[2 * hp + 1]));
                                    L2[r][hp] = __ffma2_rn(cl, __fadd2_rn(xpair, ypair), L2[r][hp]);
                                }
                            }
                        }
                        const float2 gz2 = make_float2(gz, gz), ngz2 = make_float2(-gz, -gz);
                        const float2 dt22 = make_float2(P.dt2, P.dt2);
#pragma unroll
                        for (int r = 0; r < RPT; ++r) {
                            const VP pm4 = ldv<PX>(st + C::OFF_PM / C::ES + sidx + r * TX);
                            const VP qm4 = ldv<PX>(st + C::OFF_QM / C::ES + sidx + r * TX);
                            const VP vx4 = ldv<PX>(st + C::OFF_VX / C::ES + sidx + r * TX);
                            const VP vn4 = ldv<PX>(st + C::OFF_VN / C::ES + sidx + r * TX);
                            const VP vz4 = ldv<PX>(st + C::OFF_VZ / C::ES + sidx + r * TX);
                            const bool src_here = src_col[r] && (k == P.src_k);
#pragma unroll
                            for (int hp = 0; hp < NPAIR; ++hp) {
                                const int c = 2 * hp;
                                auto qp = [&](int slot) {
                                    const VP &qq = q[r][slot];
                                    return make_float2(qq[c], qq[c + 1]);
                                };
                                // Eq. 5: ascending m, D = w0 q_{k-Rz}; D = fma(w_m, q_{k-Rz+m}, D)
                                float2 D = __fmul2_rn(make_float2(zr[0], zr[0]), qp(u % NQ));
#pragma unroll
                                for (int m = 1; m < NQ; ++m)
                                    D = __ffma2_rn(make_float2(zr[m], zr[m]), qp((u + m) % NQ), D);
                                const float2 vD = __fmul2_rn(make_float2(vz4[c], vz4[c + 1]), D);
                                float2 Fp = __ffma2_rn(make_float2(vx4[c], vx4[c + 1]), L2[r][hp], vD);
                                float2 Fq = __ffma2_rn(make_float2(vn4[c], vn4[c + 1]), L2[r][hp], vD);
                                if (src_here && (src_c >> 1) == hp) {
                                    const float sv = P.s_table ? P.s_table[P.s_index] : P.s;
                                    if (src_c & 1) {
                                        if (P.src_mask & 1) Fp.y = __fadd_rn(Fp.y, sv);
                                        if (P.src_mask & 2) Fq.y = __fadd_rn(Fq.y, sv);
                                    } else {
                                        if (P.src_mask & 1) Fp.x = __fadd_rn(Fp.x, sv);
                                        if (P.src_mask & 2) Fq.x = __fadd_rn(Fq.x, sv);
                                    }
                                }
                                if constexpr (IO) {
                                    inject(r, xg + c, Fp.x, Fq.x);
                                    inject(r, xg + c + 1, Fp.y, Fq.y);
                                }
                                const float2 gxy2 = make_float2(gxy[r][c], gxy[r][c + 1]);
                                const float2 g = __fmul2_rn(gxy2, gz2);     // (gx gy) gz
                                const float2 ng = __fmul2_rn(gxy2, ngz2);   // -g exactly (sign-symmetric RN)
                                const float2 pc = pc2[r][hp], qc = qp((u + RZ) % NQ);
                                // 2 u^n as u + u (exact, equal to 2 * u)
                                const float2 pnv = __fmul2_rn(g, __ffma2_rn(dt22, Fp, __ffma2_rn(ng, make_float2(pm4[c], pm4[c + 1]), __fadd2_rn(pc, pc))));
                                const float2 qnv = __fmul2_rn(g, __ffma2_rn(dt22, Fq, __ffma2_rn(ng, make_float2(qm4[c], qm4[c + 1]), __fadd2_rn(qc, qc))));
                                pn[r][c] = pnv.x;
                                pn[r][c + 1] = pnv.y;
                                qn[r][c] = qnv.x;
                                qn[r][c + 1] = qnv.y;
                            }
                        }
                    } else {
                        // Eq. 4 / h^2, canonical order: L = c0 p; L = fma(c_l, xpair + ypair, L)
                        T L[RPT][PX];
                        T pc[RPT][PX];   // p^n at the points (2 u^n term)
#pragma unroll
                        for (int r = 0; r < RPT; ++r) {
                            // x window of row r: elements [PX tx, PX tx + PX + 2RA) of smem row r + R, read
                            // as PX-vectors at the point of use (identical loads are CSE'd), so
                            // only the chunks of the current radius stay live
                            const T *prow = pbase + (r + R) * C::PW;
                            auto wx = [&](int i) { return ldv<PX>(prow + PX * (i / PX))[i % PX]; };
#pragma unroll
                            for (int c = 0; c < PX; ++c) {
                                pc[r][c] = wx(RA + c);
                                L[r][c] = P.cxy[0] * pc[r][c];
                            }
#pragma unroll
                            for (int l = 1; l <= R; ++l) {
                                // y neighbours of row r at distance l: smem rows r+R+l, r+R-l at x offset RA
                                const VP yp = ldv<PX>(pbase + (r + R + l) * C::PW + RA);
                                const VP ym = ldv<PX>(pbase + (r + R - l) * C::PW + RA);
#pragma unroll
                                for (int c = 0; c < PX; ++c) {
                                    const T xpair = wx(RA + c + l) + wx(RA + c - l);
                                    const T ypair = yp[c] + ym[c];
                                    L[r][c] = fma_rn(P.cxy[l], xpair + ypair, L[r][c]);
                                }
                            }
                        }
                        // stage data below is read at the point of use (register pressure at
                        // R_z >= 6); the stage is released after the last shared-memory read
#pragma unroll
                        for (int r = 0; r < RPT; ++r) {
                            const VP pm4 = ldv<PX>(st + C::OFF_PM / C::ES + sidx + r * TX);
                            const VP qm4 = ldv<PX>(st + C::OFF_QM / C::ES + sidx + r * TX);
                            const VP vx4 = ldv<PX>(st + C::OFF_VX / C::ES + sidx + r * TX);
                            const VP vn4 = ldv<PX>(st + C::OFF_VN / C::ES + sidx + r * TX);
                            const VP vz4 = ldv<PX>(st + C::OFF_VZ / C::ES + sidx + r * TX);
                            const bool src_here = src_col[r] && (k == P.src_k);
#pragma unroll
                            for (int c = 0; c < PX; ++c) {
                                // Eq. 5: ascending m, D = w0 q_{k-Rz}; D = fma(w_m, q_{k-Rz+m}, D)
                                T D = zr[0] * q[r][u % NQ][c];
#pragma unroll
                                for (int m = 1; m < NQ; ++m) D = fma_rn(zr[m], q[r][(u + m) % NQ][c], D);
                                const T vD = vz4[c] * D;
                                T Fp = fma_rn(vx4[c], L[r][c], vD);
                                T Fq = fma_rn(vn4[c], L[r][c], vD);
                                if (src_here && c == src_c) {
                                    const T sv = P.s_table ? P.s_table[P.s_index] : P.s;
                                    if (P.src_mask & 1) Fp = Fp + sv;
                                    if (P.src_mask & 2) Fq = Fq + sv;
                                }
                                if constexpr (IO) inject(r, xg + c, Fp, Fq);
                                const T g = gxy[r][c] * gz;   // (gx gy) gz
                                pn[r][c] = g * fma_rn(P.dt2, Fp, fma_rn(-g, pm4[c], T(2) * pc[r][c]));
                                qn[r][c] = g * fma_rn(P.dt2, Fq, fma_rn(-g, qm4[c], T(2) * q[r][(u + RZ) % NQ][c]));
                            }
                        }
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty[stage]);
                    if (leader) prod.issue(P, smem, full, empty);
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                    if constexpr (IO) record_points<T, RPT, PX>(P, k, y0, TY, y0 + tg * RPT, xg, pn, qn);
#pragma unroll
                    for (int r = 0; r < RPT; ++r) {
                        if (store_ok[r]) {
                            const long long off = (long long)k * P.zs;
                            stv(pout[r] + off, pn[r]);
                            stv(qout[r] + off, qn[r]);
                            if constexpr (PEER) {
                                // the neighbours' halo rows, straight over NVLink (edge tile rows
                                // only; a row goes to both sides when nyl < 2R)
                                const int yl = y0 + tg * RPT + r;
                                if (P.peer_lo != nullptr && yl < R)
                                    stv(P.peer_lo + (long long)k * P.peer_zs_lo + (long long)yl * P.ys + xg, pn[r]);
                                if (P.peer_hi != nullptr && yl >= P.nyl - R)
                                    stv(P.peer_hi + (long long)k * P.peer_zs_hi +
                                             (long long)(yl - (P.nyl - R)) * P.ys + xg,
                                         pn[r]);
                            }
                        }
                    }
                }
            }
        }
        if constexpr (PEER) {
            if (P.edge_ctr != nullptr && item < P.edge_items) {
                // fused multi-GPU step: this edge item's stores (own rows and the neighbours'
                // halo rows) are done; the last edge item to finish raises the neighbours' flags
                named_bar_sync(1, NCONS_WARPS * 32);
                if (threadIdx.x == 0) {
                    __threadfence_system();
                    if (atomicAdd(P.edge_ctr, 1ULL) + 1 == P.edge_target) {
                        __threadfence_system();
#pragma unroll
                        for (int i = 0; i < 4; ++i)
                            if (P.sig[i] != nullptr)
                                asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(P.sig[i]), "r"(P.sig_val[i])
                                             : "memory");
                    }
                }
            }
        }
        if (P.sync_ctr && round < rounds - 1) {
            // every CTA arrives once per non-final round, whether or not it has another item
            named_bar_sync(1, NCONS_WARPS * 32);
            if (threadIdx.x == 0) atomicAdd(P.sync_ctr, 1ULL);
        }
    }
}

}  // namespace vti
