// vti_adjoint.cu -- the adjoint (transpose) recurrence of the VTI step (the
// backward leg of adjoint-state FWI; PAPER.md l.18-19 names FWI and RTM as the propagator's
// users). The forward step X^{n+1} = M X^n, M = [[g(2 + dt^2 A), -g^2], [I, 0]] with
//   A u = (vx2 L p + vz2 D q, vn2 L p + vz2 D q)            (Eqs. 1-2, 4-5)
// has the transpose recurrence, in the damping-scaled adjoint variable psi = g a,
//   psi^{m-1} = g (2 psi^m - g psi^{m+1} + dt^2 (A^T psi^m + inj)),
//   A^T psi = (L (vx2 psi_p + vn2 psi_q), D^T (vz2 (psi_p + psi_q))),
// L symmetric on the zero exterior and (D^T y)_k = sum_m w^z[k+Rz-m][m] y_{k+Rz-m}. The
// coefficient fields act BEFORE the derivatives here: s1 = vx2 psi_p + vn2 psi_q is needed on the
// R_xy apron of every tile, s2 = vz2 (psi_p + psi_q) along z. Canonical operation order (bitwise
// equal to the oracle's vto_adjoint_ex): s1 = fma(vx2, psi_p, vn2*psi_q), s2 = vz2*(psi_p + psi_q);
// L = c0 s1; L = fma(c_l, (x+ + x-) + (y+ + y-), L); DT = 0, DT = fma(w[k'][m], s2(k'), DT) for
// m = 0..2Rz, k' = k+Rz-m inside the grid; F_p = L (+ inj), F_q = DT (+ inj);
// psi^{m-1} = g*fma(dt2, F, fma(-g, psi^{m+1}, 2 psi^m)).
//
// Forms (adj_form picks one; every form gives the same bits):
//   * TMA one-pass (k_adj_tma): per plane, the halo'd psi_p, psi_q, vx2, vn2 boxes arrive by TMA
//     and the CTA forms the s1 tile in shared memory; 36 B/pt in fp32 like the forward step.
//   * TMA two-pass (k_adj_s1, then k_adj_tma2): s1 in HBM, read back as one halo'd box; chained
//     across the steps of a call (each step also writes the next step's s1: 44 B/pt, one launch
//     per step after the first). Y-slab groups run this form with the neighbours' s1 rows
//     copied into each slab's halo between steps.
//   * cp.async forms (k_adj_fused one-pass; k_adj_prep + k_adj_step two-pass): the round-2 first
//     versions, for radii without a TMA entry and as A/B baselines (VTI_ADJ_TMA=0).
#include "vti_internal.h"

namespace {

template <typename T>
__device__ __forceinline__ T fma_x(T a, T b, T c);
template <>
__device__ __forceinline__ float fma_x<float>(float a, float b, float c) { return __fmaf_rn(a, b, c); }
template <>
__device__ __forceinline__ double fma_x<double>(double a, double b, double c) { return __fma_rn(a, b, c); }

// s1 = fma(vx2, psi_p, vn2*psi_q), s2 = vz2*(psi_p + psi_q) over the interior (halo untouched = 0)
template <typename T>
__global__ void k_adj_prep(const T *__restrict__ pp, const T *__restrict__ pq, const T *__restrict__ vx2,
                           const T *__restrict__ vn2, const T *__restrict__ vz2, T *__restrict__ s1,
                           T *__restrict__ s2, int nx, int nyl, int nz, long long ys, long long zs)
{
    const int64_t n = (int64_t)nz * nyl * nx;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const int x = (int)(t % nx);
        const int64_t r = t / nx;
        const int y = (int)(r % nyl);
        const int k = (int)(r / nyl);
        const int64_t a = y * ys + k * zs + x;
        const T p = pp[a], q = pq[a];
        s1[a] = fma_x<T>(vx2[a], p, vn2[a] * q);
        s2[a] = vz2[a] * (p + q);
    }
}

template <typename T>
struct AdjParams {
    const T *s1, *s2;              // interior views (row 0, plane 0) (two-pass form)
    const T *vx, *vn, *vz;         // model interior views (one-pass form)
    const T *pc, *qc;              // psi^m
    T *po, *qo;                    // psi^{m+1} in, psi^{m-1} out (in place)
    T *s1o;                        // chained TMA two-pass form: s1 of psi^{m-1} out (interior view)
    const T *zrow;                 // [nz][zrow_stride]: w^z[k][0..2Rz], gz[k]
    int zrow_stride;
    const T *gx, *gy;
    T cxy[MAX_R + 1];
    T dt2;
    int nx, nyl, nz;
    long long ys, zs;
    // N4 point sets (nullable): injection into F after the operator, receivers of psi^{m-1}
    const int *inj_off;
    const int2 *inj_ent;
    const T *inj_row;              // this step's trace row, or NULL
    int inj_mask;
    const int *rec_off;
    const int2 *rec_ent;
    T *rec_row;                    // this step's receiver row [n][nf], or NULL
    int rec_mask;
    int y_lo, y_hi;                // rows of s1 the two-pass stencil may read: [y_lo, y_hi) (local rows;
                                   // beyond [0, nyl) the neighbours' rows copied into the halo)
};

// the column of the CSR entry for point x of row (k, yl), or -1
__device__ __forceinline__ int ps_lookup(const int *off, const int2 *ent, int nyl, int k, int yl, int x)
{
    const long long b = (long long)k * nyl + yl;
    int lo = off[b], hi = off[b + 1];
    if (lo == hi) return -1;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (ent[mid].x < x) lo = mid + 1;
        else hi = mid;
    }
    return (lo < off[b + 1] && ent[lo].x == x) ? lo : -1;
}

// The stencils and update, marching z: one CTA per (64 x 8 tile, z-chunk), 16 x 8 threads
// of 4 x points each (the forward kernel's mapping). Per plane the s1 tile with its R_xy apron
// is staged in shared memory (zero outside the slab), s2 marches in a (2R_z+1)-deep register
// queue, and D^T takes the transposed weight diagonal w^z[k+Rz-m][m] from the plane table.
constexpr int ADJ_TY = 8;
constexpr int ADJ_ZCHUNK = 64;

template <typename T, int R, int RZ>
__global__ void __launch_bounds__(16 * ADJ_TY) k_adj_step(const AdjParams<T> A, int ntx, int nty)
{
    constexpr int NQ = 2 * RZ + 1;
    constexpr int RA = (R + 3) / 4 * 4;   // apron rounded to whole 4-vectors
    constexpr int PW = 64 + 2 * RA, PH = ADJ_TY + 2 * R;
    __shared__ __align__(16) T tile[2][PH * PW];
    const int b = blockIdx.x;
    const int itx = b % ntx, ity = (b / ntx) % nty, izc = b / (ntx * nty);
    const int x0 = itx * 64, y0 = ity * ADJ_TY;
    const int kb = izc * ADJ_ZCHUNK, ke = min(A.nz, kb + ADJ_ZCHUNK);
    const int tx = threadIdx.x & 15, tg = threadIdx.x >> 4;
    const int xg = x0 + 4 * tx, yl = y0 + tg;
    const bool own = xg < A.nx && yl < A.nyl;
    // s2 column queue: slot m holds plane k - RZ + m
    T q[NQ][4];
    auto load4 = [&](const T *base, int k, T (&v)[4]) {   // 16-byte loads (rows are padded to 32 points)
#pragma unroll
        for (int c = 0; c < 4; ++c) v[c] = T(0);
        if (!own || k < 0 || k >= A.nz) return;
        const V4<T> w = ldv<4>(base + (int64_t)yl * A.ys + (int64_t)k * A.zs + xg);
#pragma unroll
        for (int c = 0; c < 4; ++c) v[c] = (xg + c < A.nx) ? w[c] : T(0);
    };
#pragma unroll
    for (int m = 0; m < NQ - 1; ++m) load4(A.s2, kb - RZ + m, q[m + 1]);
    const T gy = own ? A.gy[yl] : T(0);
    // s1 tile of plane k -> buffer (k & 1) with cp.async (out-of-slab elements zero-filled), so
    // plane k+1 is in flight while plane k is computed
    auto stage = [&](int k) {
        T *dst = tile[k & 1];
        for (int e = threadIdx.x; e < PH * PW; e += 16 * ADJ_TY) {
            const int r = e / PW, c = e % PW;
            const int yy = y0 - R + r, xx = x0 - RA + c;
            const bool in = yy >= A.y_lo && yy < A.y_hi && xx >= 0 && xx < A.nx;
            const T *src = in ? A.s1 + (int64_t)yy * A.ys + (int64_t)k * A.zs + xx : A.s1;
            const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst + e);
            if constexpr (sizeof(T) == 8)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(in ? 8 : 0) : "memory");
            else
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(d), "l"(src), "r"(in ? 4 : 0) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    if (kb < ke) stage(kb);
    for (int k = kb; k < ke; ++k) {
#pragma unroll
        for (int m = 0; m < NQ - 1; ++m)
#pragma unroll
            for (int c = 0; c < 4; ++c) q[m][c] = q[m + 1][c];
        load4(A.s2, k + RZ, q[NQ - 1]);
        __syncthreads();   // every thread is done with buffer (k+1) & 1 (plane k-1)
        if (k + 1 < ke) {
            stage(k + 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");   // plane k landed
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();   // plane k visible to every thread
        if (own) {
            const T *row = tile[k & 1] + (tg + R) * PW + RA + 4 * tx;   // this thread's first point
            T L[4], DT[4], Fp[4], Fq[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                // L(s1), canonical pairing (x pair + y pair); zero exterior in the staged tile
                L[c] = A.cxy[0] * row[c];
#pragma unroll
                for (int l = 1; l <= R; ++l)
                    L[c] = fma_x<T>(A.cxy[l], (row[c + l] + row[c - l]) + (row[c + l * PW] + row[c - l * PW]), L[c]);
                // D^T(s2): ascending m over planes k' = k + RZ - m inside the grid
                DT[c] = T(0);
            }
#pragma unroll
            for (int m = 0; m < NQ; ++m) {
                const int kk = k + RZ - m;
                if (kk < 0 || kk >= A.nz) continue;
                const T w = A.zrow[(int64_t)kk * A.zrow_stride + m];
#pragma unroll
                for (int c = 0; c < 4; ++c) DT[c] = fma_x<T>(w, q[NQ - 1 - m][c], DT[c]);
            }
            const T gz = A.zrow[(int64_t)k * A.zrow_stride + NQ];
            const int64_t a0 = (int64_t)yl * A.ys + (int64_t)k * A.zs + xg;
            const V4<T> po4 = ldv<4>(A.po + a0), qo4 = ldv<4>(A.qo + a0), gx4 = ldv<4>(A.gx + xg);
            const V4<T> pc4 = ldv<4>(A.pc + a0), qc4 = ldv<4>(A.qc + a0);
            T pn[4], qn[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const int i = xg + c;
                Fp[c] = L[c];
                Fq[c] = DT[c];
                if (A.inj_row != nullptr && i < A.nx) {
                    const int e = ps_lookup(A.inj_off, A.inj_ent, A.nyl, k, yl, i);
                    if (e >= 0) {
                        const T v = A.inj_row[A.inj_ent[e].y];
                        if (A.inj_mask & 1) Fp[c] = Fp[c] + v;
                        if (A.inj_mask & 2) Fq[c] = Fq[c] + v;
                    }
                }
                const T g = (gx4[c] * gy) * gz;
                pn[c] = g * fma_x<T>(A.dt2, Fp[c], fma_x<T>(-g, po4[c], T(2) * pc4[c]));
                qn[c] = g * fma_x<T>(A.dt2, Fq[c], fma_x<T>(-g, qo4[c], T(2) * qc4[c]));
            }
            if (xg + 4 <= A.nx) {   // whole vector inside the row
                stv(A.po + a0, pn);
                stv(A.qo + a0, qn);
            } else {
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    if (xg + c < A.nx) {
                        A.po[a0 + c] = pn[c];
                        A.qo[a0 + c] = qn[c];
                    }
            }
            if (A.rec_row != nullptr) {   // receivers of psi^{m-1} (duplicates allowed: every entry)
                const long long rb = (long long)k * A.nyl + yl;
                const int nf = (A.rec_mask & 1) + ((A.rec_mask >> 1) & 1);
                for (int e = A.rec_off[rb]; e < A.rec_off[rb + 1]; ++e) {
                    const int c = A.rec_ent[e].x - xg;
                    if (c < 0 || c >= 4) continue;
                    T vp = pn[0], vq = qn[0];
#pragma unroll
                    for (int cc = 1; cc < 4; ++cc)
                        if (c == cc) {
                            vp = pn[cc];
                            vq = qn[cc];
                        }
                    T *o = A.rec_row + (int64_t)A.rec_ent[e].y * nf;
                    if (A.rec_mask & 1) *o++ = vp;
                    if (A.rec_mask & 2) *o = vq;
                }
            }
        }
    }
}

// One-pass form: the coefficient products are formed inside the stencil kernel, so a step
// reads psi and the model once (36 B/pt like the forward step instead of 60 over two passes).
// Per plane, cp.async stages psi_p, psi_q, vx2, vn2 tiles with the R_xy apron (double-buffered,
// zero-filled outside the slab), the CTA forms the s1 tile in shared memory, and each thread
// forms s2 = vz2 (psi_p + psi_q) of plane k + R_z for its register queue. Same arithmetic as
// k_adj_prep + k_adj_step, so the same bits.
template <typename T, int R, int RZ, int TY>
struct AdjFusedCfg {
    static constexpr int RA = (R + 3) / 4 * 4;
    static constexpr int PW = 64 + 2 * RA, PH = TY + 2 * R, TE = PH * PW;
    static constexpr int VEC = 16 / (int)sizeof(T);   // elements per 16-byte cp.async
    static constexpr int SMEM = 9 * TE * (int)sizeof(T);   // [2][4][TE] inputs + [TE] s1
};

template <typename T, int R, int RZ, int TY>
__global__ void __launch_bounds__(16 * TY) k_adj_fused(const AdjParams<T> A, int ntx, int nty)
{
    using F = AdjFusedCfg<T, R, RZ, TY>;
    constexpr int NQ = 2 * RZ + 1, RA = F::RA, PW = F::PW, PH = F::PH, TE = F::TE, VEC = F::VEC;
    constexpr int NT = 16 * TY;
    extern __shared__ __align__(16) uint8_t adj_smem[];
    T *inb = reinterpret_cast<T *>(adj_smem);   // [2][4][TE]: psi_p, psi_q, vx2, vn2
    T *s1t = inb + 8 * TE;
    const int b = blockIdx.x;
    const int itx = b % ntx, ity = (b / ntx) % nty, izc = b / (ntx * nty);
    const int x0 = itx * 64, y0 = ity * TY;
    const int kb = izc * ADJ_ZCHUNK, ke = min(A.nz, kb + ADJ_ZCHUNK);
    const int tx = threadIdx.x & 15, tg = threadIdx.x >> 4;
    const int xg = x0 + 4 * tx, yl = y0 + tg;
    const bool own = xg < A.nx && yl < A.nyl;
    const T *src4[4] = {A.pc, A.qc, A.vx, A.vn};
    auto stage = [&](int k) {
        T *dst = inb + (k & 1) * 4 * TE;
        for (int e = threadIdx.x; e < TE / VEC; e += NT) {
            const int r = (e * VEC) / PW, c = (e * VEC) % PW;
            const int yy = y0 - R + r, xx = x0 - RA + c;
            const bool rowin = yy >= 0 && yy < A.nyl;
            // valid bytes of this 16-byte chunk (zero fill beyond nx and outside the slab)
            const int nvalid = (!rowin || xx >= A.nx || xx + VEC <= 0) ? 0 : min(VEC, A.nx - xx);
            const bool whole_left = xx >= 0;   // chunks never straddle x = 0 (x0 - RA is a multiple of 4)
            const int bytes = whole_left ? nvalid * (int)sizeof(T) : 0;
            const int64_t off = rowin && whole_left ? (int64_t)yy * A.ys + (int64_t)k * A.zs + xx : 0;
#pragma unroll
            for (int f = 0; f < 4; ++f) {
                const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst + f * TE + e * VEC);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src4[f] + off), "r"(bytes)
                             : "memory");
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    // s2 = vz2 (psi_p + psi_q) of plane k at this thread's 4 points (0 outside the grid)
    auto s2_of = [&](int k, T (&v)[4]) {   // 16-byte loads (rows are padded to 32 points)
#pragma unroll
        for (int c = 0; c < 4; ++c) v[c] = T(0);
        if (!own || k < 0 || k >= A.nz) return;
        const int64_t a = (int64_t)yl * A.ys + (int64_t)k * A.zs + xg;
        const V4<T> vz = ldv<4>(A.vz + a), pp = ldv<4>(A.pc + a), qq = ldv<4>(A.qc + a);
#pragma unroll
        for (int c = 0; c < 4; ++c)
            if (xg + c < A.nx) v[c] = vz[c] * (pp[c] + qq[c]);
    };
    T q[NQ][4];
#pragma unroll
    for (int m = 0; m < NQ - 1; ++m) s2_of(kb - RZ + m, q[m + 1]);
    const T gy = own ? A.gy[yl] : T(0);
    if (kb < ke) stage(kb);
    for (int k = kb; k < ke; ++k) {
#pragma unroll
        for (int m = 0; m < NQ - 1; ++m)
#pragma unroll
            for (int c = 0; c < 4; ++c) q[m][c] = q[m + 1][c];
        s2_of(k + RZ, q[NQ - 1]);
        __syncthreads();   // every thread is done with s1t and with buffer (k+1) & 1 (plane k-1)
        if (k + 1 < ke) {
            stage(k + 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");   // plane k landed
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();   // plane k inputs visible to every thread
        const T *pin = inb + (k & 1) * 4 * TE;
        for (int e = threadIdx.x; e < TE; e += NT)   // s1 = fma(vx2, psi_p, vn2 * psi_q) with the apron
            s1t[e] = fma_x<T>(pin[2 * TE + e], pin[e], pin[3 * TE + e] * pin[TE + e]);
        __syncthreads();
        if (own) {
            const int ctr = (tg + R) * PW + RA + 4 * tx;   // this thread's first point in the tile
            const T *row = s1t + ctr;
            T L[4], DT[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                L[c] = A.cxy[0] * row[c];
#pragma unroll
                for (int l = 1; l <= R; ++l)
                    L[c] = fma_x<T>(A.cxy[l], (row[c + l] + row[c - l]) + (row[c + l * PW] + row[c - l * PW]), L[c]);
                DT[c] = T(0);
            }
#pragma unroll
            for (int m = 0; m < NQ; ++m) {
                const int kk = k + RZ - m;
                if (kk < 0 || kk >= A.nz) continue;
                const T w = A.zrow[(int64_t)kk * A.zrow_stride + m];
#pragma unroll
                for (int c = 0; c < 4; ++c) DT[c] = fma_x<T>(w, q[NQ - 1 - m][c], DT[c]);
            }
            const T gz = A.zrow[(int64_t)k * A.zrow_stride + NQ];
            const int64_t a0 = (int64_t)yl * A.ys + (int64_t)k * A.zs + xg;
            const V4<T> po4 = ldv<4>(A.po + a0), qo4 = ldv<4>(A.qo + a0), gx4 = ldv<4>(A.gx + xg);
            const V4<T> pc4 = ldv<4>(pin + ctr), qc4 = ldv<4>(pin + TE + ctr);
            T pn[4], qn[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const int i = xg + c;
                T Fp = L[c], Fq = DT[c];
                if (A.inj_row != nullptr && i < A.nx) {
                    const int e = ps_lookup(A.inj_off, A.inj_ent, A.nyl, k, yl, i);
                    if (e >= 0) {
                        const T v = A.inj_row[A.inj_ent[e].y];
                        if (A.inj_mask & 1) Fp = Fp + v;
                        if (A.inj_mask & 2) Fq = Fq + v;
                    }
                }
                const T g = (gx4[c] * gy) * gz;
                pn[c] = g * fma_x<T>(A.dt2, Fp, fma_x<T>(-g, po4[c], T(2) * pc4[c]));
                qn[c] = g * fma_x<T>(A.dt2, Fq, fma_x<T>(-g, qo4[c], T(2) * qc4[c]));
            }
            if (xg + 4 <= A.nx) {   // whole vector inside the row
                stv(A.po + a0, pn);
                stv(A.qo + a0, qn);
            } else {
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    if (xg + c < A.nx) {
                        A.po[a0 + c] = pn[c];
                        A.qo[a0 + c] = qn[c];
                    }
            }
            if (A.rec_row != nullptr) {   // receivers of psi^{m-1} (duplicates allowed: every entry)
                const long long rb = (long long)k * A.nyl + yl;
                const int nf = (A.rec_mask & 1) + ((A.rec_mask >> 1) & 1);
                for (int e = A.rec_off[rb]; e < A.rec_off[rb + 1]; ++e) {
                    const int c = A.rec_ent[e].x - xg;
                    if (c < 0 || c >= 4) continue;
                    T vp = pn[0], vq = qn[0];
#pragma unroll
                    for (int cc = 1; cc < 4; ++cc)
                        if (c == cc) {
                            vp = pn[cc];
                            vq = qn[cc];
                        }
                    T *o = A.rec_row + (int64_t)A.rec_ent[e].y * nf;
                    if (A.rec_mask & 1) *o++ = vp;
                    if (A.rec_mask & 2) *o = vq;
                }
            }
        }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
}

template <typename T, int TY>
static vti_status launch_adj_fused_ty(vti_s *h, const AdjParams<T> &A)
{
    const int ntx = (h->cfg.nx + 63) / 64, nty = (h->nyl + TY - 1) / TY;
    const int nzc = (h->cfg.nz + ADJ_ZCHUNK - 1) / ADJ_ZCHUNK;
    const int R = h->R, RZ = h->RZ;
#define ADJF_CASE(r, rz)                                                                                   \
    if (R == r && RZ == rz) {                                                                              \
        const int smem = AdjFusedCfg<T, r, rz, TY>::SMEM;                                                  \
        CU(h, cudaFuncSetAttribute((const void *)k_adj_fused<T, r, rz, TY>,                                \
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, smem));                    \
        k_adj_fused<T, r, rz, TY><<<ntx * nty * nzc, 16 * TY, smem, h->stream>>>(A, ntx, nty);            \
        CU(h, cudaGetLastError());                                                                         \
        return VTI_OK;                                                                                     \
    }
    ADJF_CASE(4, 4)
    ADJF_CASE(8, 4)
    ADJF_CASE(6, 6)
    ADJF_CASE(12, 8)
#undef ADJF_CASE
    return fail(h, VTI_E_UNSUPPORTED, "no adjoint kernel for (%d, %d)", R, RZ);
}

// fp32: 16-row tiles (env VTI_ADJ_TY=8 for 8); fp64: 8-row tiles (shared memory)
template <typename T>
static vti_status launch_adj_fused(vti_s *h, const AdjParams<T> &A)
{
    static const int ty = getenv("VTI_ADJ_TY") ? atoi(getenv("VTI_ADJ_TY")) : 16;
    if (sizeof(T) == 4 && ty == 16) return launch_adj_fused_ty<T, 16>(h, A);
    return launch_adj_fused_ty<T, 8>(h, A);
}

template <typename T>
static vti_status launch_adj_step(vti_s *h, const AdjParams<T> &A, int grid)
{
    const int R = h->R, RZ = h->RZ;
    const int ntx = (h->cfg.nx + 63) / 64, nty = (h->nyl + ADJ_TY - 1) / ADJ_TY;
    const int nzc = (h->cfg.nz + ADJ_ZCHUNK - 1) / ADJ_ZCHUNK;
    (void)grid;
#define ADJ_CASE(r, rz)                                                                          \
    if (R == r && RZ == rz) {                                                                    \
        k_adj_step<T, r, rz><<<ntx * nty * nzc, 16 * ADJ_TY, 0, h->stream>>>(A, ntx, nty);       \
        CU(h, cudaGetLastError());                                                               \
        return VTI_OK;                                                                           \
    }
    ADJ_CASE(4, 4)
    ADJ_CASE(8, 4)
    ADJ_CASE(6, 6)
    ADJ_CASE(12, 8)
#undef ADJ_CASE
    return fail(h, VTI_E_UNSUPPORTED, "no adjoint kernel for (%d, %d)", R, RZ);
}

// ---------------------------------------------------------------- TMA form (single slab default)
// The forward kernel's structure applied to the transpose. A persistent CTA walks (64 x TY tile,
// z-chunk) items. A producer warp streams, per plane k, into an mbarrier ring
// (cp.async.bulk.tensor, zero fill outside the grid):
//   * the halo'd psi_p, psi_q, vx2, vn2 boxes of plane k (the s1 apron);
//   * the interior psi_p, psi_q, vz2 boxes of plane k + Rz (the s2 queue front);
//   * the interior psi^{m+1} boxes of plane k;
//   * plane k's row of the transposed z weights wT[k][m] = w^z[k+Rz-m][m] (0 outside the grid).
// Consumers form the s1 tile with its apron in shared memory (double-buffered: one named barrier
// per plane), push s2(k + Rz) into a (2Rz+1)-deep register queue, take their own psi^m, psi^{m+1}
// and D^T, release the stage, then apply L to s1 and update. DRAM: psi^m (2), model (3) and
// psi^{m+1} (2) read once, psi^{m-1} (2) written = 36 B/pt in fp32 like the forward step; the
// aprons and the Rz-ahead psi boxes come back from L2. Same canonical arithmetic as k_adj_prep +
// k_adj_step (a skipped out-of-grid D^T term equals an fma with weight 0 and s2 = 0 bit for bit:
// DT starts at +0 and +0 + (+-0) = +0), so the same bits as the oracle.
template <typename T, int R, int RZ, int TY, int ST, int PX = 4>
struct AdjTmaCfg {
    static constexpr int ES = (int)sizeof(T);
    static constexpr int RA = (R + 3) / 4 * 4;
    static constexpr int PW = TX + 2 * RA, PH = TY + 2 * R, TE = PW * PH;
    static constexpr int NQ = 2 * RZ + 1;
    static constexpr int ZROW = ((NQ + 1 + 3) / 4) * 4;   // = the forward table's row (Cfg::ZROW)
    static constexpr int P_BYTES = align128(TE * ES);
    static constexpr int S_BYTES = TX * TY * ES;
    static constexpr int OFF_HP = 0, OFF_HQ = P_BYTES, OFF_HX = 2 * P_BYTES, OFF_HN = 3 * P_BYTES;
    static constexpr int OFF_IP = 4 * P_BYTES, OFF_IQ = OFF_IP + S_BYTES, OFF_VZ = OFF_IQ + S_BYTES;
    static constexpr int OFF_OP = OFF_VZ + S_BYTES, OFF_OQ = OFF_OP + S_BYTES, OFF_ZR = OFF_OQ + S_BYTES;
    static constexpr int STAGE = align128(OFF_ZR + ZROW * ES);
    static constexpr uint32_t FULL_TX = 4 * TE * ES + 5 * S_BYTES + ZROW * ES;
    static constexpr uint32_t PRIME_TX = 3 * S_BYTES;
    static constexpr int OFF_S1 = ST * STAGE;               // [2][P_BYTES]: s1 of planes k (even / odd)
    static constexpr int OFF_BAR = OFF_S1 + 2 * P_BYTES;
    static constexpr int SMEM = OFF_BAR + 2 * ST * 8;
    static constexpr int TPR = TX / PX;                     // consumer threads per tile row
    static constexpr int NCONS = TPR * TY;                  // consumer threads, PX x points each
    static constexpr int NT = NCONS + 32;                   // + the producer warp
    static_assert(PW % 4 == 0 && PW <= 256 && PH <= 256, "TMA box");
};

template <typename T>
struct AdjTmaParams {
    CUtensorMap tm[9];   // halo'd psi_p^m, psi_q^m, vx2, vn2; interior psi_p^m, psi_q^m, vz2, psi_p^{m+1}, psi_q^{m+1}
    AdjParams<T> A;      // A.zrow: the transposed rows [nz][ZROW] (w^T[k][0..2Rz], gz[k])
    int ntx, nty, zchunk, items;
};

template <int TY, typename T>
__device__ __forceinline__ void adj_item(const AdjTmaParams<T> &P, int item, int &x0, int &y0, int &kb, int &ke)
{
    const int tx = item % P.ntx, r = item / P.ntx;
    x0 = tx * TX;
    y0 = (r % P.nty) * TY;
    kb = (r / P.nty) * P.zchunk;
    ke = min(P.A.nz, kb + P.zchunk);
}

template <typename T, int R, int RZ, int TY, int ST, int PX, bool IO>
__global__ void __launch_bounds__(AdjTmaCfg<T, R, RZ, TY, ST, PX>::NT, 1)
    k_adj_tma(const __grid_constant__ AdjTmaParams<T> P)
{
    using C = AdjTmaCfg<T, R, RZ, TY, ST, PX>;
    using VP = Vec<T, PX>;
    constexpr int NQ = C::NQ, RA = C::RA, PW = C::PW, ES = C::ES, NCONS = C::NCONS, TPR = C::TPR;
    constexpr bool SHIFT = NQ > 9;   // i-cache: NQ unrolled copies of a deep body miss (ncu: no_instructions)
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + C::OFF_BAR);
    uint64_t *empty = full + ST;
    const AdjParams<T> &A = P.A;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < ST; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NCONS / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        for (int i = 0; i < 9; ++i) prefetch_tmap(&P.tm[i]);
    }
    __syncthreads();
    // programmatic dependent launch: the prologue above overlaps the previous kernel's tail; every
    // global access below waits for its completion (a no-op without the launch attribute)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    int stage = 0;
    uint32_t phase = 0;
    if (warp == NCONS / 32) {   // producer: one lane walks the load sequence of every item
        if (lane != 0) return;
        for (int item = blockIdx.x; item < P.items; item += gridDim.x) {
            int x0, y0, kb, ke;
            adj_item<TY>(P, item, x0, y0, kb, ke);
            const int nload = (ke - kb) + 2 * RZ;
            for (int t = 0; t < nload; ++t) {
                mbar_wait(&empty[stage], phase ^ 1);
                uint8_t *st = smem + stage * C::STAGE;
                uint64_t *bar = &full[stage];
                if (t < 2 * RZ) {   // priming: s2 inputs of planes kb - Rz .. kb + Rz - 1
                    const int kk = kb - RZ + t;
                    mbar_arrive_expect_tx(bar, C::PRIME_TX);
                    tma_load_3d(st + C::OFF_IP, &P.tm[4], x0, y0, kk, bar);
                    tma_load_3d(st + C::OFF_IQ, &P.tm[5], x0, y0, kk, bar);
                    tma_load_3d(st + C::OFF_VZ, &P.tm[6], x0, y0, kk, bar);
                } else {
                    const int k = kb + t - 2 * RZ;
                    mbar_arrive_expect_tx(bar, C::FULL_TX);
                    // halo'd views: row y0 of the view is local row y0 - R
                    tma_load_3d(st + C::OFF_HP, &P.tm[0], x0 - RA, y0, k, bar);
                    tma_load_3d(st + C::OFF_HQ, &P.tm[1], x0 - RA, y0, k, bar);
                    tma_load_3d(st + C::OFF_HX, &P.tm[2], x0 - RA, y0, k, bar);
                    tma_load_3d(st + C::OFF_HN, &P.tm[3], x0 - RA, y0, k, bar);
                    tma_load_3d(st + C::OFF_IP, &P.tm[4], x0, y0, k + RZ, bar);
                    tma_load_3d(st + C::OFF_IQ, &P.tm[5], x0, y0, k + RZ, bar);
                    tma_load_3d(st + C::OFF_VZ, &P.tm[6], x0, y0, k + RZ, bar);
                    tma_load_3d(st + C::OFF_OP, &P.tm[7], x0, y0, k, bar);
                    tma_load_3d(st + C::OFF_OQ, &P.tm[8], x0, y0, k, bar);
                    bulk_load(st + C::OFF_ZR, A.zrow + (size_t)k * C::ZROW, C::ZROW * ES, bar);
                }
                if (++stage == ST) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
        return;
    }

    // consumers: TPR x TY threads, PX consecutive x points each
    const int tx = threadIdx.x % TPR, tg = threadIdx.x / TPR;
    const int sidx = tg * TX + PX * tx;   // this thread's first point in an interior box
    T *s1buf = reinterpret_cast<T *>(smem + C::OFF_S1);
    int par = 0;
    for (int item = blockIdx.x; item < P.items; item += gridDim.x) {
        int x0, y0, kb, ke;
        adj_item<TY>(P, item, x0, y0, kb, ke);
        const int xg = x0 + PX * tx, yl = y0 + tg;
        const bool own = xg < A.nx && yl < A.nyl;
        const T gy = yl < A.nyl ? A.gy[yl] : T(0);
        const VP gx4 = ldv<PX>(A.gx + xg);
        T q[NQ][PX];   // slot (u + j) % NQ holds s2 of plane k - Rz + j
        auto push_s2 = [&](const T *st, T (&v)[PX]) {
            const VP ip = ldv<PX>(st + C::OFF_IP / ES + sidx), iq = ldv<PX>(st + C::OFF_IQ / ES + sidx);
            const VP vz = ldv<PX>(st + C::OFF_VZ / ES + sidx);
#pragma unroll
            for (int c = 0; c < PX; ++c) v[c] = vz[c] * (ip[c] + iq[c]);
        };
#pragma unroll
        for (int t = 0; t < 2 * RZ; ++t) {
            mbar_wait(&full[stage], phase);
            push_s2(reinterpret_cast<const T *>(smem + stage * C::STAGE), q[SHIFT ? t + 1 : t]);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[stage]);
            if (++stage == ST) {
                stage = 0;
                phase ^= 1;
            }
        }
        // plane k; slot (u + j) % NQ of the queue holds s2 of plane k - Rz + j
        auto plane = [&](const int k, const int u) {
            mbar_wait(&full[stage], phase);
            const T *st = reinterpret_cast<const T *>(smem + stage * C::STAGE);
            // s1 = fma(vx2, psi_p, vn2 * psi_q) over the whole box (apron included)
            T *s1 = s1buf + par * (C::P_BYTES / ES);
            par ^= 1;
            for (int e = threadIdx.x; e < C::TE / 4; e += NCONS) {
                const V4<T> a = ldv<4>(st + C::OFF_HP / ES + 4 * e), b = ldv<4>(st + C::OFF_HQ / ES + 4 * e);
                const V4<T> x = ldv<4>(st + C::OFF_HX / ES + 4 * e), n = ldv<4>(st + C::OFF_HN / ES + 4 * e);
                T v[4];
#pragma unroll
                for (int c = 0; c < 4; ++c) v[c] = fma_x<T>(x[c], a[c], n[c] * b[c]);
                stv(s1 + 4 * e, v);
            }
            push_s2(st, q[(u + 2 * RZ) % NQ]);   // s2 of plane k + Rz
            const int ctr = (tg + R) * PW + RA + PX * tx;
            const VP pc4 = ldv<PX>(st + C::OFF_HP / ES + ctr), qc4 = ldv<PX>(st + C::OFF_HQ / ES + ctr);
            const VP po4 = ldv<PX>(st + C::OFF_OP / ES + sidx), qo4 = ldv<PX>(st + C::OFF_OQ / ES + sidx);
            const T *zr = st + C::OFF_ZR / ES;
            // D^T(s2): ascending m over planes k + Rz - m, weights w^T[k][m]
            T DT[PX];
#pragma unroll
            for (int c = 0; c < PX; ++c) DT[c] = T(0);
#pragma unroll
            for (int m = 0; m < NQ; ++m) {
                const T w = zr[m];
#pragma unroll
                for (int c = 0; c < PX; ++c) DT[c] = fma_x<T>(w, q[(u + 2 * RZ - m) % NQ][c], DT[c]);
            }
            const T gz = zr[NQ];
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[stage]);
            if (++stage == ST) {
                stage = 0;
                phase ^= 1;
            }
            named_bar_sync(1, NCONS);   // the s1 tile of plane k is complete
            // L(s1), canonical pairing (x pair + y pair)
            const T *base = s1 + tg * PW + PX * tx;   // smem row tg = tile row tg - R
            const T *prow = base + R * PW;
            auto wx = [&](int i) { return ldv<PX>(prow + PX * (i / PX))[i % PX]; };
            T L[PX];
#pragma unroll
            for (int c = 0; c < PX; ++c) L[c] = A.cxy[0] * wx(RA + c);
#pragma unroll
            for (int l = 1; l <= R; ++l) {
                const VP yp = ldv<PX>(base + (R + l) * PW + RA), ym = ldv<PX>(base + (R - l) * PW + RA);
#pragma unroll
                for (int c = 0; c < PX; ++c)
                    L[c] = fma_x<T>(A.cxy[l], (wx(RA + c + l) + wx(RA + c - l)) + (yp[c] + ym[c]), L[c]);
            }
            if (!own) return;
            T pn[PX], qn[PX];
#pragma unroll
            for (int c = 0; c < PX; ++c) {
                T Fp = L[c], Fq = DT[c];
                if constexpr (IO) {
                    const int i = xg + c;
                    if (A.inj_row != nullptr && i < A.nx) {
                        const int e = ps_lookup(A.inj_off, A.inj_ent, A.nyl, k, yl, i);
                        if (e >= 0) {
                            const T v = A.inj_row[A.inj_ent[e].y];
                            if (A.inj_mask & 1) Fp = Fp + v;
                            if (A.inj_mask & 2) Fq = Fq + v;
                        }
                    }
                }
                const T g = (gx4[c] * gy) * gz;
                pn[c] = g * fma_x<T>(A.dt2, Fp, fma_x<T>(-g, po4[c], T(2) * pc4[c]));
                qn[c] = g * fma_x<T>(A.dt2, Fq, fma_x<T>(-g, qo4[c], T(2) * qc4[c]));
            }
            const int64_t a0 = (int64_t)yl * A.ys + (int64_t)k * A.zs + xg;
            if (xg + PX <= A.nx) {
                stv(A.po + a0, pn);
                stv(A.qo + a0, qn);
            } else {
#pragma unroll
                for (int c = 0; c < PX; ++c)
                    if (xg + c < A.nx) {
                        A.po[a0 + c] = pn[c];
                        A.qo[a0 + c] = qn[c];
                    }
            }
            if constexpr (IO) {
                if (A.rec_row != nullptr) {   // receivers of psi^{m-1} (duplicates allowed: every entry)
                    const long long rb = (long long)k * A.nyl + yl;
                    const int nf = (A.rec_mask & 1) + ((A.rec_mask >> 1) & 1);
                    for (int e = A.rec_off[rb]; e < A.rec_off[rb + 1]; ++e) {
                        const int c = A.rec_ent[e].x - xg;
                        if (c < 0 || c >= PX) continue;
                        T vp = pn[0], vq = qn[0];
#pragma unroll
                        for (int cc = 1; cc < PX; ++cc)
                            if (c == cc) {
                                vp = pn[cc];
                                vq = qn[cc];
                            }
                        T *o = A.rec_row + (int64_t)A.rec_ent[e].y * nf;
                        if (A.rec_mask & 1) *o++ = vp;
                        if (A.rec_mask & 2) *o = vq;
                    }
                }
            }
        };
        if constexpr (SHIFT) {   // deep queues: one loop body, the queue shifted by register moves
            for (int k = kb; k < ke; ++k) {
#pragma unroll
                for (int m = 0; m < NQ - 1; ++m)
#pragma unroll
                    for (int c = 0; c < PX; ++c) q[m][c] = q[m + 1][c];
                plane(k, 0);
            }
        } else {   // the queue index unrolled NQ times: no moves, NQ copies of the body
            for (int kbase = kb; kbase < ke; kbase += NQ) {
#pragma unroll
                for (int u = 0; u < NQ; ++u) {
                    if (kbase + u >= ke) break;
                    plane(kbase + u, u);
                }
            }
        }
    }
}

// ---------------------------------------------------------------- TMA two-pass form
// Pass 1 (k_adj_s1): s1 = fma(vx2, psi_p, vn2 psi_q) over the slab, vectorised (20 B/pt fp32).
// Pass 2 (k_adj_tma2): the forward kernel's shape with one halo'd box. Per plane k the producer
// streams the halo'd s1 box, psi_p, psi_q, vz2 of plane k + Rz (the s2 queue front), psi^m and
// psi^{m+1} of plane k and the transposed weight row; consumers (PX x points each) read
// everything from the stage -- no shared-memory pass and no CTA barrier per plane. DRAM: s1,
// psi^m (2), vz2, psi^{m+1} (2) read, psi^{m-1} (2) written = 32 B/pt fp32 (52 with pass 1).
// y-slab groups take their neighbours' s1 rows in the halo rows (vti_group_step_adjoint).
template <typename T>
__global__ void k_adj_s1(const T *__restrict__ pp, const T *__restrict__ pq, const T *__restrict__ vx2,
                         const T *__restrict__ vn2, T *__restrict__ s1, int nx4, int nyl, long long ys, long long zs)
{
    asm volatile("griddepcontrol.wait;" ::: "memory");   // programmatic dependent launch (see k_adj_tma)
    const int k = blockIdx.y, n = nyl * nx4;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
        const int y = t / nx4, x = (t - y * nx4) * 4;
        const int64_t a = (int64_t)y * ys + (int64_t)k * zs + x;
        const V4<T> p = ldv<4>(pp + a), q = ldv<4>(pq + a), vx = ldv<4>(vx2 + a), vn = ldv<4>(vn2 + a);
        T v[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) v[c] = fma_x<T>(vx[c], p[c], vn[c] * q[c]);
        stv(s1 + a, v);
    }
}

template <typename T, int R, int RZ, int TY, int ST, int PX, bool CH>
struct AdjTma2Cfg {
    static constexpr int ES = (int)sizeof(T);
    static constexpr int RA = (R + 3) / 4 * 4;
    static constexpr int PW = TX + 2 * RA, PH = TY + 2 * R, TE = PW * PH;
    static constexpr int NQ = 2 * RZ + 1;
    static constexpr int ZROW = ((NQ + 1 + 3) / 4) * 4;
    static constexpr int P_BYTES = align128(TE * ES);
    static constexpr int S_BYTES = TX * TY * ES;
    static constexpr int OFF_S1 = 0, OFF_IP = P_BYTES, OFF_IQ = OFF_IP + S_BYTES, OFF_VZ = OFF_IQ + S_BYTES;
    static constexpr int OFF_PC = OFF_VZ + S_BYTES, OFF_QC = OFF_PC + S_BYTES;
    static constexpr int OFF_OP = OFF_QC + S_BYTES, OFF_OQ = OFF_OP + S_BYTES;
    static constexpr int OFF_VX = OFF_OQ + S_BYTES, OFF_VN = OFF_VX + (CH ? S_BYTES : 0);   // CH only
    static constexpr int OFF_ZR = OFF_VN + (CH ? S_BYTES : 0);
    static constexpr int STAGE = align128(OFF_ZR + ZROW * ES);
    static constexpr uint32_t FULL_TX = TE * ES + (CH ? 9 : 7) * S_BYTES + ZROW * ES;
    static constexpr uint32_t PRIME_TX = 3 * S_BYTES;
    static constexpr int OFF_BAR = ST * STAGE;
    static constexpr int SMEM = OFF_BAR + 2 * ST * 8;
    static constexpr int TPR = TX / PX;
    static constexpr int NCONS = TY * TPR;
    static constexpr int NT = NCONS + 32;
    static_assert(PW % 4 == 0 && PW <= 256 && PH <= 256, "TMA box");
    static_assert(NCONS % 32 == 0, "whole consumer warps");
};

template <typename T, int R, int RZ, int TY, int ST, int PX, bool IO, bool CH, int MINB>
__global__ void __launch_bounds__(AdjTma2Cfg<T, R, RZ, TY, ST, PX, CH>::NT, MINB)
    k_adj_tma2(const __grid_constant__ AdjTmaParams<T> P)
{
    using C = AdjTma2Cfg<T, R, RZ, TY, ST, PX, CH>;
    using VP = Vec<T, PX>;
    constexpr int NQ = C::NQ, RA = C::RA, PW = C::PW, ES = C::ES, NCONS = C::NCONS, TPR = C::TPR;
    constexpr bool SHIFT = NQ > 9;   // i-cache: NQ unrolled copies of a deep body miss (ncu: no_instructions)
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + C::OFF_BAR);
    uint64_t *empty = full + ST;
    const AdjParams<T> &A = P.A;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < ST; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NCONS / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        for (int i = 0; i < (CH ? 8 : 6); ++i) prefetch_tmap(&P.tm[i]);
    }
    __syncthreads();
    asm volatile("griddepcontrol.wait;" ::: "memory");   // programmatic dependent launch (see k_adj_tma)
    int stage = 0;
    uint32_t phase = 0;
    if (warp == NCONS / 32) {   // producer
        if (lane != 0) return;
        for (int item = blockIdx.x; item < P.items; item += gridDim.x) {
            int x0, y0, kb, ke;
            adj_item<TY>(P, item, x0, y0, kb, ke);
            const int nload = (ke - kb) + 2 * RZ;
            for (int t = 0; t < nload; ++t) {
                mbar_wait(&empty[stage], phase ^ 1);
                uint8_t *st = smem + stage * C::STAGE;
                uint64_t *bar = &full[stage];
                if (t < 2 * RZ) {
                    const int kk = kb - RZ + t;
                    mbar_arrive_expect_tx(bar, C::PRIME_TX);
                    tma_load_3d(st + C::OFF_IP, &P.tm[1], x0, y0, kk, bar);
                    tma_load_3d(st + C::OFF_IQ, &P.tm[2], x0, y0, kk, bar);
                    tma_load_3d(st + C::OFF_VZ, &P.tm[3], x0, y0, kk, bar);
                } else {
                    const int k = kb + t - 2 * RZ;
                    mbar_arrive_expect_tx(bar, C::FULL_TX);
                    tma_load_3d(st + C::OFF_S1, &P.tm[0], x0 - RA, y0, k, bar);   // halo'd: view row y0 = local y0 - R
                    tma_load_3d(st + C::OFF_IP, &P.tm[1], x0, y0, k + RZ, bar);
                    tma_load_3d(st + C::OFF_IQ, &P.tm[2], x0, y0, k + RZ, bar);
                    tma_load_3d(st + C::OFF_VZ, &P.tm[3], x0, y0, k + RZ, bar);
                    tma_load_3d(st + C::OFF_PC, &P.tm[1], x0, y0, k, bar);
                    tma_load_3d(st + C::OFF_QC, &P.tm[2], x0, y0, k, bar);
                    tma_load_3d(st + C::OFF_OP, &P.tm[4], x0, y0, k, bar);
                    tma_load_3d(st + C::OFF_OQ, &P.tm[5], x0, y0, k, bar);
                    if constexpr (CH) {
                        tma_load_3d(st + C::OFF_VX, &P.tm[6], x0, y0, k, bar);
                        tma_load_3d(st + C::OFF_VN, &P.tm[7], x0, y0, k, bar);
                    }
                    bulk_load(st + C::OFF_ZR, A.zrow + (size_t)k * C::ZROW, C::ZROW * ES, bar);
                }
                if (++stage == ST) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
        return;
    }

    const int tx = threadIdx.x % TPR, tg = threadIdx.x / TPR;
    const int sidx = tg * TX + PX * tx;
    for (int item = blockIdx.x; item < P.items; item += gridDim.x) {
        int x0, y0, kb, ke;
        adj_item<TY>(P, item, x0, y0, kb, ke);
        const int xg = x0 + PX * tx, yl = y0 + tg;
        const bool own = xg < A.nx && yl < A.nyl;
        const T gy = yl < A.nyl ? A.gy[yl] : T(0);
        const VP gxv = ldv<PX>(A.gx + xg);
        T q[NQ][PX];
        auto push_s2 = [&](const T *st, T (&v)[PX]) {
            const VP ip = ldv<PX>(st + C::OFF_IP / ES + sidx), iq = ldv<PX>(st + C::OFF_IQ / ES + sidx);
            const VP vz = ldv<PX>(st + C::OFF_VZ / ES + sidx);
#pragma unroll
            for (int c = 0; c < PX; ++c) v[c] = vz[c] * (ip[c] + iq[c]);
        };
#pragma unroll
        for (int t = 0; t < 2 * RZ; ++t) {
            mbar_wait(&full[stage], phase);
            push_s2(reinterpret_cast<const T *>(smem + stage * C::STAGE), q[SHIFT ? t + 1 : t]);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[stage]);
            if (++stage == ST) {
                stage = 0;
                phase ^= 1;
            }
        }
        // plane k; slot (u + j) % NQ of the queue holds s2 of plane k - Rz + j
        auto plane = [&](const int k, const int u) {
            mbar_wait(&full[stage], phase);
            const T *st = reinterpret_cast<const T *>(smem + stage * C::STAGE);
            push_s2(st, q[(u + 2 * RZ) % NQ]);
            const VP pcv = ldv<PX>(st + C::OFF_PC / ES + sidx), qcv = ldv<PX>(st + C::OFF_QC / ES + sidx);
            const VP pov = ldv<PX>(st + C::OFF_OP / ES + sidx), qov = ldv<PX>(st + C::OFF_OQ / ES + sidx);
            VP vxv, vnv;
            if constexpr (CH) {
                vxv = ldv<PX>(st + C::OFF_VX / ES + sidx);
                vnv = ldv<PX>(st + C::OFF_VN / ES + sidx);
            }
            const T *zr = st + C::OFF_ZR / ES;
            T DT[PX];
#pragma unroll
            for (int c = 0; c < PX; ++c) DT[c] = T(0);
#pragma unroll
            for (int m = 0; m < NQ; ++m) {
                const T w = zr[m];
#pragma unroll
                for (int c = 0; c < PX; ++c) DT[c] = fma_x<T>(w, q[(u + 2 * RZ - m) % NQ][c], DT[c]);
            }
            const T gz = zr[NQ];
            // L(s1) from the staged box, canonical pairing (x pair + y pair)
            const T *base = st + C::OFF_S1 / ES + tg * PW + PX * tx;
            const T *prow = base + R * PW;
            auto wx = [&](int i) { return ldv<PX>(prow + PX * (i / PX))[i % PX]; };
            T L[PX];
#pragma unroll
            for (int c = 0; c < PX; ++c) L[c] = A.cxy[0] * wx(RA + c);
#pragma unroll
            for (int l = 1; l <= R; ++l) {
                const VP yp = ldv<PX>(base + (R + l) * PW + RA), ym = ldv<PX>(base + (R - l) * PW + RA);
#pragma unroll
                for (int c = 0; c < PX; ++c)
                    L[c] = fma_x<T>(A.cxy[l], (wx(RA + c + l) + wx(RA + c - l)) + (yp[c] + ym[c]), L[c]);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[stage]);
            if (++stage == ST) {
                stage = 0;
                phase ^= 1;
            }
            if (!own) return;
            T pn[PX], qn[PX];
#pragma unroll
            for (int c = 0; c < PX; ++c) {
                T Fp = L[c], Fq = DT[c];
                if constexpr (IO) {
                    const int i = xg + c;
                    if (A.inj_row != nullptr && i < A.nx) {
                        const int e = ps_lookup(A.inj_off, A.inj_ent, A.nyl, k, yl, i);
                        if (e >= 0) {
                            const T v = A.inj_row[A.inj_ent[e].y];
                            if (A.inj_mask & 1) Fp = Fp + v;
                            if (A.inj_mask & 2) Fq = Fq + v;
                        }
                    }
                }
                const T g = (gxv[c] * gy) * gz;
                pn[c] = g * fma_x<T>(A.dt2, Fp, fma_x<T>(-g, pov[c], T(2) * pcv[c]));
                qn[c] = g * fma_x<T>(A.dt2, Fq, fma_x<T>(-g, qov[c], T(2) * qcv[c]));
            }
            const int64_t a0 = (int64_t)yl * A.ys + (int64_t)k * A.zs + xg;
            T s1n[PX];
            if constexpr (CH) {   // the next step's s1 = fma(vx2, psi_p, vn2 * psi_q) of psi^{m-1}
#pragma unroll
                for (int c = 0; c < PX; ++c) s1n[c] = fma_x<T>(vxv[c], pn[c], vnv[c] * qn[c]);
            }
            if (xg + PX <= A.nx) {
                stv(A.po + a0, pn);
                stv(A.qo + a0, qn);
                if constexpr (CH) stv(A.s1o + a0, s1n);
            } else {
#pragma unroll
                for (int c = 0; c < PX; ++c)
                    if (xg + c < A.nx) {
                        A.po[a0 + c] = pn[c];
                        A.qo[a0 + c] = qn[c];
                        if constexpr (CH) A.s1o[a0 + c] = s1n[c];
                    }
            }
            if constexpr (IO) {
                if (A.rec_row != nullptr) {
                    const long long rb = (long long)k * A.nyl + yl;
                    const int nf = (A.rec_mask & 1) + ((A.rec_mask >> 1) & 1);
                    for (int e = A.rec_off[rb]; e < A.rec_off[rb + 1]; ++e) {
                        const int c = A.rec_ent[e].x - xg;
                        if (c < 0 || c >= PX) continue;
                        T vp = pn[0], vq = qn[0];
#pragma unroll
                        for (int cc = 1; cc < PX; ++cc)
                            if (c == cc) {
                                vp = pn[cc];
                                vq = qn[cc];
                            }
                        T *o = A.rec_row + (int64_t)A.rec_ent[e].y * nf;
                        if (A.rec_mask & 1) *o++ = vp;
                        if (A.rec_mask & 2) *o = vq;
                    }
                }
            }
        };
        if constexpr (SHIFT) {   // deep queues: one loop body, the queue shifted by register moves
            for (int k = kb; k < ke; ++k) {
#pragma unroll
                for (int m = 0; m < NQ - 1; ++m)
#pragma unroll
                    for (int c = 0; c < PX; ++c) q[m][c] = q[m + 1][c];
                plane(k, 0);
            }
        } else {   // the queue index unrolled NQ times: no moves, NQ copies of the body
            for (int kbase = kb; kbase < ke; kbase += NQ) {
#pragma unroll
                for (int u = 0; u < NQ; ++u) {
                    if (kbase + u >= ke) break;
                    plane(kbase + u, u);
                }
            }
        }
    }
}

// wT[k][m] = w^z[k+Rz-m][m] for planes inside the grid, else 0; wT[k][NQ] = gz[k]
template <typename T>
__global__ void k_adj_wt(const T *__restrict__ zrow, T *__restrict__ wt, int nz, int rz, int stride)
{
    const int NQ = 2 * rz + 1;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nz * stride; e += gridDim.x * blockDim.x) {
        const int k = e / stride, m = e % stride;
        T v = T(0);
        if (m < NQ) {
            const int kk = k + rz - m;
            if (kk >= 0 && kk < nz) v = zrow[(size_t)kk * stride + m];
        } else if (m == NQ) {
            v = zrow[(size_t)k * stride + NQ];
        }
        wt[e] = v;
    }
}

// launches of the TMA adjoint forms: programmatic dependent launch (env VTI_PDL=0: plain)
static cudaError_t adj_launch(vti_s *h, const void *fn, dim3 grid, dim3 block, void **args, size_t smem)
{
    static const bool pdl = !getenv("VTI_PDL") || atoi(getenv("VTI_PDL")) != 0;
    cudaLaunchConfig_t lc = {};
    lc.gridDim = grid;
    lc.blockDim = block;
    lc.dynamicSmemBytes = smem;
    lc.stream = h->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelExC(&lc, fn, args);
}

struct AdjTmaEntry {
    int es, r, rz, form, ty, px, st, minb;   // form 1: one-pass k_adj_tma; form 2: k_adj_s1 + k_adj_tma2;
                                             // st: ring depth; minb: __launch_bounds__ CTAs per SM
    const void *fn, *fn_io;        // form 2: the last step of a call (no s1 out)
    int smem, threads, zrow;
    const void *fn_ch, *fn_ch_io;  // form 2: chained steps (s1 of psi^{m-1} out)
    int smem_ch;
};

template <typename T, int R, int RZ, int TY, int ST, int PX = 4>
constexpr AdjTmaEntry adj_tma1()
{
    using C = AdjTmaCfg<T, R, RZ, TY, ST, PX>;
    static_assert(C::SMEM <= 227 * 1024, "one-pass adjoint stage ring exceeds the per-CTA shared memory");
    return {C::ES, R, RZ, 1, TY, PX, ST, 1, (const void *)k_adj_tma<T, R, RZ, TY, ST, PX, false>,
            (const void *)k_adj_tma<T, R, RZ, TY, ST, PX, true>, C::SMEM, C::NT, C::ZROW, nullptr, nullptr, 0};
}

template <typename T, int R, int RZ, int TY, int ST, int PX, int MINB = 1>
constexpr AdjTmaEntry adj_tma2()
{
    using C = AdjTma2Cfg<T, R, RZ, TY, ST, PX, false>;
    using CC = AdjTma2Cfg<T, R, RZ, TY, ST, PX, true>;
    static_assert(CC::SMEM <= 227 * 1024, "chained adjoint stage ring exceeds the per-CTA shared memory");
    return {C::ES, R, RZ, 2, TY, PX, ST, MINB, (const void *)k_adj_tma2<T, R, RZ, TY, ST, PX, false, false, MINB>,
            (const void *)k_adj_tma2<T, R, RZ, TY, ST, PX, true, false, MINB>, C::SMEM, C::NT, C::ZROW,
            (const void *)k_adj_tma2<T, R, RZ, TY, ST, PX, false, true, MINB>,
            (const void *)k_adj_tma2<T, R, RZ, TY, ST, PX, true, true, MINB>, CC::SMEM};
}

// Per (precision, radii) the first eligible entry is the default. Env: VTI_ADJ_FORM=1|2 and
// VTI_ADJ_TMA_TY / VTI_ADJ_TMA_PX restrict the choice; y-slab groups need form 2.
static const AdjTmaEntry *find_adj_tma(int es, int r, int rz, bool group)
{
    static const AdjTmaEntry table[] = {
        adj_tma1<float, 4, 4, 8, 3>(),        adj_tma1<float, 4, 4, 16, 2>(),    adj_tma2<float, 4, 4, 8, 4, 4>(),
        adj_tma1<float, 8, 4, 16, 2>(),       adj_tma2<float, 8, 4, 8, 4, 4>(),
        adj_tma1<float, 6, 6, 16, 2>(),       adj_tma2<float, 6, 6, 8, 4, 4>(),
        adj_tma2<float, 12, 8, 8, 3, 4>(),    adj_tma2<float, 12, 8, 8, 4, 4>(), adj_tma1<float, 12, 8, 16, 2>(),
        adj_tma2<double, 4, 4, 8, 3, 4>(),    adj_tma2<double, 4, 4, 8, 2, 4>(), adj_tma1<double, 4, 4, 8, 2>(),
        adj_tma2<double, 8, 4, 8, 3, 4>(),    adj_tma2<double, 8, 4, 8, 2, 2>(),
        adj_tma2<double, 6, 6, 8, 3, 4>(),    adj_tma2<double, 6, 6, 8, 2, 2>(),
        adj_tma2<double, 12, 8, 4, 3, 2>(),   adj_tma2<double, 12, 8, 8, 2, 2>(),
    };
    static const int want_form = getenv("VTI_ADJ_FORM") ? atoi(getenv("VTI_ADJ_FORM")) : 0;
    static const int want_ty = getenv("VTI_ADJ_TMA_TY") ? atoi(getenv("VTI_ADJ_TMA_TY")) : 0;
    static const int want_px = getenv("VTI_ADJ_TMA_PX") ? atoi(getenv("VTI_ADJ_TMA_PX")) : 0;
    static const int want_st = getenv("VTI_ADJ_TMA_ST") ? atoi(getenv("VTI_ADJ_TMA_ST")) : 0;
    static const int want_mb = getenv("VTI_ADJ_TMA_MINB") ? atoi(getenv("VTI_ADJ_TMA_MINB")) : 0;
    for (const AdjTmaEntry &e : table)
        if (e.es == es && e.r == r && e.rz == rz && (!group || e.form == 2) && (!want_form || e.form == want_form) &&
            (!want_ty || e.ty == want_ty) && (!want_px || e.px == want_px) && (!want_st || e.st == want_st) &&
            (!want_mb || e.minb == want_mb))
            return &e;
    return nullptr;
}

static const AdjTmaEntry *adj_tma_of(const vti_s *h)
{
    static const bool on = !getenv("VTI_ADJ_TMA") || atoi(getenv("VTI_ADJ_TMA")) != 0;
    if (!on) return nullptr;
    return find_adj_tma(h->es, h->R, h->RZ, h->cfg.nranks > 1);
}

// builds the transposed weight rows (once) and the entry's tensor maps of both buffer parities
static vti_status ensure_adj_tma(vti_s *h, const AdjTmaEntry *E, int &ctas)
{
    if (h->adj_tma < 0) return fail(h, VTI_E_CUDA, "adjoint TMA kernel setup failed earlier");
    if (h->adj_tma == 0) {
        h->adj_tma = -1;
        if (E->zrow != h->K->zrow) return fail(h, VTI_E_CUDA, "adjoint z-row stride mismatch");
        const size_t bytes = (size_t)h->cfg.nz * E->zrow * h->es;
        cudaError_t e = cudaMalloc(&h->adj_wt, bytes);
        if (e != cudaSuccess) return fail(h, VTI_E_CUDA, "cudaMalloc(%zu bytes): %s", bytes, cudaGetErrorString(e));
        h->device_bytes += (int64_t)bytes;
        if (h->es == 8)
            k_adj_wt<double><<<64, 256, 0, h->stream>>>((const double *)h->zrow, (double *)h->adj_wt, h->cfg.nz, h->RZ,
                                                      E->zrow);
        else
            k_adj_wt<float><<<64, 256, 0, h->stream>>>((const float *)h->zrow, (float *)h->adj_wt, h->cfg.nz, h->RZ,
                                                     E->zrow);
        CU(h, cudaGetLastError());
        const int RA = (h->R + 3) / 4 * 4, PW = TX + 2 * RA, PH = E->ty + 2 * h->R;
        const CUtensorMapL2promotion hp = CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
        vti_status s;
        for (int c = 0; c < 2; ++c) {
            CUtensorMap *tm = h->adj_tm[c];
            if (E->form == 1) {
                void *halo[4] = {h->pbuf[c], h->qbuf[c], h->vx2, h->vn2};
                for (int i = 0; i < 4; ++i)
                    if ((s = encode(h, &tm[i], halo[i], h->rows, PW, PH, hp)) != VTI_OK) return s;
                void *inter[5] = {h->p_int(c), h->q_int(c), h->in(h->vz2), h->p_int(1 - c), h->q_int(1 - c)};
                for (int i = 0; i < 5; ++i)
                    if ((s = encode(h, &tm[4 + i], inter[i], h->nyl, TX, E->ty)) != VTI_OK) return s;
            } else {   // tm[0] (the s1 view) is taken from adj_tm_s1 at launch
                void *inter[7] = {h->p_int(c),     h->q_int(c),   h->in(h->vz2), h->p_int(1 - c),
                                  h->q_int(1 - c), h->in(h->vx2), h->in(h->vn2)};
                for (int i = 0; i < 7; ++i)
                    if ((s = encode(h, &tm[1 + i], inter[i], h->nyl, TX, E->ty)) != VTI_OK) return s;
            }
        }
        if (E->form == 2)
            for (int b = 0; b < 2; ++b)
                if ((s = encode(h, &h->adj_tm_s1[b], h->adj_s[b], h->rows, PW, PH, hp)) != VTI_OK) return s;
        int occ = 0;
        for (const void *fn : {E->fn, E->fn_io})
            CU(h, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, E->smem));
        CU(h, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, E->fn, E->threads, E->smem));
        if (occ < 1) return fail(h, VTI_E_CUDA, "adjoint TMA kernel cannot be resident (smem %d B)", E->smem);
        h->adj_tma = occ * h->sms;   // the grid cap
        if (E->fn_ch) {
            for (const void *fn : {E->fn_ch, E->fn_ch_io})
                CU(h, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, E->smem_ch));
            CU(h, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, E->fn_ch, E->threads, E->smem_ch));
            if (occ < 1) return fail(h, VTI_E_CUDA, "adjoint TMA kernel cannot be resident (smem %d B)", E->smem_ch);
            h->adj_tma_ch = occ * h->sms;
        }
    }
    ctas = h->adj_tma;
    return VTI_OK;
}

// form 2: s1 of psi^m is in scratch buffer sb; chain: also write the next step's s1 into 1 - sb
template <typename T>
static vti_status launch_adj_tma(vti_s *h, const AdjTmaEntry *E, const AdjParams<T> &A, bool io, int sb, bool chain)
{
    int ctas = 0;
    vti_status s = ensure_adj_tma(h, E, ctas);
    if (s != VTI_OK) return s;
    AdjTmaParams<T> P;
    memcpy(P.tm, h->adj_tm[h->cur], sizeof(P.tm));
    if (E->form == 2) P.tm[0] = h->adj_tm_s1[sb];
    chain = chain && E->form == 2;
    if (chain) ctas = h->adj_tma_ch;
    P.A = A;
    P.A.zrow = (const T *)h->adj_wt;
    P.A.s1o = chain ? (T *)h->in(h->adj_s[1 - sb]) : nullptr;
    P.ntx = (h->cfg.nx + TX - 1) / TX;
    P.nty = (h->nyl + E->ty - 1) / E->ty;
    const int tiles = P.ntx * P.nty;
    static const int zenv = getenv("VTI_ADJ_ZCHUNK") ? atoi(getenv("VTI_ADJ_ZCHUNK")) : 0;
    // about 6 items per resident CTA, z-chunks of >= 32 planes (the 2R_z priming loads per item)
    // unless that leaves CTAs idle (small grids: chunks down to 4 planes)
    const int want = (6 * ctas + tiles - 1) / tiles;
    int nzc = std::max(1, std::min((h->cfg.nz + 31) / 32, want));
    if (tiles * nzc < ctas) nzc = std::max(1, std::min((h->cfg.nz + 3) / 4, want));
    P.zchunk = zenv > 0 ? zenv : (h->cfg.nz + nzc - 1) / nzc;
    nzc = (h->cfg.nz + P.zchunk - 1) / P.zchunk;
    P.items = tiles * nzc;
    const int grid = std::min(P.items, ctas);
    void *args[] = {&P};
    const void *fn = chain ? (io ? E->fn_ch_io : E->fn_ch) : (io ? E->fn_io : E->fn);
    CU(h, adj_launch(h, fn, dim3(grid), dim3(E->threads), args, chain ? E->smem_ch : E->smem));
    return VTI_OK;
}

// Which form. The TMA forms (above) when compiled for the handle's precision and radii; the
// table's first entry per (precision, radii) is the measured best on one B200
// (tools/adjoint_rate.py, profiles/r02/adjoint_tma_r02.txt, Gpoints/s):
//   fp32: one-pass C2 (4,4) 172-174 (8-row tiles, 3 stages, 2 CTAs/SM), C3 (8,4) 139-141 and
//         C5 (6,6) 135-136 (16-row tiles); chained two-pass N1 (12,8) 137 (one-pass: 29-54);
//   fp64: chained two-pass, 4 x points per thread and 3 stages: C2 72, C3 63, C5 66.5; for
//         (12,8) 2 x points per thread on 4-row tiles, 3 stages: N1 64 (8-row tiles: 56).
// Before them, the cp.async forms: fp32 one-pass C2 78.1, C3 81.4, C5 82.2, N1 38.7; fp64
// C2 36.9, C3 31.2, C5 34.1, N1 19.3 (two-pass at R_xy >= 8). With VTI_ADJ_TMA=0 those run:
// y-slab groups the two-pass one, single slabs the one-pass one (VTI_ADJ_TWO_PASS=1/0 forces
// either) except fp64 at R_xy >= 8.
enum AdjForm { ADJ_FUSED = 0, ADJ_TWO_PASS = 1, ADJ_TMA1 = 2, ADJ_TMA2 = 3 };

static AdjForm adj_form(const vti_s *h, const AdjTmaEntry **E = nullptr)
{
    const AdjTmaEntry *e = adj_tma_of(h);
    if (E) *E = e;
    if (e) return e->form == 1 ? ADJ_TMA1 : ADJ_TMA2;
    if (h->cfg.nranks > 1) return ADJ_TWO_PASS;
    static const int env = getenv("VTI_ADJ_TWO_PASS") ? atoi(getenv("VTI_ADJ_TWO_PASS")) : -1;
    if (env >= 0) return env != 0 ? ADJ_TWO_PASS : ADJ_FUSED;
    return h->es == 8 && h->R >= 8 ? ADJ_TWO_PASS : ADJ_FUSED;
}

// the scratch s1 (and, for the cp.async two-pass form, s2) is needed
static bool adj_needs_s1(const vti_s *h)
{
    const AdjForm f = adj_form(h);
    return f == ADJ_TWO_PASS || f == ADJ_TMA2;
}

// Two-pass forms, first launch (phase 1 of a step): s1 (k_adj_s1) or s1, s2 (k_adj_prep).
template <typename T>
static vti_status adjoint_prep_t(vti_s *h, int sb = 0)
{
    const int c = h->cur;
    if (adj_form(h) == ADJ_TMA2) {
        const int nx4 = (int)(h->nxp / 4), n = h->nyl * nx4;
        const dim3 grid((unsigned)std::min((n + 255) / 256, 64), (unsigned)h->cfg.nz);
        const T *pp = (const T *)h->p_int(c), *pq = (const T *)h->q_int(c);
        const T *vx = (const T *)h->in(h->vx2), *vn = (const T *)h->in(h->vn2);
        T *s1 = (T *)h->in(h->adj_s[sb]);
        long long ys = h->ys, zs = h->zs;
        int nyl = h->nyl, nx4v = nx4;
        void *args[] = {&pp, &pq, &vx, &vn, &s1, &nx4v, &nyl, &ys, &zs};
        CU(h, adj_launch(h, (const void *)k_adj_s1<T>, grid, dim3(256), args, 0));
    } else {
        k_adj_prep<T><<<4 * h->sms, 256, 0, h->stream>>>((const T *)h->p_int(c), (const T *)h->q_int(c),
                                                       (const T *)h->in(h->vx2), (const T *)h->in(h->vn2),
                                                       (const T *)h->in(h->vz2), (T *)h->in(h->adj_s[0]),
                                                       (T *)h->in(h->adj_s[1]), h->cfg.nx, h->nyl, h->cfg.nz,
                                                       h->ys, h->zs);
    }
    CU(h, cudaGetLastError());
    return VTI_OK;
}

// One adjoint step. Two-pass forms: prep = run the first pass (s1 of psi^m into scratch sb)
// here; the chained TMA form (chain) also writes the next step's s1 into scratch 1 - sb.
template <typename T>
static vti_status adjoint_step_t(vti_s *h, bool prep = true, int sb = 0, bool chain = false)
{
    const int c = h->cur, o = 1 - c;
    const int grid = 4 * h->sms;
    const AdjTmaEntry *E = nullptr;
    const AdjForm form = adj_form(h, &E);
    const bool two_pass = form == ADJ_TWO_PASS || form == ADJ_TMA2;
    T *s1 = nullptr, *s2 = nullptr;
    if (two_pass) {
        s1 = (T *)h->in(h->adj_s[sb]);
        if (form == ADJ_TWO_PASS) s2 = (T *)h->in(h->adj_s[1]);
        if (prep) {
            vti_status st = adjoint_prep_t<T>(h, sb);
            if (st != VTI_OK) return st;
        }
    }
    AdjParams<T> A;
    A.s1 = s1;
    A.s2 = s2;
    A.vx = (const T *)h->in(h->vx2);
    A.vn = (const T *)h->in(h->vn2);
    A.vz = (const T *)h->in(h->vz2);
    A.pc = (const T *)h->p_int(c);
    A.qc = (const T *)h->q_int(c);
    A.po = (T *)h->p_int(o);
    A.qo = (T *)h->q_int(o);
    A.zrow = (const T *)h->zrow;
    A.zrow_stride = h->K->zrow;
    A.gx = (const T *)h->gx;
    A.gy = (const T *)h->gy;
    for (int l = 0; l <= MAX_R; ++l) A.cxy[l] = l <= h->R ? (T)h->cxy[l] : T(0);
    A.dt2 = (T)(h->cfg.dt * h->cfg.dt);
    A.nx = h->cfg.nx;
    A.nyl = h->nyl;
    A.nz = h->cfg.nz;
    A.ys = h->ys;
    A.zs = h->zs;
    const long long irow = (long long)(h->n - h->inj_t_first);   // time index m of this step
    const bool inj = h->inj_set.n > 0 && irow >= 0 && irow < h->inj_nt;
    A.inj_off = h->inj_set.off;
    A.inj_ent = h->inj_set.ent;
    A.inj_row = inj ? (const T *)h->inj_tr + irow * h->inj_cols : nullptr;
    A.inj_mask = h->inj_mask;
    const bool rec = h->rec_set.n > 0 && h->rec_steps < h->rec_cap;
    const int nf = (h->rec_mask & 1) + ((h->rec_mask >> 1) & 1);
    A.rec_off = h->rec_set.off;
    A.rec_ent = h->rec_set.ent;
    A.rec_row = rec ? (T *)h->traces + (size_t)h->rec_steps * h->nrec * nf : nullptr;
    A.rec_mask = h->rec_mask;
    // a local group's slab reads its neighbours' s1 rows, copied into its halo (vti_group_step_adjoint)
    A.y_lo = h->cfg.rank > 0 ? -h->R : 0;
    A.y_hi = h->cfg.rank < h->cfg.nranks - 1 ? h->nyl + h->R : h->nyl;
    const bool io = A.inj_row != nullptr || A.rec_row != nullptr;
    switch (form) {
    case ADJ_TMA1:
    case ADJ_TMA2: return launch_adj_tma<T>(h, E, A, io, sb, chain);
    case ADJ_TWO_PASS: return launch_adj_step<T>(h, A, grid);
    default: return launch_adj_fused<T>(h, A);
    }
}

}  // namespace

static vti_status ensure_adj_scratch(vti_s *h)
{
    if (!adj_needs_s1(h) || h->adj_s[0]) return VTI_OK;
    // the two-pass forms' coefficient-weighted fields s1 (and s2): the slab's geometry, zero halo
    const size_t bytes = h->total_elems() * h->es;
    for (int b = 0; b < 2; ++b) {   // s1, s2 (cp.async form) or two s1 buffers (chained TMA form)
        cudaError_t e = cudaMalloc(&h->adj_s[b], bytes);
        if (e != cudaSuccess) return fail(h, VTI_E_CUDA, "cudaMalloc(%zu bytes): %s", bytes, cudaGetErrorString(e));
        CU(h, cudaMemsetAsync(h->adj_s[b], 0, bytes, h->stream));
        h->device_bytes += (int64_t)bytes;
    }
    return VTI_OK;
}

// s1's R boundary rows of the neighbour on `side` (0: rank-1, its last rows; 1: rank+1, its
// first rows) into this slab's halo rows, on this handle's stream (the copy engine reads the
// neighbour's memory directly, any device).
static vti_status copy_s1_halo(vti_s *h, const vti_s *nb, int side, int sb = 0)
{
    const char *src = nb->in(nb->adj_s[sb]) + (size_t)(side == 0 ? nb->nyl - nb->R : 0) * nb->ys * nb->es;
    char *dst = h->in(h->adj_s[sb]) + (side == 0 ? -(long long)h->R : (long long)h->nyl) * h->ys * h->es;
    // [z][y][x]: R rows are contiguous within each plane; [y][z][x]: one block
    const size_t width = (size_t)h->R * h->ys * h->es;
    const size_t height = h->layout_zyx ? (size_t)h->cfg.nz : 1;
    const size_t spitch = h->layout_zyx ? (size_t)nb->zs * nb->es : width;
    const size_t dpitch = h->layout_zyx ? (size_t)h->zs * h->es : width;
    CU(h, cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, cudaMemcpyDefault, h->stream));
    return VTI_OK;
}

// a group slab's bookkeeping after one adjoint step
static vti_status adjoint_advance(vti_s *h)
{
    h->cur = 1 - h->cur;
    h->n -= 1;
    h->halo_dirty = true;   // p's halo rows are stale for a later forward step: re-publish then
    if (h->rec_set.n > 0) h->rec_steps = std::min(h->rec_cap, h->rec_steps + 1);
    if (h->cfg.check_every > 0 && h->n % h->cfg.check_every == 0) return check_finite(h);
    return VTI_OK;
}

extern "C" {

vti_status vti_group_step_adjoint(vti_t *hs, int32_t n, int32_t nsteps)
{
    if (!hs || n < 1 || nsteps < 0) return VTI_E_PARAM;
    if (n == 1) return vti_step_adjoint(hs[0], nsteps);
    for (int i = 0; i < n; ++i) {
        if (!hs[i]) return VTI_E_PARAM;
        if (hs[i]->cfg.nranks != n || hs[i]->cfg.rank != i || !hs[i]->group_mode)
            return fail(hs[i], VTI_E_STATE, "handle %d is not rank %d of a %d-handle local group", i, i, n);
        if (!hs[i]->model_set) return fail(hs[i], VTI_E_STATE, "model not set");
        if (hs[i]->n != hs[0]->n || hs[i]->cur != hs[0]->cur)
            return fail(hs[i], VTI_E_STATE, "time indices or buffer parity differ inside the group");
    }
    vti_status s;
    for (int i = 0; i < n; ++i) {
        CU(hs[i], cudaSetDevice(hs[i]->cfg.device));
        if ((s = ensure_adj_scratch(hs[i])) != VTI_OK) return s;
    }
    if (adj_form(hs[0]) == ADJ_TMA2) {
        // chained TMA form: the first pass once, its s1 halo rows exchanged (pack, copies between
        // the slabs' send / recv buffers, unpack: the NCCL path's sequence, vti_transport.cu);
        // then per step the kernel, which also writes the next s1 into the other buffer, and
        // the exchange of that buffer's rows
        std::vector<void *> bufs(n);
        for (int i = 0; i < n; ++i) {
            vti_s *h = hs[i];
            CU(h, cudaSetDevice(h->cfg.device));
            s = h->es == 8 ? adjoint_prep_t<double>(h, 0) : adjoint_prep_t<float>(h, 0);
            if (s != VTI_OK) return s;
            bufs[i] = h->adj_s[0];
        }
        if ((s = rows_exchange(hs, n, bufs.data(), false)) != VTI_OK) return s;
        int sb = 0;
        for (int it = 0; it < nsteps; ++it) {
            const bool chain = it + 1 < nsteps;
            for (int i = 0; i < n; ++i) {
                vti_s *h = hs[i];
                CU(h, cudaSetDevice(h->cfg.device));
                s = h->es == 8 ? adjoint_step_t<double>(h, false, sb, chain) : adjoint_step_t<float>(h, false, sb, chain);
                if (s != VTI_OK) return s;
                if ((s = adjoint_advance(h)) != VTI_OK) return s;
                bufs[i] = h->adj_s[1 - sb];
            }
            if (chain && (s = rows_exchange(hs, n, bufs.data(), false)) != VTI_OK) return s;
            sb ^= 1;
        }
        return VTI_OK;
    }
    for (int it = 0; it < nsteps; ++it) {
        // 1. s1, s2 of every slab; a slab's rows may be overwritten only once its neighbours
        //    copied the previous step's (their ev_comm, recorded after those copies)
        for (int i = 0; i < n; ++i) {
            vti_s *h = hs[i];
            CU(h, cudaSetDevice(h->cfg.device));
            if (it > 0) {
                if (i > 0) CU(h, cudaStreamWaitEvent(h->stream, hs[i - 1]->ev_comm, 0));
                if (i < n - 1) CU(h, cudaStreamWaitEvent(h->stream, hs[i + 1]->ev_comm, 0));
            }
            s = h->es == 8 ? adjoint_prep_t<double>(h) : adjoint_prep_t<float>(h);
            if (s != VTI_OK) return s;
            CU(h, cudaEventRecord(h->ev_edge, h->stream));
        }
        // 2. the neighbours' boundary rows of s1 into each halo
        for (int i = 0; i < n; ++i) {
            vti_s *h = hs[i];
            CU(h, cudaSetDevice(h->cfg.device));
            for (int side = 0; side < 2; ++side) {
                const int j = side == 0 ? i - 1 : i + 1;
                if (j < 0 || j >= n) continue;
                CU(h, cudaStreamWaitEvent(h->stream, hs[j]->ev_edge, 0));
                if ((s = copy_s1_halo(h, hs[j], side)) != VTI_OK) return s;
            }
            CU(h, cudaEventRecord(h->ev_comm, h->stream));
        }
        // 3. the stencils and update of every slab
        for (int i = 0; i < n; ++i) {
            vti_s *h = hs[i];
            CU(h, cudaSetDevice(h->cfg.device));
            s = h->es == 8 ? adjoint_step_t<double>(h, false) : adjoint_step_t<float>(h, false);
            if (s != VTI_OK) return s;
            if ((s = adjoint_advance(h)) != VTI_OK) return s;
        }
    }
    return VTI_OK;
}

vti_status vti_step_adjoint(vti_t h, int32_t nsteps)
{
    if (!h) return VTI_E_PARAM;
    if (nsteps < 0) return fail(h, VTI_E_PARAM, "nsteps < 0");
    if (!h->model_set) return fail(h, VTI_E_STATE, "model not set (vti_set_model)");
    // y-slabs, one process per slab: the chained TMA form with the s1 rows over NCCL or CUDA IPC
    const bool mp = h->cfg.nranks > 1;
    if (mp && h->group_mode)
        return fail(h, VTI_E_STATE, "a local group's slabs step together: vti_group_step_adjoint");
    if (mp && !h->comm_nccl && !h->peer)
        return fail(h, VTI_E_STATE, "nranks > 1 needs an nccl_id at create time or vti_ipc_connect");
    if (mp && adj_form(h) != ADJ_TMA2)
        return fail(h, VTI_E_UNSUPPORTED, "no two-pass TMA adjoint kernel for this precision and radius pair");
    CU(h, cudaSetDevice(h->cfg.device));
    vti_status s0 = ensure_adj_scratch(h);
    if (s0 != VTI_OK) return s0;
    // the chained TMA two-pass form runs its first pass once per call: each step then writes the
    // next step's s1 (scratch buffers alternate), the last one does not
    static const bool chain_on = !getenv("VTI_ADJ_CHAIN") || atoi(getenv("VTI_ADJ_CHAIN")) != 0;
    const bool chained = adj_form(h) == ADJ_TMA2 && chain_on;
    int sb = 0;
    vti_s *const hv[1] = {h};
    for (int it = 0; it < nsteps; ++it) {
        const bool prep = !chained || it == 0, chain = chained && it + 1 < nsteps;
        vti_status s;
        if (mp && prep) {   // s1 of the state the caller left, then its halo rows
            if ((s = h->es == 8 ? adjoint_prep_t<double>(h, sb) : adjoint_prep_t<float>(h, sb)) != VTI_OK) return s;
            void *b0 = h->adj_s[sb];
            if ((s = h->peer ? rows_exchange_peer(h, b0) : rows_exchange(hv, 1, &b0, true)) != VTI_OK) return s;
        }
        s = h->es == 8 ? adjoint_step_t<double>(h, prep && !mp, sb, chain) : adjoint_step_t<float>(h, prep && !mp, sb, chain);
        if (s != VTI_OK) return s;
        if (mp) h->halo_dirty = true;   // p's halo rows are stale for a later forward step
        if (mp && chain) {
            void *b1 = h->adj_s[1 - sb];
            if ((s = h->peer ? rows_exchange_peer(h, b1) : rows_exchange(hv, 1, &b1, true)) != VTI_OK) return s;
        }
        if (chain) sb ^= 1;
        h->cur = 1 - h->cur;
        h->n -= 1;   // the adjoint runs backward in time
        if (h->rec_set.n > 0) h->rec_steps = std::min(h->rec_cap, h->rec_steps + 1);
        if (h->cfg.check_every > 0 && h->n % h->cfg.check_every == 0) {
            if ((s = check_finite(h)) != VTI_OK) return s;
        }
    }
    return VTI_OK;
}

}  // extern "C"
