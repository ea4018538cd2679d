// vti_adjoint.cu -- the adjoint (transpose) recurrence of the VTI step (the
// backward leg of adjoint-state FWI; PAPER.md l.18-19 names FWI and RTM as the propagator's
// users). The forward step X^{n+1} = M X^n, M = [[g(2 + dt^2 A), -g^2], [I, 0]] with
//   A u = (vx2 L p + vz2 D q, vn2 L p + vz2 D q)            (Eqs. 1-2, 4-5)
// has the transpose recurrence, in the damping-scaled adjoint variable psi = g a,
//   psi^{m-1} = g (2 psi^m - g psi^{m+1} + dt^2 (A^T psi^m + inj)),
//   A^T psi = (L (vx2 psi_p + vn2 psi_q), D^T (vz2 (psi_p + psi_q))),
// L symmetric on the zero exterior and (D^T y)_k = sum_m w^z[k+Rz-m][m] y_{k+Rz-m}. The
// coefficient fields act BEFORE the derivatives here, so a step is two launches: k_adj_prep
// forms s1 = vx2 psi_p + vn2 psi_q and s2 = vz2 (psi_p + psi_q) over the slab, and k_adj_step
// applies L to s1, D^T to s2 and the update. Canonical operation order (bitwise equal to the
// oracle's vto_adjoint_ex): s1 = fma(vx2, psi_p, vn2*psi_q), s2 = vz2*(psi_p + psi_q);
// L = c0 s1; L = fma(c_l, (x+ + x-) + (y+ + y-), L); DT = 0, DT = fma(w[k'][m], s2(k'), DT) for
// m = 0..2Rz, k' = k+Rz-m inside the grid; F_p = L (+ inj), F_q = DT (+ inj);
// psi^{m-1} = g*fma(dt2, F, fma(-g, psi^{m+1}, 2 psi^m)).
//
// k_adj_prep is elementwise; k_adj_step marches z per (tile, z-chunk) with the s1 tile staged in
// shared memory and s2 in a register queue (the forward kernel's structure, plain loads instead
// of its TMA ring). Single-slab handles only (the s1 cross would need the neighbours' psi and
// model rows).
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

// Which form (single slab), measured on B200 with vectorised loads (tools/adjoint_rate.py,
// profiles/r02/adjoint_rate_r02.txt): fp32 one-pass (16-row tiles) vs two-pass: C2 78.1 vs 56.2,
// C3 81.4 vs 53.0, N1 38.7 vs 37.3 Gpoints/s; fp64 one-pass (8-row tiles, the shared-memory
// limit) wins at R_xy = 4 and 6 (C2 36.9 vs 34.3, C5 34.1 vs 25.6) and loses at 8 and 12 (C3
// 20.1 vs 31.2, N1 14.5 vs 19.3). Y-slab groups always run the two-pass form (the s1 halo rows
// come from the neighbours). Env VTI_ADJ_TWO_PASS=1/0 forces either on a single slab.
static bool adj_two_pass(const vti_s *h)
{
    if (h->cfg.nranks > 1) return true;
    static const int env = getenv("VTI_ADJ_TWO_PASS") ? atoi(getenv("VTI_ADJ_TWO_PASS")) : -1;
    return env >= 0 ? env != 0 : (h->es == 8 && h->R >= 8);
}

// Two-pass form, first launch: s1, s2 of the slab (phase 1 of a step).
template <typename T>
static vti_status adjoint_prep_t(vti_s *h)
{
    const int c = h->cur;
    k_adj_prep<T><<<4 * h->sms, 256, 0, h->stream>>>((const T *)h->p_int(c), (const T *)h->q_int(c),
                                                   (const T *)h->in(h->vx2), (const T *)h->in(h->vn2),
                                                   (const T *)h->in(h->vz2), (T *)h->in(h->adj_s[0]),
                                                   (T *)h->in(h->adj_s[1]), h->cfg.nx, h->nyl, h->cfg.nz, h->ys,
                                                   h->zs);
    CU(h, cudaGetLastError());
    return VTI_OK;
}

template <typename T>
static vti_status adjoint_step_t(vti_s *h, bool prep = true)
{
    const int c = h->cur, o = 1 - c;
    const int grid = 4 * h->sms;
    const bool two_pass = adj_two_pass(h);
    T *s1 = nullptr, *s2 = nullptr;
    if (two_pass) {
        s1 = (T *)h->in(h->adj_s[0]);
        s2 = (T *)h->in(h->adj_s[1]);
        if (prep) {
            vti_status st = adjoint_prep_t<T>(h);
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
    return two_pass ? launch_adj_step<T>(h, A, grid) : launch_adj_fused<T>(h, A);
}

}  // namespace

static vti_status ensure_adj_scratch(vti_s *h)
{
    if (!adj_two_pass(h) || h->adj_s[0]) return VTI_OK;
    // the two-pass form's coefficient-weighted fields s1, s2: the slab's geometry, zero halo
    const size_t bytes = h->total_elems() * h->es;
    for (int b = 0; b < 2; ++b) {
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
static vti_status copy_s1_halo(vti_s *h, const vti_s *nb, int side)
{
    const char *src = nb->in(nb->adj_s[0]) + (size_t)(side == 0 ? nb->nyl - nb->R : 0) * nb->ys * nb->es;
    char *dst = h->in(h->adj_s[0]) + (side == 0 ? -(long long)h->R : (long long)h->nyl) * h->ys * h->es;
    // [z][y][x]: R rows are contiguous within each plane; [y][z][x]: one block
    const size_t width = (size_t)h->R * h->ys * h->es;
    const size_t height = h->layout_zyx ? (size_t)h->cfg.nz : 1;
    const size_t spitch = h->layout_zyx ? (size_t)nb->zs * nb->es : width;
    const size_t dpitch = h->layout_zyx ? (size_t)h->zs * h->es : width;
    CU(h, cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, cudaMemcpyDefault, h->stream));
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
            h->cur = 1 - h->cur;
            h->n -= 1;
            h->halo_dirty = true;   // p's halo rows are stale for a later forward step: re-publish then
            if (h->rec_set.n > 0) h->rec_steps = std::min(h->rec_cap, h->rec_steps + 1);
            if (h->cfg.check_every > 0 && h->n % h->cfg.check_every == 0 && (s = check_finite(h)) != VTI_OK)
                return s;
        }
    }
    return VTI_OK;
}

vti_status vti_step_adjoint(vti_t h, int32_t nsteps)
{
    if (!h) return VTI_E_PARAM;
    if (nsteps < 0) return fail(h, VTI_E_PARAM, "nsteps < 0");
    if (!h->model_set) return fail(h, VTI_E_STATE, "model not set (vti_set_model)");
    if (h->cfg.nranks != 1)
        return fail(h, VTI_E_STATE, "vti_step_adjoint is single-slab only; y-slabs: vti_group_step_adjoint");
    CU(h, cudaSetDevice(h->cfg.device));
    vti_status s0 = ensure_adj_scratch(h);
    if (s0 != VTI_OK) return s0;
    for (int it = 0; it < nsteps; ++it) {
        vti_status s = h->es == 8 ? adjoint_step_t<double>(h) : adjoint_step_t<float>(h);
        if (s != VTI_OK) return s;
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
