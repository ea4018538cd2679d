/*
 * oracle/vti_oracle.c -- CPU ORACLE FOR THE VTI STEP.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, tools/oracle_digests.py, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm may load this library. The product path (paper_1410_1387_b200/, the
 * C-ABI in include/vti.h) never calls it and shares no code with it.
 *
 * A plain, slow, obviously correct implementation of one time step of the
 * reduced elastic VTI propagator of arXiv 1410.1387 (PAPER.md = the paper's
 * text; "P:n" = its line n):
 *
 *   Eq. 1  p_tt = vx2 (p_xx + p_yy) + vz2 q_zz + s(t) delta(x - x_i)
 *   Eq. 2  q_tt = vn2 (p_xx + p_yy) + vz2 q_zz
 *   Ricker s = (1 - 2 pi^2 f^2 t^2) exp(-pi^2 f^2 t^2), f = 15 Hz
 *   Eq. 3  u^{n+1} - 2 u^n + u^{n-1} = dt^2 F(u^n),  t^n = n dt
 *   Eq. 4  h^2 (d_xx + d_yy) p ~ w0 p + sum_l w_l (p_{i+l} + p_{i-l} + p_{j+l} + p_{j-l})
 *   Eq. 5  d_zz q ~ sum_{l=-Rz}^{Rz} w^z_{k,l} q_{k+l}   (dz absorbed)
 *   P:87-90          Cerjan damping in the embedding band; zero exterior for
 *                    R_xy points in x, y and R_z in z.
 *
 * Readings where the paper is silent (DESIGN.md "Readings" lists all of them):
 *   c1  z-sum runs l = -Rz..Rz (2Rz+1 weights); row m = l + Rz.
 *   c3  cxy_l = w^xy_l / h^2 computed in double and rounded once to T.
 *   c6  source at the nearest grid point, no cell-volume normalisation,
 *       added into F_p (mask bit 1) and/or F_q (mask bit 2, test mode).
 *   c7  source delay t0: s(t^n) = ricker(n dt - t0).
 *   c8  u^0 = u^{-1} = 0 unless the caller supplies a state; step n uses s(n dt).
 *   c9  damping g = exp(-(alpha (W - d))^2) for d = min(idx, N-1-idx) < W,
 *       product over the three axes, applied as u^{n+1} = g (2u^n - g u^{n-1}
 *       + dt^2 F)  (the "damp next, cur, prev" rule of SPEC.md l.214, exactly
 *       equal on the observable level).
 *   c12 accumulation order (fp32 "canonical" mode): L = c0*p, then for
 *       l = 1..R  L = fma(c_l, (p_{i+l}+p_{i-l}) + (p_{j+l}+p_{j-l}), L);
 *       D = w0*q_{k-Rz}, then D = fma(w_m, q_{k-Rz+m}, D) for m = 1..2Rz;
 *       F = fma(v, L, vz2*D); u^{n+1} = g*fma(dt2, F, fma(-g, u^{n-1}, 2u^n)).
 *   Ricker: x = pi*f*tau, a = x*x, s = (1 - 2a)*exp(-a), in double, then
 *       s_n = (float)(amp*s).
 *
 * Build (by __graft_entry__.build()):  gcc -O2 -ffp-contract=off -fno-fast-math
 *   -fopenmp -shared -fPIC.  No FTZ/DAZ: subnormals are IEEE.
 *   Every point is independent, so results do not depend on the thread count.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
    int32_t nx, ny, nz;          /* interior extents, damping band included (c10) */
    int32_t r_xy, r_z;           /* stencil radii */
    double h;                    /* dx = dy [m] */
    double dt;                   /* [s] */
    int32_t damp_width;          /* W (0 = no damping) */
    double damp_alpha;           /* alpha */
    int32_t src_i, src_j, src_k; /* source grid point (0-based, interior); src_i < 0: none */
    double src_f, src_t0, src_amp;
    int32_t src_mask;            /* 1 = into F_p (Eq. 1), 2 = into F_q, 3 = both */
} vto_params;

/* Ricker wavelet, at time t with delay t0 (reading c7). */
double vto_ricker(double t, double f, double t0)
{
    double x = M_PI * f * (t - t0);
    double a = x * x;
    return (1.0 - 2.0 * a) * exp(-a);
}

/* Cerjan taper value at index idx of an axis with n points (reading c9). */
double vto_damping(int32_t idx, int32_t n, int32_t W, double alpha)
{
    int32_t d = idx < n - 1 - idx ? idx : n - 1 - idx;
    if (d >= W) return 1.0;
    double a = alpha * (double)(W - d);
    return exp(-(a * a));
}

void vto_damping_profile_f32(int32_t n, int32_t W, double alpha, float *out)
{
    for (int32_t i = 0; i < n; ++i) out[i] = (float)vto_damping(i, n, W, alpha);
}

int vto_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

static double now_s(void)
{
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

static int check_params(const vto_params *P)
{
    if (P->nx < 1 || P->ny < 1 || P->nz < 1) return 2;
    if (P->r_xy < 1 || P->r_z < 1 || !(P->h > 0.0) || !(P->dt > 0.0)) return 1;
    if (P->damp_width < 0) return 1;
    if (P->damp_width > 0 && (2 * P->damp_width >= P->nx || 2 * P->damp_width >= P->ny ||
                              2 * P->damp_width >= P->nz)) return 2;
    return 0;
}

/*
 * One definition of the per-point update, instantiated for T = float (the
 * canonical fp32 mode) and T = double. pc[] = the Eq. 4 cross of p^n:
 * pc[0] = p(i,j,k), pc[l] = p(i+l), pc[R+l] = p(i-l), pc[2R+l] = p(j+l),
 * pc[3R+l] = p(j-l); qc[m] = q^n(i,j,k-Rz+m), m = 0..2Rz (Eq. 5).
 */
#define DEFINE_ORACLE(T, SFX, FMA)                                                              \
static void point_##SFX(int R, int Rz, const T *cxy, const T *wzrow, T dt2, T g,               \
                        const T *pc, const T *qc, T pm, T qm, T vx2, T vn2, T vz2,             \
                        int src_bits, T s, int inj_bits, T inj, T *pn, T *qn)                  \
{                                                                                              \
    /* Eq. 4 divided by h^2 (reading c3): L = (p_xx + p_yy) */                                  \
    T L = cxy[0] * pc[0];                                                                      \
    for (int l = 1; l <= R; ++l)                                                               \
        L = FMA(cxy[l], (pc[l] + pc[R + l]) + (pc[2 * R + l] + pc[3 * R + l]), L);             \
    /* Eq. 5: D = q_zz, ascending l = -Rz..Rz */                                               \
    T D = wzrow[0] * qc[0];                                                                    \
    for (int m = 1; m <= 2 * Rz; ++m)                                                          \
        D = FMA(wzrow[m], qc[m], D);                                                           \
    /* Eqs. 1-2: F_p = vx2 L + vz2 D (+ s), F_q = vn2 L + vz2 D */                             \
    T vD = vz2 * D;                                                                            \
    T Fp = FMA(vx2, L, vD);                                                                    \
    if (src_bits & 1) Fp = Fp + s;                                                             \
    if (inj_bits & 1) Fp = Fp + inj;  /* injected trace sample (N4), after the source */       \
    T Fq = FMA(vn2, L, vD);                                                                    \
    if (src_bits & 2) Fq = Fq + s;                                                             \
    if (inj_bits & 2) Fq = Fq + inj;                                                           \
    /* Eq. 3 with Cerjan damping (reading c9) */                                               \
    *pn = g * FMA(dt2, Fp, FMA(-g, pm, (T)2 * pc[0]));                                         \
    *qn = g * FMA(dt2, Fq, FMA(-g, qm, (T)2 * qc[Rz]));                                        \
}                                                                                              \
                                                                                               \
/* Single-point evaluation of step n from caller-gathered neighbourhoods. */                   \
int vto_point_##SFX(const vto_params *P, const T *wxy, const T *wzrow, int32_t i, int32_t j,  \
                    int32_t k, int64_t n, const T *pc, const T *qc, T pm, T qm, T vx2, T vn2,  \
                    T vz2, T *out2)                                                            \
{                                                                                              \
    int rc = check_params(P);                                                                  \
    if (rc) return rc;                                                                         \
    int R = P->r_xy, Rz = P->r_z;                                                              \
    T cxy[64];                                                                                 \
    if (R >= 64) return 1;                                                                     \
    for (int l = 0; l <= R; ++l) cxy[l] = (T)((double)wxy[l] / (P->h * P->h));                 \
    T dt2 = (T)(P->dt * P->dt);                                                                \
    int W = P->damp_width;                                                                     \
    T gx = (T)vto_damping(i, P->nx, W, P->damp_alpha);                                         \
    T gy = (T)vto_damping(j, P->ny, W, P->damp_alpha);                                         \
    T gz = (T)vto_damping(k, P->nz, W, P->damp_alpha);                                         \
    T g = (gx * gy) * gz;                                                                      \
    int bits = (P->src_i == i && P->src_j == j && P->src_k == k) ? P->src_mask : 0;            \
    T s = (T)(P->src_amp * vto_ricker((double)n * P->dt, P->src_f, P->src_t0));                \
    point_##SFX(R, Rz, cxy, wzrow, dt2, g, pc, qc, pm, qm, vx2, vn2, vz2, bits, s, 0, (T)0,    \
                &out2[0], &out2[1]);                                                           \
    return 0;                                                                                  \
}                                                                                              \
                                                                                               \
/*                                                                                             \
 * One step (level n -> n+1) on the whole x-y extent of planes [k0, k0+nk) of the GLOBAL       \
 * grid of P, from caller-supplied plane windows (user layout, x fastest):                     \
 *   p, pm, qm, vx2, vn2, vz2 : [nk][ny][nx]      planes k0 .. k0+nk-1                         \
 *   q                        : [nk+2Rz][ny][nx]  planes k0-Rz .. k0+nk+Rz-1; planes outside     \
 *                              0..nz-1 are never read (zero exterior)                 \
 *   wz                       : the full [nz][2Rz+1] table (row = global plane)                 \
 * Outputs pn, qn : [nk][ny][nx] = u^{n+1} on those planes. Same point_ update as vto_run.      \
 */                                                                                            \
int vto_step_planes_##SFX(const vto_params *P, const T *wxy, const T *wz, int32_t k0,          \
                          int32_t nk, int64_t n, const T *p, const T *q, const T *pm,          \
                          const T *qm, const T *vx2, const T *vn2, const T *vz2, T *pn,        \
                          T *qn)                                                               \
{                                                                                              \
    int rc = check_params(P);                                                                  \
    if (rc) return rc;                                                                         \
    const int R = P->r_xy, Rz = P->r_z, nx = P->nx, ny = P->ny, nz = P->nz;                    \
    if (R >= 64 || Rz >= 64) return 1;                                                         \
    if (k0 < 0 || nk < 0 || k0 + nk > nz) return 2;                                           \
    T cxy[64];                                                                                 \
    for (int l = 0; l <= R; ++l) cxy[l] = (T)((double)wxy[l] / (P->h * P->h));                 \
    const T dt2 = (T)(P->dt * P->dt);                                                          \
    const T s = (T)(P->src_amp * vto_ricker((double)n * P->dt, P->src_f, P->src_t0));          \
    const int64_t plane = (int64_t)nx * ny;                                                    \
    _Pragma("omp parallel for collapse(2)")                                                    \
    for (int kk = 0; kk < nk; ++kk)                                                            \
        for (int j = 0; j < ny; ++j)                                                           \
            for (int i = 0; i < nx; ++i) {                                                     \
                const int k = k0 + kk;                                                         \
                const int64_t u = (int64_t)kk * plane + (int64_t)j * nx + i;                   \
                T pc[4 * 64 + 1], qc[2 * 64 + 1];                                              \
                pc[0] = p[u];                                                                  \
                for (int l = 1; l <= R; ++l) {                                                 \
                    pc[l] = i + l < nx ? p[u + l] : (T)0;                                      \
                    pc[R + l] = i - l >= 0 ? p[u - l] : (T)0;                                  \
                    pc[2 * R + l] = j + l < ny ? p[u + (int64_t)l * nx] : (T)0;                \
                    pc[3 * R + l] = j - l >= 0 ? p[u - (int64_t)l * nx] : (T)0;                \
                }                                                                              \
                for (int m = 0; m <= 2 * Rz; ++m) {                                            \
                    const int kq = k - Rz + m;   /* window plane kk + m */                     \
                    qc[m] = (kq >= 0 && kq < nz) ? q[(int64_t)(kk + m) * plane + (int64_t)j * nx + i] \
                                                 : (T)0;                                       \
                }                                                                              \
                const T gx = (T)vto_damping(i, nx, P->damp_width, P->damp_alpha);              \
                const T gy = (T)vto_damping(j, ny, P->damp_width, P->damp_alpha);              \
                const T gz = (T)vto_damping(k, nz, P->damp_width, P->damp_alpha);              \
                const T g = (gx * gy) * gz;                                                    \
                const int bits = (P->src_i == i && P->src_j == j && P->src_k == k)             \
                                     ? P->src_mask : 0;                                        \
                point_##SFX(R, Rz, cxy, wz + (int64_t)k * (2 * Rz + 1), dt2, g, pc, qc, pm[u], \
                            qm[u], vx2[u], vn2[u], vz2[u], bits, s, 0, (T)0, &pn[u], &qn[u]);  \
            }                                                                                  \
    return 0;                                                                                  \
}                                                                                              \
                                                                                               \
/*                                                                                             \
 * Run nsteps steps starting at time level n0, time index n0, n0+dir, ... (dir = +1, or -1    \
 * for the time-reversed recurrence u^{n-1} = g (2u^n - g u^{n+1} + dt^2 F(u^n)), i.e. the    \
 * same Eq. 3 with the stored level playing u^{n+1}). Arrays are interior-only, user layout    \
 * [z][y][x] (x fastest). On entry p,q = u^{n0}, pm,qm = u^{n0-dir}; on exit p,q =            \
 * u^{n0+dir*nsteps}, pm,qm = u^{n0+dir*(nsteps-1)}. *seconds (if non-NULL) receives the wall  \
 * time of the step loop only.                                                                 \
 * Trace injection (N4, the backward leg of RTM/FWI): at the step that       \
 * evaluates F(u^n), if inj_t_first <= n < inj_t_first + inj_nt, the sample                    \
 * inj_tr[(n - inj_t_first) * n_inj + r] is added into F_p (inj_mask bit 1) and/or F_q (bit 2) \
 * at the distinct GLOBAL point inj_ijk[3r..3r+2], after the Ricker source.                    \
 * Receivers: after each step, u^{new} of the fields in rec_mask (p before q) at rec_ijk[3r..]  \
 * is stored at rec_out[(step * n_rec + r) * nf + f].                                          \
 */                                                                                            \
int vto_run_ex_##SFX(const vto_params *P, const T *wxy, const T *wz, const T *vx2,            \
                     const T *vn2, const T *vz2, T *p, T *q, T *pm, T *qm, int64_t n0,         \
                     int32_t nsteps, int32_t dir, int32_t nthreads, int32_t n_inj,             \
                     const int32_t *inj_ijk, int32_t inj_mask, int32_t inj_nt,                 \
                     int64_t inj_t_first, const T *inj_tr, int32_t n_rec,                      \
                     const int32_t *rec_ijk, int32_t rec_mask, T *rec_out, double *seconds)    \
{                                                                                              \
    int rc = check_params(P);                                                                  \
    if (rc) return rc;                                                                         \
    if (dir != 1 && dir != -1) return 1;                                                       \
    if (n_inj < 0 || n_rec < 0 || (n_inj > 0 && (!inj_ijk || !inj_tr || inj_nt < 0 ||          \
        inj_mask < 1 || inj_mask > 3)) || (n_rec > 0 && (!rec_ijk || !rec_out ||                \
        rec_mask < 1 || rec_mask > 3))) return 1;                                              \
    const int R = P->r_xy, Rz = P->r_z, nx = P->nx, ny = P->ny, nz = P->nz;                    \
    int32_t *inj_at = NULL;  /* interior point -> injection index r, or -1 */                  \
    if (n_inj > 0) {                                                                           \
        inj_at = (int32_t *)malloc(sizeof(int32_t) * (size_t)nx * ny * nz);                   \
        if (!inj_at) return 3;                                                                 \
        for (int64_t u = 0; u < (int64_t)nx * ny * nz; ++u) inj_at[u] = -1;                    \
        for (int r = 0; r < n_inj; ++r) {                                                      \
            const int i = inj_ijk[3 * r], j = inj_ijk[3 * r + 1], k = inj_ijk[3 * r + 2];      \
            if (i < 0 || i >= nx || j < 0 || j >= ny || k < 0 || k >= nz) { free(inj_at); return 2; } \
            const int64_t u = ((int64_t)k * ny + j) * nx + i;                                  \
            if (inj_at[u] >= 0) { free(inj_at); return 1; }  /* points must be distinct */    \
            inj_at[u] = r;                                                                     \
        }                                                                                      \
    }                                                                                          \
    for (int r = 0; r < n_rec; ++r) {                                                          \
        const int i = rec_ijk[3 * r], j = rec_ijk[3 * r + 1], k = rec_ijk[3 * r + 2];          \
        if (i < 0 || i >= nx || j < 0 || j >= ny || k < 0 || k >= nz) { free(inj_at); return 2; } \
    }                                                                                          \
    const int rec_nf = (rec_mask & 1) + ((rec_mask >> 1) & 1);                                 \
    const int64_t X = nx + 2 * R, Y = ny + 2 * R, Z = nz + 2 * Rz;                             \
    const int64_t npad = X * Y * Z;                                                            \
    T *buf[4];                                                                                 \
    for (int b = 0; b < 4; ++b) {                                                              \
        buf[b] = (T *)calloc((size_t)npad, sizeof(T));  /* zero exterior */          \
        if (!buf[b]) { for (int c = 0; c < b; ++c) free(buf[c]); free(inj_at); return 3; }     \
    }                                                                                          \
    T *Pc = buf[0], *Qc = buf[1], *Pm = buf[2], *Qm = buf[3];                                  \
    _Pragma("omp parallel for collapse(2)")                                                    \
    for (int k = 0; k < nz; ++k)                                                               \
        for (int j = 0; j < ny; ++j)                                                           \
            for (int i = 0; i < nx; ++i) {                                                     \
                int64_t u = ((int64_t)k * ny + j) * nx + i;                                    \
                int64_t a = ((int64_t)(k + Rz) * Y + (j + R)) * X + (i + R);                   \
                Pc[a] = p[u]; Qc[a] = q[u]; Pm[a] = pm[u]; Qm[a] = qm[u];                      \
            }                                                                                  \
    T cxy[64];                                                                                 \
    if (R >= 64) { for (int b = 0; b < 4; ++b) free(buf[b]); free(inj_at); return 1; }        \
    for (int l = 0; l <= R; ++l) cxy[l] = (T)((double)wxy[l] / (P->h * P->h));                 \
    const T dt2 = (T)(P->dt * P->dt);                                                          \
    T *gx = (T *)malloc(sizeof(T) * nx), *gy = (T *)malloc(sizeof(T) * ny),                    \
      *gz = (T *)malloc(sizeof(T) * nz);                                                       \
    for (int i = 0; i < nx; ++i) gx[i] = (T)vto_damping(i, nx, P->damp_width, P->damp_alpha);  \
    for (int j = 0; j < ny; ++j) gy[j] = (T)vto_damping(j, ny, P->damp_width, P->damp_alpha);  \
    for (int k = 0; k < nz; ++k) gz[k] = (T)vto_damping(k, nz, P->damp_width, P->damp_alpha);  \
    const int nt = nthreads > 0 ? nthreads : vto_max_threads();                                \
    double t_start = now_s();                                                                  \
    for (int32_t step = 0; step < nsteps; ++step) {                                            \
        const int64_t n = n0 + (int64_t)dir * step;                                            \
        const T s = (T)(P->src_amp * vto_ricker((double)n * P->dt, P->src_f, P->src_t0));      \
        const int inj_row_ok = n_inj > 0 && n >= inj_t_first && n < inj_t_first + inj_nt;     \
        const T *inj_row = inj_row_ok ? inj_tr + (n - inj_t_first) * (int64_t)n_inj : NULL;    \
        _Pragma("omp parallel for collapse(2) schedule(static) num_threads(nt)")                \
        for (int k = 0; k < nz; ++k)                                                           \
            for (int j = 0; j < ny; ++j)                                                       \
                for (int i = 0; i < nx; ++i) {                                                 \
                    T pc[4 * 64 + 1], qc[2 * 64 + 1];                                          \
                    const int64_t a = ((int64_t)(k + Rz) * Y + (j + R)) * X + (i + R);         \
                    const int64_t u = ((int64_t)k * ny + j) * nx + i;                          \
                    pc[0] = Pc[a];                                                             \
                    for (int l = 1; l <= R; ++l) {                                             \
                        pc[l] = Pc[a + l];                                                     \
                        pc[R + l] = Pc[a - l];                                                 \
                        pc[2 * R + l] = Pc[a + l * X];                                         \
                        pc[3 * R + l] = Pc[a - l * X];                                         \
                    }                                                                          \
                    for (int m = 0; m <= 2 * Rz; ++m) qc[m] = Qc[a + (int64_t)(m - Rz) * X * Y]; \
                    const T g = (gx[i] * gy[j]) * gz[k];                                       \
                    const int bits = (P->src_i == i && P->src_j == j && P->src_k == k)         \
                                         ? P->src_mask : 0;                                    \
                    const int ir = inj_row ? inj_at[u] : -1;                                   \
                    T pn, qn;                                                                  \
                    point_##SFX(R, Rz, cxy, wz + (int64_t)k * (2 * Rz + 1), dt2, g, pc, qc,    \
                                Pm[a], Qm[a], vx2[u], vn2[u], vz2[u], bits, s,                 \
                                ir >= 0 ? inj_mask : 0, ir >= 0 ? inj_row[ir] : (T)0, &pn, &qn); \
                    Pm[a] = pn;  /* u^{n+1} overwrites u^{n-1} in place */                     \
                    Qm[a] = qn;                                                                \
                }                                                                              \
        T *t;                                                                                  \
        t = Pc; Pc = Pm; Pm = t;                                                               \
        t = Qc; Qc = Qm; Qm = t;                                                               \
        for (int r = 0; r < n_rec; ++r) {   /* receivers: the level just computed */           \
            const int i = rec_ijk[3 * r], j = rec_ijk[3 * r + 1], k = rec_ijk[3 * r + 2];      \
            const int64_t a = ((int64_t)(k + Rz) * Y + (j + R)) * X + (i + R);                \
            T *o = rec_out + ((int64_t)step * n_rec + r) * rec_nf;                             \
            if (rec_mask & 1) *o++ = Pc[a];                                                    \
            if (rec_mask & 2) *o = Qc[a];                                                      \
        }                                                                                      \
    }                                                                                          \
    double t_end = now_s();                                                                    \
    if (seconds) *seconds = t_end - t_start;                                                   \
    _Pragma("omp parallel for collapse(2)")                                                    \
    for (int k = 0; k < nz; ++k)                                                               \
        for (int j = 0; j < ny; ++j)                                                           \
            for (int i = 0; i < nx; ++i) {                                                     \
                int64_t u = ((int64_t)k * ny + j) * nx + i;                                    \
                int64_t a = ((int64_t)(k + Rz) * Y + (j + R)) * X + (i + R);                   \
                p[u] = Pc[a]; q[u] = Qc[a]; pm[u] = Pm[a]; qm[u] = Qm[a];                      \
            }                                                                                  \
    free(gx); free(gy); free(gz);                                                              \
    free(inj_at);                                                                              \
    for (int b = 0; b < 4; ++b) free(buf[b]);                                                  \
    return 0;                                                                                  \
}                                                                                              \
                                                                                               \
/*                                                                                             \
 * Adjoint (transpose) recurrence (the backward leg of adjoint-state FWI).   \
 * The forward step is X^{n+1} = M X^n on X = (u^n, u^{n-1}), M = [[g(2 + dt^2 A), -g^2],        \
 * [I, 0]], with A u = (vx2 L p + vz2 D q, vn2 L p + vz2 D q) (Eqs. 1-2, 4-5). Its transpose    \
 * M^T, written in the damping-scaled adjoint variable psi = g a, has the same form with A^T:    \
 *   psi^{m-1} = g (2 psi^m - g psi^{m+1} + dt^2 (A^T psi^m + inj)),                           \
 *   A^T psi = (L (vx2 psi_p + vn2 psi_q), D^T (vz2 (psi_p + psi_q))),                          \
 * L symmetric on the zero exterior, (D^T y)_k = sum_m w^z[k+Rz-m][m] y_{k+Rz-m} (Eq. 5's rows   \
 * transposed). Canonical order: s1 = fma(vx2, psi_p, vn2*psi_q); s2 = vz2*(psi_p + psi_q);      \
 * L(s1) as in point_; DT = 0, then for m = 0..2Rz with k' = k+Rz-m inside the grid             \
 * DT = fma(w^z[k'][m], s2(k'), DT); F_p = L (+ inj), F_q = DT (+ inj);                         \
 * psi^{m-1} = g*fma(dt2, F, fma(-g, psi^{m+1}, 2*psi^m)). No Ricker term (adjoint sources come   \
 * as injected traces, row = time index m - inj_t_first); receivers record psi^{m-1}.           \
 * On entry p,q = psi^{m0}, pm,qm = psi^{m0+1}; on exit p,q = psi^{m0-nsteps}, pm,qm = the      \
 * level after it. Injection points must be distinct.                                           \
 */                                                                                            \
int vto_adjoint_ex_##SFX(const vto_params *P, const T *wxy, const T *wz, const T *vx2,        \
                         const T *vn2, const T *vz2, T *p, T *q, T *pm, T *qm, int64_t m0,     \
                         int32_t nsteps, int32_t nthreads, int32_t n_inj,                      \
                         const int32_t *inj_ijk, int32_t inj_mask, int32_t inj_nt,             \
                         int64_t inj_t_first, const T *inj_tr, int32_t n_rec,                  \
                         const int32_t *rec_ijk, int32_t rec_mask, T *rec_out)                 \
{                                                                                              \
    int rc = check_params(P);                                                                  \
    if (rc) return rc;                                                                         \
    if (n_inj < 0 || n_rec < 0 || (n_inj > 0 && (!inj_ijk || !inj_tr || inj_nt < 0 ||          \
        inj_mask < 1 || inj_mask > 3)) || (n_rec > 0 && (!rec_ijk || !rec_out ||                \
        rec_mask < 1 || rec_mask > 3))) return 1;                                              \
    const int R = P->r_xy, Rz = P->r_z, nx = P->nx, ny = P->ny, nz = P->nz;                    \
    if (R >= 64 || Rz >= 64) return 1;                                                         \
    const int64_t N = (int64_t)nx * ny * nz;                                                   \
    for (int r = 0; r < n_rec; ++r) {                                                          \
        const int i = rec_ijk[3 * r], j = rec_ijk[3 * r + 1], k = rec_ijk[3 * r + 2];          \
        if (i < 0 || i >= nx || j < 0 || j >= ny || k < 0 || k >= nz) return 2;                \
    }                                                                                          \
    int32_t *inj_at = (int32_t *)malloc(sizeof(int32_t) * (size_t)N);                          \
    T *s1 = (T *)calloc((size_t)N, sizeof(T)), *s2 = (T *)calloc((size_t)N, sizeof(T));         \
    T *nxt_p = (T *)malloc(sizeof(T) * (size_t)N), *nxt_q = (T *)malloc(sizeof(T) * (size_t)N);  \
    if (!inj_at || !s1 || !s2 || !nxt_p || !nxt_q) {                                           \
        free(inj_at); free(s1); free(s2); free(nxt_p); free(nxt_q); return 3;                  \
    }                                                                                          \
    for (int64_t u = 0; u < N; ++u) inj_at[u] = -1;                                            \
    for (int r = 0; r < n_inj; ++r) {                                                          \
        const int i = inj_ijk[3 * r], j = inj_ijk[3 * r + 1], k = inj_ijk[3 * r + 2];          \
        const int64_t u = ((int64_t)k * ny + j) * nx + i;                                      \
        if (i < 0 || i >= nx || j < 0 || j >= ny || k < 0 || k >= nz || inj_at[u] >= 0) {      \
            free(inj_at); free(s1); free(s2); free(nxt_p); free(nxt_q);                        \
            return (i < 0 || i >= nx || j < 0 || j >= ny || k < 0 || k >= nz) ? 2 : 1;         \
        }                                                                                      \
        inj_at[u] = r;                                                                         \
    }                                                                                          \
    T cxy[64];                                                                                 \
    for (int l = 0; l <= R; ++l) cxy[l] = (T)((double)wxy[l] / (P->h * P->h));                 \
    const T dt2 = (T)(P->dt * P->dt);                                                          \
    const int nt = nthreads > 0 ? nthreads : vto_max_threads();                                \
    const int rec_nf = (rec_mask & 1) + ((rec_mask >> 1) & 1);                                 \
    T *cp = p, *cq = q, *op = pm, *oq = qm;   /* psi^m and psi^{m+1} */                        \
    for (int32_t step = 0; step < nsteps; ++step) {                                            \
        const int64_t m = m0 - step;                                                           \
        const T *inj_row = (n_inj > 0 && m >= inj_t_first && m < inj_t_first + inj_nt)         \
                               ? inj_tr + (m - inj_t_first) * (int64_t)n_inj : NULL;           \
        _Pragma("omp parallel for num_threads(nt)")                                            \
        for (int64_t u = 0; u < N; ++u) {                                                      \
            s1[u] = FMA(vx2[u], cp[u], vn2[u] * cq[u]);                                        \
            s2[u] = vz2[u] * (cp[u] + cq[u]);                                                  \
        }                                                                                      \
        _Pragma("omp parallel for collapse(2) num_threads(nt)")                                \
        for (int k = 0; k < nz; ++k)                                                           \
            for (int j = 0; j < ny; ++j)                                                       \
                for (int i = 0; i < nx; ++i) {                                                 \
                    const int64_t u = ((int64_t)k * ny + j) * nx + i;                          \
                    T L = cxy[0] * s1[u];                                                      \
                    for (int l = 1; l <= R; ++l) {                                             \
                        const T xp = i + l < nx ? s1[u + l] : (T)0;                            \
                        const T xm = i - l >= 0 ? s1[u - l] : (T)0;                            \
                        const T yp = j + l < ny ? s1[u + (int64_t)l * nx] : (T)0;              \
                        const T ym = j - l >= 0 ? s1[u - (int64_t)l * nx] : (T)0;              \
                        L = FMA(cxy[l], (xp + xm) + (yp + ym), L);                             \
                    }                                                                          \
                    T DT = (T)0;                                                               \
                    for (int mm = 0; mm <= 2 * Rz; ++mm) {                                     \
                        const int kk = k + Rz - mm;                                            \
                        if (kk < 0 || kk >= nz) continue;                                      \
                        DT = FMA(wz[(int64_t)kk * (2 * Rz + 1) + mm],                          \
                                 s2[((int64_t)kk * ny + j) * nx + i], DT);                     \
                    }                                                                          \
                    T Fp = L, Fq = DT;                                                         \
                    const int ir = inj_row ? inj_at[u] : -1;                                   \
                    if (ir >= 0 && (inj_mask & 1)) Fp = Fp + inj_row[ir];                      \
                    if (ir >= 0 && (inj_mask & 2)) Fq = Fq + inj_row[ir];                      \
                    const T g = ((T)vto_damping(i, nx, P->damp_width, P->damp_alpha) *         \
                                 (T)vto_damping(j, ny, P->damp_width, P->damp_alpha)) *        \
                                (T)vto_damping(k, nz, P->damp_width, P->damp_alpha);           \
                    nxt_p[u] = g * FMA(dt2, Fp, FMA(-g, op[u], (T)2 * cp[u]));                 \
                    nxt_q[u] = g * FMA(dt2, Fq, FMA(-g, oq[u], (T)2 * cq[u]));                 \
                }                                                                              \
        memcpy(op, nxt_p, sizeof(T) * (size_t)N);   /* psi^{m-1} over psi^{m+1} */              \
        memcpy(oq, nxt_q, sizeof(T) * (size_t)N);                                              \
        T *t;                                                                                  \
        t = cp; cp = op; op = t;                                                               \
        t = cq; cq = oq; oq = t;                                                               \
        for (int r = 0; r < n_rec; ++r) {                                                      \
            const int64_t u = ((int64_t)rec_ijk[3 * r + 2] * ny + rec_ijk[3 * r + 1]) * nx +   \
                              rec_ijk[3 * r];                                                  \
            T *o = rec_out + ((int64_t)step * n_rec + r) * rec_nf;                             \
            if (rec_mask & 1) *o++ = cp[u];                                                    \
            if (rec_mask & 2) *o = cq[u];                                                      \
        }                                                                                      \
    }                                                                                          \
    if (cp != p) {   /* results back in the caller's arrays: p,q current, pm,qm the other */   \
        memcpy(nxt_p, p, sizeof(T) * (size_t)N); memcpy(p, cp, sizeof(T) * (size_t)N);        \
        memcpy(pm, nxt_p, sizeof(T) * (size_t)N);                                              \
        memcpy(nxt_q, q, sizeof(T) * (size_t)N); memcpy(q, cq, sizeof(T) * (size_t)N);        \
        memcpy(qm, nxt_q, sizeof(T) * (size_t)N);                                              \
    }                                                                                          \
    free(inj_at); free(s1); free(s2); free(nxt_p); free(nxt_q);                                \
    return 0;                                                                                  \
}                                                                                              \
                                                                                               \
/* Forward run, Ricker source only (the path every pin in tests/test_oracle_pins.py drives). */ \
int vto_run_##SFX(const vto_params *P, const T *wxy, const T *wz, const T *vx2,               \
                  const T *vn2, const T *vz2, T *p, T *q, T *pm, T *qm, int64_t n0,            \
                  int32_t nsteps, int32_t nthreads, double *seconds)                           \
{                                                                                              \
    return vto_run_ex_##SFX(P, wxy, wz, vx2, vn2, vz2, p, q, pm, qm, n0, nsteps, 1, nthreads,  \
                            0, NULL, 0, 0, 0, NULL, 0, NULL, 0, NULL, seconds);                \
}

DEFINE_ORACLE(float, f32, fmaf)
DEFINE_ORACLE(double, f64, fma)
