/*
 * vti.h -- C ABI of the B200-native VTI propagator step (arXiv 1410.1387).
 *
 * One time step advances the coupled p/q wavefields of the reduced elastic
 * VTI system (Eqs. 1-2) with the centred leapfrog of Eq. 3
 * (l.47-53):  u^{n+1} = g (2 u^n - g u^{n-1} + dt^2 F(u^n)),  u = (p, q),
 *   F_p = vx2 L(p) + vz2 D(q) + s(t^n) delta(x - x_src),
 *   F_q = vn2 L(p) + vz2 D(q),
 * with L the symmetric R_xy-radius x-y Laplacian of Eq. 4 (l.74-78), D the
 * variable-spacing z second derivative of Eq. 5 (l.82-87, 2R_z+1 weights per
 * plane k), s the Ricker wavelet of l.44-45, g the separable Cerjan taper of
 * l.87-89 and a zero exterior (l.89-90).
 *
 * Conventions (all entry points):
 *  - Every call returns a vti_status; on error the handle (if any) keeps a
 *    message readable with vti_last_error(). No call aborts the process.
 *  - Ownership: the library owns all device memory behind a vti_t. Caller
 *    buffers are borrowed for the duration of the call only (copied in/out).
 *    Pointers may be host memory or device memory (UVA): the library detects
 *    which with cudaPointerGetAttributes. Before reading or writing a caller's
 *    device buffer the library synchronises the device, so buffers produced
 *    on any stream are safe to pass; such calls are setup-time, not hot-path.
 *  - User layout of every 3-D array: [z][y][x], x fastest,
 *    interior points only (no halo, no padding). With nranks > 1 an array
 *    covers this rank's y-slab only: [nz][ny_local][nx] (see vti_slab).
 *  - Precision: fp32 (default; the BASELINE.json path) or fp64 (cfg.precision
 *    = 64) storage and arithmetic, in one fixed "canonical"
 *    operation order (reading c12), so results are bitwise
 *    reproducible. Array entry points come in pairs: the plain name takes
 *    float*, the _f64 name double*; calling the other precision's entry point
 *    is VTI_E_PARAM.
 *  - Threading: a handle is single-writer; calls on one handle must not race.
 *  - Asynchrony: vti_step enqueues work on the handle's stream and returns;
 *    vti_get_fields / vti_sync synchronise.
 */
#ifndef VTI_H
#define VTI_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VTI_ABI_VERSION 5
#define VTI_IPC_BYTES 512   /* size of a vti_ipc_export blob */

typedef struct vti_s *vti_t;

typedef enum {
    VTI_OK = 0,
    VTI_E_PARAM = 1,        /* bad scalar argument: radius, h, dt, mask, NULL pointer */
    VTI_E_GEOMETRY = 2,     /* bad extents: nz < 2R_z+1, 2W >= extent, y-slabs thinner than R_xy (l.59, l.136) */
    VTI_E_MODEL = 3,        /* vz2 <= 0 or non-finite model value */
    VTI_E_ANISO = 4,        /* reserved: strict eps >= delta check (warn-only by default) */
    VTI_E_INSTABILITY = 5,  /* non-finite wavefield detected (check_every > 0) */
    VTI_E_INDEX = 6,        /* source or plane range outside the domain */
    VTI_E_CUDA = 7,         /* CUDA runtime / driver failure (message has the CUDA error) */
    VTI_E_COMM = 8,         /* halo transport failure: NCCL, CUDA IPC or stream memory operations (nranks > 1) */
    VTI_E_STATE = 9,        /* call not valid in the handle's current state */
    VTI_E_UNSUPPORTED = 10  /* (r_xy, r_z) pair not compiled into this library */
} vti_status;

typedef struct {
    int32_t nx, ny, nz;     /* GLOBAL interior extents incl. the damping band (c10); ny global */
    double h;               /* dx = dy [m] (Eq. 4 is for h^2-scaled weights) */
    int32_t r_xy, r_z;      /* radii; compiled pairs: (4,4) (8,4) (6,6) (12,8) */
    double dt;              /* time step [s]; used as float32 dt^2 = (float)(dt*dt) */
    int32_t damp_width;     /* Cerjan width W in points per face (0 = off) */
    double damp_alpha;      /* Cerjan alpha (default 0.015) */
    int32_t device;         /* CUDA device ordinal */
    void *stream;           /* cudaStream_t to run on, or NULL (library creates one) */
    int32_t rank, nranks;   /* y-slab index / count; (0, 1) on a single GPU */
    const void *nccl_id;    /* 128-byte ncclUniqueId shared by all ranks (nranks > 1);
                               NULL with nranks > 1 = "local group" mode (vti_group_step) */
    int32_t check_every;    /* > 0: test for non-finite values every this many steps */
    int32_t precision;      /* 32 (or 0) = fp32, 64 = fp64 */
} vti_config;

typedef struct {
    int32_t y0, ny_local;   /* this rank's rows [y0, y0 + ny_local) of the global grid */
    int32_t nx_pad;         /* padded x stride (floats) of the internal layout */
    int32_t layout;         /* 0: internal [z][y][x] (default), 1: [y][z][x] (env VTI_LAYOUT=yzx) */
    int32_t tile_x, tile_y; /* CTA tile of the step kernel */
    int32_t rows_per_thread, producer_warp; /* step-kernel variant (see vti_set_variant) */
    int32_t points_per_thread; /* consecutive x points per thread: 4, or 2 (float2 / double2 variants) */
    int32_t small_kernel;   /* 1: small-grid kernel (one CTA per tile-plane item, all loads at once) */
    int32_t zchunk;         /* planes per work item */
    int32_t grid;           /* CTAs launched per step (persistent) */
    int32_t work_items;     /* tiles x z-chunks per step */
    int32_t launches_per_step; /* library kernels per step: 1 (one slab, or a fused peer step); otherwise
                                  edge + interior step kernels (+ one pack and one unpack kernel per
                                  neighbour with NCCL) */
    int64_t device_bytes;   /* device memory owned by the handle */
    int64_t time_index;     /* n: fields hold u^n and u^{n-1} */
    int32_t steps_per_launch; /* > 1: the multi-step small-grid kernel, one cooperative launch per
                                 vti_step call of up to this many steps (single slab, small grids) */
} vti_info;

/* Library ABI version (VTI_ABI_VERSION). */
int32_t vti_abi_version(void);

/* Static text for a status code. */
const char *vti_status_string(vti_status s);

/* y-slab of rank cfg->rank: rows [*y0, *y0 + *ny_local), the first ny % nranks
 * ranks getting one extra row. Host-only; never touches the GPU. */
vti_status vti_slab(const vti_config *cfg, int32_t *y0, int32_t *ny_local);

typedef struct {
    int32_t y0, ny_local;            /* this rank's slab (vti_slab) */
    int32_t ntx, nty;                /* 64 x tile_y tiles over the slab */
    int32_t edge_lo, edge_hi;        /* nranks > 1: tile rows [0, edge_lo) and [edge_hi, nty) are the edge launch
                                        (every tile row touching the first or last r_xy rows); [edge_lo, edge_hi)
                                        the interior launch */
    int32_t zchunk;                  /* planes per work item, single launch over all tile rows */
    int32_t zchunk_edge, zchunk_inner; /* the same for the edge / interior launches */
    int32_t items, grid;             /* work items and CTAs of the single launch */
} vti_plan_info;

/* The schedule the library would use for cfg with tile height tile_y on a GPU
 * with `sms` multiprocessors and `ctas_per_sm` resident step CTAs per SM.
 * Host-only (never touches the GPU): the same functions vti_create uses.
 * Errors: PARAM / GEOMETRY as vti_create's validation. */
vti_status vti_plan(const vti_config *cfg, int32_t tile_y, int32_t sms, int32_t ctas_per_sm, vti_plan_info *out);

/* Fill out[128] with a fresh ncclUniqueId (rank 0 calls it, then broadcasts).
 * VTI_E_COMM if NCCL cannot be loaded. */
vti_status vti_nccl_unique_id(void *out128);

/*
 * Create a propagator. w_xy: R_xy+1 float32 weights of Eq. 4 for the
 * h^2-scaled Laplacian (w_xy[0] = centre). w_z: nz*(2R_z+1) float32 weights of
 * Eq. 5, row k = plane k (global), column m = l + R_z for l = -R_z..R_z, dz
 * absorbed (1/m^2). Fields start at zero (u^0 = u^{-1} = 0, reading c8), the
 * model at zero (must be set before stepping), no source.
 * Errors: PARAM, GEOMETRY, UNSUPPORTED, CUDA, COMM. On error *out = NULL.
 */
vti_status vti_create(vti_t *out, const vti_config *cfg, const float *w_xy, const float *w_z);

/* Same with double weights; needs cfg->precision = 64 (with vti_create an
 * fp64 handle gets the float weights widened exactly). */
vti_status vti_create_f64(vti_t *out, const vti_config *cfg, const double *w_xy, const double *w_z);

/* Upload this rank's model slab (vx2 = nu_x^2, vn2 = nu_n^2, vz2 = nu_z^2 [m^2/s^2],
 * PAPER.md l.39-43), each [nz][ny_local][nx]. Errors: PARAM (NULL), MODEL
 * (vz2 <= 0 or non-finite anywhere), CUDA. vn2 > vx2 (eps < delta) is
 * accepted; vti_model_warnings() reports how many points had it (reading c5). */
vti_status vti_set_model(vti_t h, const float *vx2, const float *vn2, const float *vz2);

/* Same for planes [k0, k0+nk) only: arrays are [nk][ny_local][nx]. */
vti_status vti_set_model_planes(vti_t h, int32_t k0, int32_t nk, const float *vx2,
                                const float *vn2, const float *vz2);
vti_status vti_set_model_f64(vti_t h, const double *vx2, const double *vn2, const double *vz2);
vti_status vti_set_model_planes_f64(vti_t h, int32_t k0, int32_t nk, const double *vx2,
                                    const double *vn2, const double *vz2);

/* Points with vn2 > vx2 (eps < delta) seen by vti_set_model* so far. */
int64_t vti_model_warnings(vti_t h);

/*
 * Point source s(t) delta(x - x_src) of Eq. 1: Ricker wavelet
 * s(t^n) = amp * (1 - 2a) exp(-a), a = (pi f (n dt - t0))^2, evaluated in
 * double on the host and rounded once to float32 per step; added into F_p
 * (field_mask bit 1, Eq. 1) and/or F_q (bit 2, test mode) at GLOBAL grid
 * point (i, j, k) (reading c6). One source per handle: a second call
 * replaces the first. Errors: INDEX (outside the grid), PARAM (mask not 1..3).
 * A rank whose slab does not hold row j stores the source but never injects it.
 */
vti_status vti_add_source(vti_t h, int32_t i, int32_t j, int32_t k, double f, double t0,
                          double amp, int32_t field_mask);

/* Replace the state: p,q = u^n and pm,qm = u^{n-1} (each [nz][ny_local][nx]),
 * and set the time index to n. NULL pm/qm = zero. Errors: PARAM, CUDA. */
vti_status vti_set_fields(vti_t h, const float *p, const float *q, const float *pm,
                          const float *qm, int64_t time_index);

/* Planes [k0, k0+nk) of the state (time index unchanged; pm/qm may be NULL = zero). */
vti_status vti_set_fields_planes(vti_t h, int32_t k0, int32_t nk, const float *p, const float *q,
                                 const float *pm, const float *qm);
vti_status vti_set_fields_f64(vti_t h, const double *p, const double *q, const double *pm,
                              const double *qm, int64_t time_index);
vti_status vti_set_fields_planes_f64(vti_t h, int32_t k0, int32_t nk, const double *p, const double *q,
                                     const double *pm, const double *qm);

/* Advance nsteps time steps (async on the handle's stream). With nranks > 1
 * every rank must call it with the same nsteps: p's R_xy boundary rows are
 * exchanged every step, through the neighbours' halo rows directly after
 * vti_ipc_connect (the edge launch stores them over NVLink), else with NCCL
 * (nccl_id at create time). Errors: STATE (model unset, local-group handle,
 * or nranks > 1 with neither transport), INSTABILITY (check_every), CUDA, COMM. */
vti_status vti_step(vti_t h, int32_t nsteps);

/* Build now whatever vti_step would otherwise build on its first call (the
 * 32- and 128-step CUDA graphs of small single-slab grids, both level parities), so
 * a timed region does not pay for graph capture and instantiation. Nothing is
 * executed; the state and the time index are unchanged. No-op when the handle
 * does not replay graphs. Errors: STATE (model unset), CUDA. */
vti_status vti_prepare(vti_t h);

/* vti_step bracketed by CUDA events on the handle's stream; *ms = device time
 * of the nsteps steps (synchronises). */
vti_status vti_step_timed(vti_t h, int32_t nsteps, float *ms);

/* Local group: n handles created with the same cfg except rank = 0..n-1,
 * nranks = n and nccl_id = NULL (any devices, one process). Steps them in
 * lockstep with the fused peer-memory halo transport between the handles'
 * own buffers (the protocol of vti_ipc_connect, without IPC). */
vti_status vti_group_step(vti_t *hs, int32_t n, int32_t nsteps);

/* Local group with the STAGED transport of the NCCL path instead of peer stores:
 * per step, the edge launch, a pack of the R_xy boundary rows into send buffers,
 * the exchange on each handle's comm stream (device copies from the neighbours'
 * send buffers in place of ncclSend/ncclRecv) + unpack into the halo rows,
 * overlapped with the interior launch; the next step waits on the exchanges.
 * The same handles, schedules and pack/unpack kernels as vti_step with an
 * nccl_id, so one GPU can check that path against the oracle. Results are
 * bitwise those of a single slab. Errors: PARAM, STATE, CUDA. */
vti_status vti_group_step_staged(vti_t *hs, int32_t n, int32_t nsteps);

/* Copy out u^n (level 0) or the stored u^{n-1} (level 1) of this slab into
 * p, q ([nz][ny_local][nx]; either may be NULL). Synchronises.
 * Note: with damping, the stored u^{n-1} is the undamped previous level
 * (reading c9). Errors: PARAM, CUDA. */
vti_status vti_get_fields(vti_t h, float *p, float *q, int32_t level);

/* Planes [k0, k0+nk) of vti_get_fields. */
vti_status vti_get_fields_planes(vti_t h, int32_t k0, int32_t nk, float *p, float *q, int32_t level);
vti_status vti_get_fields_f64(vti_t h, double *p, double *q, int32_t level);
vti_status vti_get_fields_planes_f64(vti_t h, int32_t k0, int32_t nk, double *p, double *q, int32_t level);

/*
 * Snapshot (N4: the forward wavefields an RTM imaging condition correlates with the backward
 * leg; "snapshot planes/volumes at a cadence"): ENQUEUE, on the handle's
 * stream and without synchronising, a copy of planes [k0, k0+nk) of u^n (level 0) or the
 * stored u^{n-1} (level 1) into p, q ([nk][ny_local][nx], either may be NULL). The buffers
 * must be device-writable (device memory, or mapped page-locked host memory) and stay valid
 * until the stream reaches the copy (vti_sync). Ordered with vti_step, so a snapshot after
 * step n holds level n. Errors: PARAM (level, precision, buffer not device-writable), INDEX.
 */
vti_status vti_snapshot_async(vti_t h, int32_t k0, int32_t nk, float *p, float *q, int32_t level);
vti_status vti_snapshot_async_f64(vti_t h, int32_t k0, int32_t nk, double *p, double *q, int32_t level);

/*
 * Receivers (the trace-extraction hook of RTM/FWI,
 * PAPER.md l.18-19): after every subsequent step, the wavefield(s) in
 * field_mask (1 = p, 2 = q, 3 = both) at the n GLOBAL grid points ijk[3r..3r+2]
 * are written to a device trace buffer, one row per step, up to capacity_steps
 * rows (recording then stops silently). The gather is fused into the step
 * kernel's store epilogue (no extra launch; CUDA-graph replays of small grids
 * stay on). Only the receivers inside this rank's slab are kept
 * (vti_receiver_info lists them); duplicates are allowed. A new call replaces the
 * set and restarts the recording. n = 0 removes all receivers.
 * Errors: PARAM, INDEX, CUDA.
 */
vti_status vti_set_receivers(vti_t h, int32_t n, const int32_t *ijk, int32_t field_mask, int32_t capacity_steps);

/*
 * Trace injection (N4: the backward leg of RTM/FWI re-injects recorded traces,
 * PAPER.md l.18-19; the forcing term of Eq. 1 generalised to n points): at the
 * step that evaluates F(u^n) (time index n, also after vti_reverse), if
 * t_first <= n < t_first + nt, traces[(n - t_first) * n + r] is added into F_p
 * (field_mask bit 1) and/or F_q (bit 2) at the GLOBAL grid point ijk[3r..3r+2],
 * after the Ricker source of vti_add_source (same operation order as the oracle).
 * traces: [nt][n] of the handle's precision, host or device pointer, copied
 * (the library owns the device copy). Points must be distinct; only those in
 * this rank's slab are injected. A new call replaces the set; n = 0 removes it.
 * Errors: PARAM (NULL, mask, nt < 0, duplicate points, wrong precision), INDEX, CUDA.
 */
vti_status vti_set_injection(vti_t h, int32_t n, const int32_t *ijk, int32_t field_mask, int32_t nt,
                             int64_t t_first, const float *traces);
vti_status vti_set_injection_f64(vti_t h, int32_t n, const int32_t *ijk, int32_t field_mask, int32_t nt,
                                 int64_t t_first, const double *traces);

/* Local receiver count, rows recorded so far, and (ids != NULL, n_local entries)
 * the caller's index of each local receiver. */
vti_status vti_receiver_info(vti_t h, int32_t *n_local, int32_t *steps_recorded, int32_t *ids);

/* Copy the recorded traces, [steps_recorded][n_local][nf] (nf = fields in the
 * mask, p before q), to out (host or device). Synchronises. */
vti_status vti_get_traces(vti_t h, float *out);
vti_status vti_get_traces_f64(vti_t h, double *out);

/*
 * Time reversal (N4, the backward propagation of RTM): swap the two stored
 * levels, so the next vti_step applies Eq. 3 backwards,
 * u^{n-1} = g (2 u^n - g u^{n+1} + dt^2 F(u^n)), with s(t^n) and the injection
 * row of time index n at the current level and the time index decreasing.
 * Without damping (W = 0) this is the exact inverse of forward stepping up to
 * rounding; calling it again restores forward stepping. vti_time_index() is the
 * current level throughout. Note: this is time reversal of the SAME operator, not
 * its adjoint (transpose): F's z operator D has per-plane weights w^z[k] (Eq. 5),
 * so D^T != D on a variable-dz grid, and the vx2/vn2/vz2 factors multiply on the
 * other side in A^T: vti_step_adjoint runs the transpose recurrence.
 */
vti_status vti_reverse(vti_t h);

/*
 * Adjoint (transpose) stepping (N4: the backward leg of adjoint-state FWI).
 * The forward step X^{n+1} = M X^n on X = (u^n, u^{n-1}), M = [[g(2 + dt^2 A), -g^2], [I, 0]],
 * A u = (vx2 L p + vz2 D q, vn2 L p + vz2 D q) (Eqs. 1-2, 4-5), has the transpose recurrence,
 * in the damping-scaled adjoint variable psi = g a:
 *   psi^{m-1} = g (2 psi^m - g psi^{m+1} + dt^2 (A^T psi^m + inj)),
 *   A^T psi = (L (vx2 psi_p + vn2 psi_q), D^T (vz2 (psi_p + psi_q))),
 * with (D^T y)_k = sum_m w^z[k+Rz-m][m] y_{k+Rz-m}. The handle's state is (psi^m, psi^{m+1})
 * (level 0 / level 1 of vti_get_fields / vti_set_fields), the time index m; each step lowers it
 * by one. Adjoint sources are injected traces (vti_set_injection, row = m - t_first, added
 * after the operator); receivers (vti_set_receivers) record psi^{m-1}; the Ricker source of
 * vti_add_source is not applied. Then <M^K X, Y> = <X, (M^T)^K Y> (the dot-product test of
 * tests/test_adjoint_gpu.py). Kernels (csrc/vti_adjoint.cu): a TMA one-pass form (the coefficient
 * products formed in the stencil kernel) or a chained two-pass form (s1 = vx2 psi_p + vn2 psi_q
 * written once per call, then each step's kernel also writes the next step's s1), whichever
 * measured faster for the precision and radii. nranks > 1, one process per slab: the chained
 * two-pass form with each step's s1 boundary rows exchanged over the handle's transport -- NCCL
 * (pack, send/recv, unpack) or, after vti_ipc_connect, CUDA IPC (rows packed straight into the
 * neighbours' receive buffers, ordered by flag words); every rank calls it with the same nsteps.
 * Local groups: vti_group_step_adjoint. Bitwise equal to the oracle's vto_adjoint_ex. Errors:
 * STATE (model unset; a local-group handle; nranks > 1 without a transport), UNSUPPORTED
 * (nranks > 1 and no two-pass kernel for the radii), PARAM, CUDA, COMM, INSTABILITY.
 */
vti_status vti_step_adjoint(vti_t h, int32_t nsteps);

/* The adjoint step for a local group of y-slab handles (created as for vti_group_step, any
 * devices): the chained two-pass form, each slab's R_xy boundary rows of s1 exchanged between
 * steps with the NCCL path's pack / copy / unpack sequence (copies between the slabs' send and
 * receive buffers standing in for send/recv); results are bitwise those of one slab. Errors:
 * PARAM, STATE, CUDA. */
vti_status vti_group_step_adjoint(vti_t *hs, int32_t n, int32_t nsteps);

/* +1 (forward) or -1 (after an odd number of vti_reverse calls). */
int32_t vti_direction(vti_t h);

/*
 * Fused peer-memory halo transport for nranks > 1 (no NCCL, no pack, copy or
 * unpack): the edge step launch stores p^{n+1} of this slab's first / last R_xy
 * rows both locally and straight into rank-1's top / rank+1's bottom halo rows
 * through CUDA-IPC peer pointers (NVLink), and flag words written and waited on
 * with stream memory operations order the steps.
 * vti_ipc_export writes this rank's VTI_IPC_BYTES blob (IPC handles of both p
 * buffers and the flag words, plus the slab geometry). After exchanging blobs
 * (e.g. an all-gather over the job's process group), every rank calls
 * vti_ipc_connect with the blob of rank-1 (lo) and rank+1 (hi), NULL at the
 * ends. A handle created with an nccl_id that is then connected uses this
 * transport instead of NCCL. Both calls are collective in effect: all ranks
 * must connect before the next vti_step, and all ranks must then step together.
 * Errors: STATE (nranks < 2), PARAM (blob of the wrong rank,
 * job, geometry, precision, layout or version), COMM (IPC or stream memory
 * operations unavailable), CUDA.
 */
vti_status vti_ipc_export(vti_t h, void *out);
vti_status vti_ipc_connect(vti_t h, const void *lo, const void *hi);

/* 0: none (single slab), 1: NCCL, 2: fused peer stores (local group or CUDA IPC). */
int32_t vti_halo_transport(vti_t h);

/* Diagnostics of the peer transport (tests): read (get8) and/or overwrite (set8) this handle's
 * eight flag words {DATA_LO, DATA_HI, ACK_LO, ACK_HI} of p's halo and the same four of the
 * adjoint's s1 rows -- the words its neighbours write --; copy R_xy halo rows of p (side 0: the
 * rows below the slab, side 1: above; level 0: u^n, 1: the stored level) to host memory
 * [nz][R_xy][nx]; vti_debug_rows copies R_xy rows of the adjoint's s1 scratch buffer what >> 1
 * (what & 1 = 0: the slab's first rows, 1: its last rows) or, what = 4 / 5, the receive buffer
 * filled by rank-1 / rank+1, to [nz][R_xy][nx]. All synchronise. Errors: PARAM, STATE, CUDA. */
vti_status vti_debug_flags(vti_t h, uint32_t *get8, const uint32_t *set8);
vti_status vti_debug_halo(vti_t h, int32_t level, int32_t side, void *out);
vti_status vti_debug_rows(vti_t h, int32_t what, void *out);

/* Block until all work on the handle's stream(s) is done. */
vti_status vti_sync(vti_t h);

/* Current time index n (number of steps taken since time index 0). */
int64_t vti_time_index(vti_t h);

/* The cudaStream_t the step kernels run on. */
void *vti_stream(vti_t h);

/* Layout / launch facts of the handle. */
vti_status vti_query(vti_t h, vti_info *info);

/* Tuning knobs (0 = library default): planes per work item, CTAs per SM. */
vti_status vti_set_tuning(vti_t h, int32_t zchunk, int32_t ctas_per_sm);

/* Select a compiled step-kernel variant: tile height (32, 30, 16, 15, 14, 10
 * or 8 rows, per precision and radius pair), dedicated TMA producer warp (1) or
 * in-line producer (0), rows per thread (1 or 2), consecutive x points per
 * thread (4, or 2: float2 / double2); -1 = any. The arithmetic (and so every result bit) is identical across variants.
 * Errors: UNSUPPORTED if no such variant is compiled for (precision, r_xy, r_z). */
vti_status vti_set_variant(vti_t h, int32_t tile_y, int32_t producer_warp, int32_t rows_per_thread,
                           int32_t points_per_thread);

typedef struct {
    int32_t tile_y, producer_warp;  /* chosen variant */
    int32_t rows_per_thread;
    int32_t points_per_thread;
    int32_t zchunk;                 /* chosen planes per work item */
    float ms_per_step;              /* its measured device time per step */
    int32_t candidates;             /* (variant, z-chunk) pairs timed */
} vti_tune_result;

/* SURVEY.md 8(f) N2 autotuner (the paper tuned its CPU blocking the same way,
 * PAPER.md l.242-243): time every compiled variant x z-chunk candidate for
 * probe_steps steps on this handle's own grid and keep the fastest. Needs the
 * model set and the initial zero state (before any vti_step / vti_set_fields):
 * probes inject no source, so the state stays zero and the time index is reset
 * to 0. out may be NULL. Errors: STATE, PARAM, CUDA. */
vti_status vti_autotune(vti_t h, int32_t probe_steps, vti_tune_result *out);

/* Last error message of the handle (or of the last failed vti_create when h is NULL). */
const char *vti_last_error(vti_t h);

/* Free the handle and its device memory (NULL is a no-op). */
vti_status vti_destroy(vti_t h);

#ifdef __cplusplus
}
#endif

#endif /* VTI_H */
