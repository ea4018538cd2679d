// vti_runtime.cu -- host runtime behind include/vti.h (B200 / sm_100a).
//
// Owns the device arrays (all seven share one geometry: nz planes x
// (ny_local + 2R) rows x nx_pad floats, internal layout [z][y][x] by default,
// R_xy halo rows on both y sides of which only p's are ever non-zero), builds
// the TMA tensor maps, the per-plane w^z + gz table and the 1-D Cerjan
// profiles, evaluates the Ricker sample per step on the host, and launches the
// step kernel(s): one launch per step on a single slab, or with nranks > 1 an
// edge launch (whose PEER kernel stores the boundary rows into the neighbours'
// halos) and an interior launch, with the transport of vti_transport.cu between
// them. Scheduling lives in vti_schedule.cu (see vti_internal.h).
#include "vti_internal.h"

// ============================================================ driver entry point
typedef CUresult (*PFN_encodeTiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                    const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode()
{
    static PFN_encodeTiled fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_encodeTiled>(p);
    });
    return fn;
}


// ============================================================ kernel table
// Compiled variants live in csrc/variants/*.cu (see vti_variants.h); the first
// match is the default for (precision, radius pair). -1 = any (env VTI_TY,
// VTI_WP, VTI_RPT, VTI_PX or vti_set_variant select the others).
static const KernelEntry *find_kernel(int esize, int r, int rz, int ty, int wp, int rpt = -1, int px = -1)
{
    static const VariantTable tables[] = {vti_variants_f32_r4(),  vti_variants_f32_r8(),  vti_variants_f32_r6(),
                                          vti_variants_f32_r12(), vti_variants_f64_r48(), vti_variants_f64_r6(),
                                          vti_variants_f64_r12()};
    // VTI_STAGES=n: only variants with an n-deep TMA ring (a measurement switch)
    static const int want_stages = getenv("VTI_STAGES") ? atoi(getenv("VTI_STAGES")) : -1;
    for (const VariantTable &t : tables)
        for (int i = 0; i < t.n; ++i) {
            const KernelEntry &e = t.e[i];
            if (e.esize == esize && e.r == r && e.rz == rz && (ty < 0 || e.ty == ty) && (wp < 0 || e.wp == wp) &&
                (rpt < 0 || e.rpt == rpt) && (px < 0 || e.px == px) && (want_stages < 0 || e.stages == want_stages))
                return &e;
        }
    return nullptr;
}

// The IO-capable variant (N4 point sets) of a radius pair: the default entry of its table.
static const KernelEntry *find_io_kernel(int esize, int r, int rz)
{
    for (int ty : {32, 30, 16, 15, 14, 12, 10, 8})
        for (int wp : {1, 0})
            for (int rpt : {1, 2})
                for (int px : {4, 2}) {
                    const KernelEntry *e = find_kernel(esize, r, rz, ty, wp, rpt, px);
                    if (e && e->fn_io) return e;
                }
    return nullptr;
}

static const SmallEntry *find_small(int esize, int r, int rz, int ty)
{
    static const SmallTable t = vti_small_kernels();
    for (int i = 0; i < t.n; ++i)
        if (t.e[i].esize == esize && t.e[i].r == r && t.e[i].rz == rz && t.e[i].ty == ty) return &t.e[i];
    return nullptr;
}

static std::vector<const KernelEntry *> all_kernels(int esize, int r, int rz)
{
    std::vector<const KernelEntry *> v;
    const KernelEntry *e;
    for (int ty : {32, 30, 16, 15, 14, 12, 10, 8})
        for (int wp : {1, 0})
            for (int rpt : {1, 2})
                for (int px : {4, 2})
                    if ((e = find_kernel(esize, r, rz, ty, wp, rpt, px)) != nullptr) v.push_back(e);
    return v;
}

// ============================================================ aux kernels
// Internal element (x, y, k) of an interior view lives at base[y * ys + k * zs + x].

// user [nk][nyl][nx] (or zero when src == NULL) -> internal planes k0..k0+nk
template <typename T>
__global__ void k_user_to_internal(const T *__restrict__ src, T *__restrict__ dst, int nk, int nyl, int nx,
                                   long long ys, long long zs, int k0)
{
    const int64_t n = (int64_t)nk * nyl * nx;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const int x = (int)(t % nx);
        const int64_t r = t / nx;
        const int y = (int)(r % nyl);
        const int k = (int)(r / nyl);
        dst[y * ys + (k0 + k) * zs + x] = src ? src[t] : T(0);
    }
}

template <typename T>
__global__ void k_internal_to_user(const T *__restrict__ src, T *__restrict__ dst, int nk, int nyl, int nx,
                                   long long ys, long long zs, int k0)
{
    const int64_t n = (int64_t)nk * nyl * nx;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const int x = (int)(t % nx);
        const int64_t r = t / nx;
        const int y = (int)(r % nyl);
        const int k = (int)(r / nyl);
        dst[t] = src[y * ys + (k0 + k) * zs + x];
    }
}

// counters: [0] vz2 <= 0 or non-finite, [1] vx2/vn2 non-finite, [2] vn2 > vx2, over planes k0..k0+nk
template <typename T>
__global__ void k_check_model(const T *__restrict__ vx2, const T *__restrict__ vn2, const T *__restrict__ vz2,
                              int nyl, int nx, long long ys, long long zs, int k0, int nk,
                              unsigned long long *counters)
{
    unsigned long long bad = 0, nonfin = 0, aniso = 0;
    const int64_t n = (int64_t)nyl * nk * nx;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const int x = (int)(t % nx);
        const int64_t r = t / nx;
        const int y = (int)(r % nyl);
        const int k = (int)(r / nyl);
        const int64_t a = y * ys + (k0 + k) * zs + x;
        const T vx = vx2[a], vn = vn2[a], vz = vz2[a];
        bad += !(vz > T(0)) || !isfinite(vz);
        nonfin += !isfinite(vx) || !isfinite(vn);
        aniso += vn > vx;
    }
    if (bad) atomicAdd(&counters[0], bad);
    if (nonfin) atomicAdd(&counters[1], nonfin);
    if (aniso) atomicAdd(&counters[2], aniso);
}

// non-finite test of u^n (p, q) over the interior
template <typename T>
__global__ void k_check_finite(const T *__restrict__ p, const T *__restrict__ q, int nyl, int nz, int nx,
                               long long ys, long long zs, unsigned int *flag)
{
    bool bad = false;
    const int64_t n = (int64_t)nyl * nz * nx;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const int x = (int)(t % nx);
        const int64_t r = t / nx;
        const int y = (int)(r % nyl);
        const int k = (int)(r / nyl);
        const int64_t a = y * ys + k * zs + x;
        bad |= !isfinite(p[a]) || !isfinite(q[a]);
    }
    if (bad) atomicOr(flag, 1u);
}

static std::mutex g_err_mu;
static std::string g_create_err;

vti_status fail(vti_s *h, vti_status s, const char *fmt, ...)
{
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (h) {
        h->err = buf;
    } else {
        std::lock_guard<std::mutex> g(g_err_mu);
        g_create_err = buf;
    }
    return s;
}


static double damping(int idx, int n, int W, double alpha)
{
    // Cerjan taper: g = exp(-(alpha (W - d))^2), d = distance to the nearest face.
    int d = idx < n - 1 - idx ? idx : n - 1 - idx;
    if (d >= W) return 1.0;
    double a = alpha * (double)(W - d);
    return exp(-(a * a));
}

static double ricker(double t, double f, double t0)
{
    // s = (1 - 2 pi^2 f^2 t^2) exp(-pi^2 f^2 t^2), evaluated as x = pi f tau, a = x^2.
    double x = M_PI * f * (t - t0);
    double a = x * x;
    return (1.0 - 2.0 * a) * exp(-a);
}

static bool is_device_ptr(const void *p)
{
    if (!p) return false;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// 3-D tensor map over (x, y, z) of an array with this handle's strides.
vti_status encode(vti_s *h, CUtensorMap *tm, void *base, int rows, int bx, int by, CUtensorMapL2promotion promo,
                  int bz)
{
    PFN_encodeTiled enc = get_encode();
    if (!enc) return fail(h, VTI_E_CUDA, "cuTensorMapEncodeTiled unavailable from the driver");
    cuuint64_t dims[3] = {(cuuint64_t)h->cfg.nx, (cuuint64_t)rows, (cuuint64_t)h->cfg.nz};
    cuuint64_t strides[2] = {(cuuint64_t)(h->ys * h->es), (cuuint64_t)(h->zs * h->es)};
    cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, (cuuint32_t)bz};
    cuuint32_t estr[3] = {1u, 1u, 1u};
    const CUtensorMapDataType dt = h->es == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    CUresult r = enc(tm, dt, 3, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, promo,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);   // NONE = zero fill: the paper's zero exterior
    if (r != CUDA_SUCCESS) return fail(h, VTI_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return VTI_OK;
}

// Device pointers handed in or out by the caller may have been produced or be
// consumed on another stream: order the library's stream after all prior work.
static vti_status order_after_caller(vti_s *h)
{
    CU(h, cudaDeviceSynchronize());
    return VTI_OK;
}


// Typed launch helpers for the auxiliary kernels.
template <typename T>
static void launch_u2i(vti_s *h, const void *src, void *dst, int nk, int k0)
{
    k_user_to_internal<T><<<launch_grid(h), 256, 0, h->stream>>>((const T *)src, (T *)dst, nk, h->nyl, h->cfg.nx,
                                                                   h->ys, h->zs, k0);
}
template <typename T>
static void launch_i2u(vti_s *h, const void *src, void *dst, int nk, int k0)
{
    k_internal_to_user<T><<<launch_grid(h), 256, 0, h->stream>>>((const T *)src, (T *)dst, nk, h->nyl, h->cfg.nx,
                                                                   h->ys, h->zs, k0);
}
static void u2i(vti_s *h, const void *src, void *dst, int nk, int k0)
{
    if (h->es == 8) launch_u2i<double>(h, src, dst, nk, k0);
    else launch_u2i<float>(h, src, dst, nk, k0);
}
static void i2u(vti_s *h, const void *src, void *dst, int nk, int k0)
{
    if (h->es == 8) launch_i2u<double>(h, src, dst, nk, k0);
    else launch_i2u<float>(h, src, dst, nk, k0);
}
// ============================================================ C ABI
extern "C" {

int32_t vti_abi_version(void) { return VTI_ABI_VERSION; }

const char *vti_status_string(vti_status s)
{
    switch (s) {
    case VTI_OK: return "ok";
    case VTI_E_PARAM: return "bad parameter";
    case VTI_E_GEOMETRY: return "bad geometry";
    case VTI_E_MODEL: return "bad model";
    case VTI_E_ANISO: return "anisotropy condition violated";
    case VTI_E_INSTABILITY: return "non-finite wavefield (instability)";
    case VTI_E_INDEX: return "index out of range";
    case VTI_E_CUDA: return "CUDA error";
    case VTI_E_COMM: return "communication error";
    case VTI_E_STATE: return "invalid state";
    case VTI_E_UNSUPPORTED: return "unsupported radius pair";
    }
    return "unknown status";
}

vti_status vti_destroy(vti_t h)
{
    if (!h) return VTI_OK;
    if (h->device_bytes || h->stream) cudaSetDevice(h->cfg.device);
    if (h->stream) cudaStreamSynchronize(h->stream);
    if (h->comm) cudaStreamSynchronize(h->comm);
    if (h->comm_nccl && nccl().ok) nccl().CommDestroy(h->comm_nccl);
    for (void *p : h->ipc_opened)   // the neighbours' mappings first
        if (p) cudaIpcCloseMemHandle(p);
    for (int b = 0; b < 2; ++b) {
        cudaFree(h->pbuf[b]);
        cudaFree(h->qbuf[b]);
        cudaFree(h->sbuf[b]);
        cudaFree(h->rbuf[b]);
    }
    for (void *p : {h->vx2, h->vn2, h->vz2, h->zrow, h->gx, h->gy, h->staging}) cudaFree(p);
    cudaFree(h->counters);
    cudaFree(h->flag);
    cudaFree(h->sync_ctr);
    cudaFree(h->edge_ctr);
    cudaFree(h->flags);
    for (DevPointSet *ps : {&h->rec_set, &h->inj_set}) {
        cudaFree(ps->off);
        cudaFree(ps->ent);
    }
    cudaFree(h->traces);
    cudaFree(h->inj_tr);
    cudaFree(h->dyn);
    cudaFree(h->done);
    cudaFree(h->s_multi);
    cudaFree(h->adj_s[0]);
    cudaFree(h->adj_s[1]);
    cudaFree(h->adj_wt);
    for (int z = 0; z < 2; ++z)
        for (int b = 0; b < 2; ++b)
            if (h->gexec[z][b]) cudaGraphExecDestroy(h->gexec[z][b]);
    cudaFree(h->s_graph);
    for (cudaEvent_t e : {h->ev_edge, h->ev_comm, h->ev_t0, h->ev_t1})
        if (e) cudaEventDestroy(e);
    if (h->comm) cudaStreamDestroy(h->comm);
    if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
    delete h;
    return VTI_OK;
}

static vti_status alloc(vti_s *h, void **p, size_t bytes)
{
    cudaError_t e = cudaMalloc(p, bytes);
    if (e != cudaSuccess) return fail(h, VTI_E_CUDA, "cudaMalloc(%zu bytes): %s", bytes, cudaGetErrorString(e));
    e = cudaMemsetAsync(*p, 0, bytes, h->stream);
    if (e != cudaSuccess) return fail(h, VTI_E_CUDA, "cudaMemset: %s", cudaGetErrorString(e));
    h->device_bytes += (int64_t)bytes;
    return VTI_OK;
}

}  // extern "C"

// Make K the step kernel of the handle: tile height, shared memory, occupancy,
// default schedule and the TMA tensor maps (whose boxes depend on TY).
static void invalidate_graphs(vti_s *h)
{
    for (int z = 0; z < 2; ++z)
        for (int b = 0; b < 2; ++b)
            if (h->gexec[z][b]) {
                cudaGraphExecDestroy(h->gexec[z][b]);
                h->gexec[z][b] = nullptr;
            }
}

static vti_status select_variant(vti_s *h, const KernelEntry *K)
{
    invalidate_graphs(h);
    h->K = K;
    h->TY = K->ty;
    h->nty = (h->nyl + h->TY - 1) / h->TY;
    h->smem_bytes = K->stages * K->stage_bytes + 2 * K->stages * 8;
    for (const void *fn : {K->fn, K->fn_peer, K->fn_io, K->fn_peer_io})
        if (fn) CU(h, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, h->smem_bytes));
    CU(h, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&h->ctas_per_sm, K->fn, K->threads, h->smem_bytes));
    if (h->ctas_per_sm < 1) return fail(h, VTI_E_CUDA, "step kernel cannot be resident (smem %d B)", h->smem_bytes);
    if (h->tune_ctas > 0) h->ctas_per_sm = std::min(h->ctas_per_sm, h->tune_ctas);
    choose_schedule(h);

    // L2 promotion of the halo'd p box (its x apron is not 256-B aligned): env VTI_P_PROMO=none|64|128|256
    CUtensorMapL2promotion ppromo = CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
    if (const char *e = getenv("VTI_P_PROMO")) {
        if (!strcmp(e, "none")) ppromo = CU_TENSOR_MAP_L2_PROMOTION_NONE;
        else if (!strcmp(e, "64")) ppromo = CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
        else if (!strcmp(e, "256")) ppromo = CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
    }
    const int RA = (h->R + 3) / 4 * 4;   // 16-byte aligned x apron (see Cfg::RA)
    const int PW = TX + 2 * RA, PH = h->TY + 2 * h->R;
    vti_status s;
    for (int b = 0; b < 2; ++b) {
        if ((s = encode(h, &h->tm_ph[b], h->pbuf[b], h->rows, PW, PH, ppromo)) != VTI_OK) return s;
        if ((s = encode(h, &h->tm_pi[b], h->p_int(b), h->nyl, TX, h->TY)) != VTI_OK) return s;
        if ((s = encode(h, &h->tm_q[b], h->q_int(b), h->nyl, TX, h->TY)) != VTI_OK) return s;
    }
    if ((s = encode(h, &h->tm_vx, h->in(h->vx2), h->nyl, TX, h->TY)) != VTI_OK) return s;
    if ((s = encode(h, &h->tm_vn, h->in(h->vn2), h->nyl, TX, h->TY)) != VTI_OK) return s;
    if ((s = encode(h, &h->tm_vz, h->in(h->vz2), h->nyl, TX, h->TY)) != VTI_OK) return s;

    // small-grid kernel (vti_small.cuh): single slab, fp32, plans of 1-plane items, default variant
    h->small = nullptr;
    static const bool small_on = !getenv("VTI_SMALL") || atoi(getenv("VTI_SMALL")) != 0;
    const SmallEntry *se = find_small(h->es, h->R, h->RZ, h->TY);
    const double pts = (double)h->cfg.nx * h->nyl * h->cfg.nz;
    if (small_on && se && !h->explicit_variant && h->cfg.nranks == 1 && h->layout_zyx &&
        (h->zchunk == 1 || pts <= 512.0 * 1024)) {
        const int NQ = 2 * h->RZ + 1;
        for (int b = 0; b < 2; ++b)
            if ((s = encode(h, &h->tm_qcol[b], h->q_int(b), h->nyl, TX, h->TY, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            NQ)) != VTI_OK)
                return s;
        for (const void *fn : {se->fn, se->fn_io, se->fn_multi, se->fn_multi_io})
            CU(h, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, se->smem));
        for (const void *fn : {se->fn_direct, se->fn_direct_io})
            CU(h, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, se->smem_direct));
        h->small = se;
        h->zchunk = 1;   // the small kernel's items are (tile, plane)
        h->nzc = h->cfg.nz;
        h->grid = h->ntx * h->nty * h->nzc;
        // multi-step form: every item's CTA must be co-resident (cooperative launch)
        int per_sm = 0, per_sm_io = 0;
        CU(h, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, se->fn_multi, se->threads, se->smem));
        CU(h, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_io, se->fn_multi_io, se->threads, se->smem));
        h->multi_slots = std::min(per_sm, per_sm_io) * h->sms;
        if (h->done_items != h->grid) {   // fresh epoch counters for this item count
            cudaFree(h->done);
            h->done = nullptr;
            CU(h, cudaMalloc((void **)&h->done, (size_t)h->grid * sizeof(unsigned int)));
            CU(h, cudaMemset(h->done, 0, (size_t)h->grid * sizeof(unsigned int)));
            h->done_items = h->grid;
            h->multi_epoch = 0;
        }
    }
    return VTI_OK;
}

// Upload a host table converting double -> T (one rounding for fp32).
static vti_status upload_table(vti_s *h, void **dst, const std::vector<double> &v)
{
    vti_status s = alloc(h, dst, v.size() * h->es);
    if (s != VTI_OK) return s;
    if (h->es == 8) {
        CU(h, cudaMemcpy(*dst, v.data(), v.size() * 8, cudaMemcpyHostToDevice));
    } else {
        std::vector<float> f(v.size());
        for (size_t i = 0; i < v.size(); ++i) f[i] = (float)v[i];
        CU(h, cudaMemcpy(*dst, f.data(), f.size() * 4, cudaMemcpyHostToDevice));
    }
    return VTI_OK;
}

// w_xy / w_z as double (exact widening of float weights for the fp32 entry point).
static vti_status create_impl(vti_s *h, const vti_config *cfg, const double *w_xy, const double *w_z)
{
    vti_status st = check_cfg(cfg);
    if (st != VTI_OK) return fail(h, st, "invalid configuration (%s)", vti_status_string(st));
    if (!w_xy || !w_z) return fail(h, VTI_E_PARAM, "NULL weights");
    h->cfg = *cfg;
    h->es = precision_bits(cfg) / 8;
    h->R = cfg->r_xy;
    h->RZ = cfg->r_z;
    int want_ty = -1, want_wp = -1, want_rpt = -1, want_px = -1;
    if (const char *e = getenv("VTI_TY")) want_ty = atoi(e);
    if (const char *e = getenv("VTI_WP")) want_wp = atoi(e);
    if (const char *e = getenv("VTI_RPT")) want_rpt = atoi(e);
    if (const char *e = getenv("VTI_PX")) want_px = atoi(e);
    h->explicit_variant = want_ty >= 0 || want_wp >= 0 || want_rpt >= 0 || want_px >= 0;
    h->K = find_kernel(h->es, h->R, h->RZ, want_ty, want_wp, want_rpt, want_px);
    if (!h->K) h->K = find_kernel(h->es, h->R, h->RZ, -1, -1);
    if (!h->K)
        return fail(h, VTI_E_UNSUPPORTED, "(r_xy, r_z) = (%d, %d) not compiled for fp%d", h->R, h->RZ, 8 * h->es);
    vti_slab(cfg, &h->y0, &h->nyl);
    // small grids are launch/latency-bound: twice the tiles with the 16-row variant of the same
    // mapping (C1 64^3: 54.7 -> 59.3 Gpoints/s); an explicit env choice wins
    if (want_ty < 0 && want_wp < 0 && want_rpt < 0 && want_px < 0 &&
        (double)cfg->nx * h->nyl * cfg->nz <= 4.0 * 1024 * 1024)
        if (const KernelEntry *k16 = find_kernel(h->es, h->R, h->RZ, 16, -1, -1, h->K->px)) h->K = k16;
    h->nxp = (cfg->nx + 31) / 32 * 32;
    h->rows = h->nyl + 2 * h->R;
    const char *lay = getenv("VTI_LAYOUT");
    h->layout_zyx = !(lay && strcmp(lay, "yzx") == 0);
    if (h->layout_zyx) {   // [z][y][x]: a tile plane is one contiguous run of rows
        h->ys = h->nxp;
        h->zs = (long long)h->rows * h->nxp;
    } else {               // [y][z][x]
        h->ys = (long long)cfg->nz * h->nxp;
        h->zs = h->nxp;
    }
    h->ntx = (cfg->nx + TX - 1) / TX;
    for (int l = 0; l <= h->R; ++l) {
        if (!std::isfinite(w_xy[l])) return fail(h, VTI_E_PARAM, "non-finite w_xy[%d]", l);
        h->cxy[l] = w_xy[l] / (cfg->h * cfg->h);   // reading c3; rounded once to T at launch
    }

    CU(h, cudaSetDevice(cfg->device));
    if (cfg->stream) {
        h->stream = (cudaStream_t)cfg->stream;
    } else {
        CU(h, cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
        h->own_stream = true;
    }
    int prio_lo, prio_hi;
    CU(h, cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    CU(h, cudaStreamCreateWithPriority(&h->comm, cudaStreamNonBlocking, prio_hi));
    CU(h, cudaEventCreateWithFlags(&h->ev_edge, cudaEventDisableTiming));
    CU(h, cudaEventCreateWithFlags(&h->ev_comm, cudaEventDisableTiming));
    CU(h, cudaEventCreate(&h->ev_t0));
    CU(h, cudaEventCreate(&h->ev_t1));
    CU(h, cudaDeviceGetAttribute(&h->sms, cudaDevAttrMultiProcessorCount, cfg->device));

    const size_t bytes = h->total_elems() * h->es;
    vti_status s;
    for (int b = 0; b < 2; ++b) {
        if ((s = alloc(h, &h->pbuf[b], bytes)) != VTI_OK) return s;
        if ((s = alloc(h, &h->qbuf[b], bytes)) != VTI_OK) return s;
    }
    if ((s = alloc(h, &h->vx2, bytes)) != VTI_OK) return s;
    if ((s = alloc(h, &h->vn2, bytes)) != VTI_OK) return s;
    if ((s = alloc(h, &h->vz2, bytes)) != VTI_OK) return s;
    if ((s = alloc(h, (void **)&h->counters, 4 * sizeof(unsigned long long))) != VTI_OK) return s;
    if ((s = alloc(h, (void **)&h->flag, sizeof(unsigned int))) != VTI_OK) return s;
    if ((s = alloc(h, (void **)&h->sync_ctr, sizeof(unsigned long long))) != VTI_OK) return s;
    if ((s = alloc(h, (void **)&h->edge_ctr, sizeof(unsigned long long))) != VTI_OK) return s;
    if (const char *e = getenv("VTI_FUSED_STEP")) h->fused_env = atoi(e) != 0;
    if (const char *e = getenv("VTI_ALIGN")) h->align_rounds = atoi(e) != 0;
    if (const char *e = getenv("VTI_GRAPH")) h->graph_enabled = atoi(e) != 0;
    if (const char *e = getenv("VTI_MULTI")) h->multi_enabled = atoi(e) != 0;
    if (cfg->nranks > 1) {
        const size_t hb = (size_t)cfg->nz * h->R * cfg->nx * h->es;
        for (int b = 0; b < 2; ++b) {
            if ((s = alloc(h, &h->sbuf[b], hb)) != VTI_OK) return s;
            if ((s = alloc(h, &h->rbuf[b], hb)) != VTI_OK) return s;
        }
        if ((s = alloc(h, (void **)&h->flags, 8 * sizeof(unsigned int))) != VTI_OK) return s;
        int flush = 0;
        if (cudaDeviceGetAttribute(&flush, cudaDevAttrCanFlushRemoteWrites, cfg->device) == cudaSuccess)
            h->flush_remote = flush != 0;
        cudaGetLastError();
    }

    // per-plane z rows: w^z[k][0..2Rz], gz[k], zero pad; 1-D Cerjan profiles (double -> T once)
    const int NQ = 2 * h->RZ + 1, ZR = h->K->zrow;
    std::vector<double> zr((size_t)cfg->nz * ZR, 0.0);
    for (int k = 0; k < cfg->nz; ++k) {
        for (int m = 0; m < NQ; ++m) {
            const double v = w_z[(size_t)k * NQ + m];
            if (!std::isfinite(v)) return fail(h, VTI_E_PARAM, "non-finite w_z[%d][%d]", k, m);
            zr[(size_t)k * ZR + m] = v;
        }
        zr[(size_t)k * ZR + NQ] = damping(k, cfg->nz, cfg->damp_width, cfg->damp_alpha);
    }
    std::vector<double> gxv((size_t)h->ntx * TX, 1.0), gyv(h->nyl);
    for (int i = 0; i < cfg->nx; ++i) gxv[i] = damping(i, cfg->nx, cfg->damp_width, cfg->damp_alpha);
    for (int j = 0; j < h->nyl; ++j) gyv[j] = damping(h->y0 + j, cfg->ny, cfg->damp_width, cfg->damp_alpha);
    CU(h, cudaStreamSynchronize(h->stream));
    if ((s = upload_table(h, &h->zrow, zr)) != VTI_OK) return s;
    if ((s = upload_table(h, &h->gx, gxv)) != VTI_OK) return s;
    if ((s = upload_table(h, &h->gy, gyv)) != VTI_OK) return s;

    if ((s = select_variant(h, h->K)) != VTI_OK) return s;

    if (cfg->nranks > 1) {
        if (cfg->nccl_id) {
            NcclApi &api = nccl();
            if (!api.ok) return fail(h, VTI_E_COMM, "%s", api.err.c_str());
            ncclUniqueId id;
            memcpy(&id, cfg->nccl_id, sizeof id);
            ncclResult_t r = api.CommInitRank(&h->comm_nccl, cfg->nranks, id, cfg->rank);
            if (r != ncclSuccess) return fail(h, VTI_E_COMM, "ncclCommInitRank: %s", api.GetErrorString(r));
        } else {
            h->group_mode = true;
        }
    }
    CU(h, cudaStreamSynchronize(h->stream));
    return VTI_OK;
}

static vti_status create_common(vti_t *out, const vti_config *cfg, const double *w_xy, const double *w_z)
{
    vti_s *h = new vti_s();
    vti_status s = create_impl(h, cfg, w_xy, w_z);
    if (s != VTI_OK) {
        {
            std::lock_guard<std::mutex> g(g_err_mu);
            g_create_err = h->err;
        }
        vti_destroy(h);
        return s;
    }
    *out = h;
    return VTI_OK;
}

static vti_status ensure_staging(vti_s *h, size_t want_bytes)
{
    if (h->staging_bytes >= want_bytes) return VTI_OK;
    cudaFree(h->staging);
    h->staging = nullptr;
    h->staging_bytes = 0;
    CU(h, cudaMalloc(&h->staging, want_bytes));
    h->staging_bytes = want_bytes;
    return VTI_OK;
}

// Planes [k0, k0+nk) of a user-layout array (host, device, or NULL = zero) -> interior view dst.
static vti_status upload_planes(vti_s *h, void *dst, const void *src, int k0, int nk)
{
    const size_t plane = (size_t)h->nyl * h->cfg.nx * h->es;   // bytes
    if (!src || is_device_ptr(src)) {
        u2i(h, src, dst, nk, k0);
        CU(h, cudaGetLastError());
        return VTI_OK;
    }
    // host source: bounce through a device staging buffer in chunks of planes
    vti_status s = ensure_staging(h, std::min<size_t>((size_t)nk * plane, std::max<size_t>(plane, (size_t)256 << 20)));
    if (s != VTI_OK) return s;
    const int chunk = (int)std::max<size_t>(1, h->staging_bytes / plane);
    for (int k = 0; k < nk; k += chunk) {
        const int m = std::min(chunk, nk - k);
        CU(h, cudaMemcpyAsync(h->staging, (const char *)src + (size_t)k * plane, (size_t)m * plane,
                              cudaMemcpyHostToDevice, h->stream));
        u2i(h, h->staging, dst, m, k0 + k);
        CU(h, cudaGetLastError());
    }
    CU(h, cudaStreamSynchronize(h->stream));   // staging is reused; host buffer may be freed after return
    return VTI_OK;
}

static vti_status download_planes(vti_s *h, void *dst, const void *src, int k0, int nk)
{
    const size_t plane = (size_t)h->nyl * h->cfg.nx * h->es;
    if (is_device_ptr(dst)) {
        i2u(h, src, dst, nk, k0);
        CU(h, cudaGetLastError());
        CU(h, cudaStreamSynchronize(h->stream));
        return VTI_OK;
    }
    vti_status s = ensure_staging(h, std::min<size_t>((size_t)nk * plane, std::max<size_t>(plane, (size_t)256 << 20)));
    if (s != VTI_OK) return s;
    const int chunk = (int)std::max<size_t>(1, h->staging_bytes / plane);
    for (int k = 0; k < nk; k += chunk) {
        const int m = std::min(chunk, nk - k);
        i2u(h, src, h->staging, m, k0 + k);
        CU(h, cudaGetLastError());
        CU(h, cudaMemcpyAsync((char *)dst + (size_t)k * plane, h->staging, (size_t)m * plane, cudaMemcpyDeviceToHost,
                              h->stream));
    }
    CU(h, cudaStreamSynchronize(h->stream));
    return VTI_OK;
}

static bool any_device(std::initializer_list<const void *> ps)
{
    for (const void *p : ps)
        if (is_device_ptr(p)) return true;
    return false;
}

static vti_status check_precision(vti_s *h, int es, const char *fn)
{
    if (h->es != es)
        return fail(h, VTI_E_PARAM, "%s: handle is fp%d, call is fp%d (use the %s entry point)", fn, 8 * h->es, 8 * es,
                    h->es == 8 ? "_f64" : "fp32");
    return VTI_OK;
}

static vti_status set_model_planes(vti_s *h, int es, int32_t k0, int32_t nk, const void *vx2, const void *vn2,
                                   const void *vz2)
{
    if (!h) return VTI_E_PARAM;
    vti_status s = check_precision(h, es, "vti_set_model");
    if (s != VTI_OK) return s;
    if (!vx2 || !vn2 || !vz2) return fail(h, VTI_E_PARAM, "NULL model array");
    if (k0 < 0 || nk < 0 || k0 + nk > h->cfg.nz)
        return fail(h, VTI_E_INDEX, "planes [%d,%d) outside [0,%d)", k0, k0 + nk, h->cfg.nz);
    CU(h, cudaSetDevice(h->cfg.device));
    if (any_device({vx2, vn2, vz2}) && (s = order_after_caller(h)) != VTI_OK) return s;
    if ((s = upload_planes(h, h->in(h->vx2), vx2, k0, nk)) != VTI_OK) return s;
    if ((s = upload_planes(h, h->in(h->vn2), vn2, k0, nk)) != VTI_OK) return s;
    if ((s = upload_planes(h, h->in(h->vz2), vz2, k0, nk)) != VTI_OK) return s;
    // validate on the device: vz2 > 0 and finite, vx2/vn2 finite, count vn2 > vx2 (reading c5)
    CU(h, cudaMemsetAsync(h->counters, 0, 4 * sizeof(unsigned long long), h->stream));
    if (h->es == 8)
        k_check_model<double><<<launch_grid(h), 256, 0, h->stream>>>(
            (const double *)h->in(h->vx2), (const double *)h->in(h->vn2), (const double *)h->in(h->vz2), h->nyl,
            h->cfg.nx, h->ys, h->zs, k0, nk, h->counters);
    else
        k_check_model<float><<<launch_grid(h), 256, 0, h->stream>>>(
            (const float *)h->in(h->vx2), (const float *)h->in(h->vn2), (const float *)h->in(h->vz2), h->nyl,
            h->cfg.nx, h->ys, h->zs, k0, nk, h->counters);
    CU(h, cudaGetLastError());
    unsigned long long cnt[3];
    CU(h, cudaMemcpyAsync(cnt, h->counters, sizeof cnt, cudaMemcpyDeviceToHost, h->stream));
    CU(h, cudaStreamSynchronize(h->stream));
    if (cnt[0]) return fail(h, VTI_E_MODEL, "%llu points with vz2 <= 0 or non-finite", cnt[0]);
    if (cnt[1]) return fail(h, VTI_E_MODEL, "%llu points with non-finite vx2/vn2", cnt[1]);
    h->aniso_warn += (int64_t)cnt[2];
    // the model counts as set once every plane has been uploaded at least once (planes never
    // uploaded still hold the zero fill of alloc(), i.e. vz2 = 0, which validation rejects)
    if ((int)h->model_planes.size() != h->cfg.nz) h->model_planes.assign(h->cfg.nz, 0);
    std::fill(h->model_planes.begin() + k0, h->model_planes.begin() + k0 + nk, 1);
    h->model_set = std::all_of(h->model_planes.begin(), h->model_planes.end(), [](char c) { return c != 0; });
    return VTI_OK;
}

static vti_status set_fields_planes(vti_s *h, int es, int32_t k0, int32_t nk, const void *p, const void *q,
                                    const void *pm, const void *qm)
{
    if (!h) return VTI_E_PARAM;
    vti_status s = check_precision(h, es, "vti_set_fields");
    if (s != VTI_OK) return s;
    if (!p || !q) return fail(h, VTI_E_PARAM, "NULL p or q");
    if (k0 < 0 || nk < 0 || k0 + nk > h->cfg.nz)
        return fail(h, VTI_E_INDEX, "planes [%d,%d) outside [0,%d)", k0, k0 + nk, h->cfg.nz);
    CU(h, cudaSetDevice(h->cfg.device));
    CU(h, cudaStreamSynchronize(h->comm));
    if (any_device({p, q, pm, qm}) && (s = order_after_caller(h)) != VTI_OK) return s;
    const int c = h->cur, o = 1 - c;
    if ((s = upload_planes(h, h->p_int(c), p, k0, nk)) != VTI_OK) return s;
    if ((s = upload_planes(h, h->q_int(c), q, k0, nk)) != VTI_OK) return s;
    if ((s = upload_planes(h, h->p_int(o), pm, k0, nk)) != VTI_OK) return s;
    if ((s = upload_planes(h, h->q_int(o), qm, k0, nk)) != VTI_OK) return s;
    CU(h, cudaStreamSynchronize(h->stream));
    h->halo_dirty = h->cfg.nranks > 1;
    h->fields_touched = true;
    return VTI_OK;
}

static vti_status get_fields_planes(vti_s *h, int es, int32_t k0, int32_t nk, void *p, void *q, int32_t level)
{
    if (!h) return VTI_E_PARAM;
    vti_status s = check_precision(h, es, "vti_get_fields");
    if (s != VTI_OK) return s;
    if (level != 0 && level != 1) return fail(h, VTI_E_PARAM, "level must be 0 (u^n) or 1 (u^{n-1})");
    if (k0 < 0 || nk < 0 || k0 + nk > h->cfg.nz)
        return fail(h, VTI_E_INDEX, "planes [%d,%d) outside [0,%d)", k0, k0 + nk, h->cfg.nz);
    CU(h, cudaSetDevice(h->cfg.device));
    CU(h, cudaStreamSynchronize(h->comm));
    if (any_device({p, q}) && (s = order_after_caller(h)) != VTI_OK) return s;
    const int b = level == 0 ? h->cur : 1 - h->cur;
    if (p && (s = download_planes(h, p, h->p_int(b), k0, nk)) != VTI_OK) return s;
    if (q && (s = download_planes(h, q, h->q_int(b), k0, nk)) != VTI_OK) return s;
    return VTI_OK;
}

// ============================================================ stepping
template <typename T>
static void fill_params(vti_s *h, StepParams<T> &P, int tr0, int ntr0, int tr1, int ntr1, int zchunk)
{
    const int c = h->cur, o = 1 - c;
    P.tm_p = h->tm_ph[c];
    P.tm_q = h->tm_q[c];
    P.tm_pm = h->tm_pi[o];
    P.tm_qm = h->tm_q[o];
    P.tm_vx = h->tm_vx;
    P.tm_vn = h->tm_vn;
    P.tm_vz = h->tm_vz;
    P.p_out = (T *)h->p_int(o);
    P.q_out = (T *)h->q_int(o);
    P.peer_lo = h->peer ? (T *)h->peer_p[0][o] : nullptr;
    P.peer_hi = h->peer ? (T *)h->peer_p[1][o] : nullptr;
    P.peer_zs_lo = h->peer_zs[0];
    P.peer_zs_hi = h->peer_zs[1];
    P.zrow = (const T *)h->zrow;
    P.gx = (const T *)h->gx;
    P.gy = (const T *)h->gy;
    for (int l = 0; l <= MAX_R; ++l) P.cxy[l] = l <= h->R ? (T)h->cxy[l] : T(0);
    P.dt2 = (T)(h->cfg.dt * h->cfg.dt);
    const bool owned = h->has_src && !h->suppress_src && h->src_j >= h->y0 && h->src_j < h->y0 + h->nyl;
    // s(t^n), t^n = n dt, double on the host, rounded once to T (reading c7)
    P.s = owned ? (T)(h->src_amp * ricker((double)h->n * h->cfg.dt, h->src_f, h->src_t0)) : T(0);
    P.s_table = nullptr;   // set by graph capture
    P.s_index = 0;
    P.src_i = h->src_i;
    P.src_j = owned ? h->src_j - h->y0 : -1;
    P.src_k = h->src_k;
    P.src_mask = owned ? h->src_mask : 0;
    P.nx = h->cfg.nx;
    P.nyl = h->nyl;
    P.nz = h->cfg.nz;
    P.ys = h->ys;
    P.zs = h->zs;
    P.ntx = h->ntx;
    P.tr0 = tr0;
    P.ntr0 = ntr0;
    P.tr1 = tr1;
    P.ntr1 = ntr1;
    P.zchunk = zchunk;
    P.nzc = (h->cfg.nz + zchunk - 1) / zchunk;
    P.items = h->ntx * (ntr0 + ntr1) * P.nzc;
    P.tr2 = 0;
    P.ntr2 = 0;
    P.edge_items = 0;
    P.edge_ctr = nullptr;
    P.edge_target = 0;
    for (int i = 0; i < 4; ++i) {
        P.sig[i] = nullptr;
        P.sig_val[i] = 0;
    }
    // N4 point sets (read only by the IO instantiations; none during autotune probes)
    const bool inj = h->inj_set.n > 0 && !h->suppress_src;
    P.inj_off = inj ? h->inj_set.off : nullptr;
    P.inj_ent = inj ? h->inj_set.ent : nullptr;
    P.inj_tr = (const T *)h->inj_tr;
    P.inj_cols = h->inj_cols;
    P.inj_mask = h->inj_mask;
    P.inj_nt = h->inj_nt;
    P.inj_row = (long long)(h->n - h->inj_t_first);   // F(u^n) at time index n
    const bool rec = h->rec_set.n > 0 && h->rec_cap > 0 && !h->suppress_src;
    P.rec_off = rec ? h->rec_set.off : nullptr;
    P.rec_ent = rec ? h->rec_set.ent : nullptr;
    P.rec_tr = (T *)h->traces;
    P.rec_cols = h->nrec;
    P.rec_mask = h->rec_mask;
    P.rec_cap = h->rec_cap;
    P.rec_row = h->rec_steps;
    P.dyn = nullptr;
    P.graph_i = 0;
}

// Fused multi-GPU launch: the interior tile rows after the edge rows, and the flags the
// last edge item raises (see StepParams::edge_items).
struct FusedDesc {
    int tr2, ntr2;
    unsigned int *sig[4];
    unsigned int sig_val[4];
};

template <typename T>
static vti_status launch_rows_t(vti_s *h, int tr0, int ntr0, int tr1, int ntr1, int zchunk, int cap,
                                const FusedDesc *fd = nullptr)
{
    StepParams<T> P;
    fill_params<T>(h, P, tr0, ntr0, tr1, ntr1, zchunk);
    if (fd) {
        P.tr2 = fd->tr2;
        P.ntr2 = fd->ntr2;
        P.edge_items = P.items;                       // edge items first
        P.items += h->ntx * fd->ntr2 * P.nzc;
        P.edge_ctr = h->edge_ctr;
        h->edge_value += (unsigned long long)P.edge_items;
        P.edge_target = h->edge_value;
        for (int i = 0; i < 4; ++i) {
            P.sig[i] = fd->sig[i];
            P.sig_val[i] = fd->sig_val[i];
        }
    }
    if (h->capturing) {   // graph node: the source sample comes from the graph's table
        P.s_table = (const T *)h->s_graph;
        P.s_index = h->capture_index;
        P.dyn = h->dyn;            // N4 trace rows from the replay header
        P.graph_i = h->capture_index;
    }
    const bool io = h->io_active() && !h->suppress_src;
    if (h->small && zchunk == 1 && tr0 == 0 && ntr0 == h->nty && ntr1 == 0) {
        // small-grid kernel: one CTA per (tile, plane) item, every load of the item at once
        SmallParams<T> S;
        S.P = P;
        S.P.sync_ctr = nullptr;
        S.P.sync_base = 0;
        S.tm_qcol = h->tm_qcol[h->cur];
        const int o = 1 - h->cur;
        S.q_cur = (const T *)h->q_int(h->cur);
        S.p_m = (const T *)h->p_int(o);
        S.q_m = (const T *)h->q_int(o);
        S.vx = (const T *)h->in(h->vx2);
        S.vn = (const T *)h->in(h->vn2);
        S.vz = (const T *)h->in(h->vz2);
        // the direct-load form (only the p tile staged by TMA; C1 86.8 -> 92.7 Gpoints/s) unless
        // VTI_SMALL_DIRECT=0 (every operand staged by TMA)
        static const bool direct = !getenv("VTI_SMALL_DIRECT") || atoi(getenv("VTI_SMALL_DIRECT")) != 0;
        cudaLaunchConfig_t sl = {};
        sl.gridDim = dim3(P.items);
        sl.blockDim = dim3(h->small->threads);
        sl.dynamicSmemBytes = direct ? h->small->smem_direct : h->small->smem;
        sl.stream = h->stream;
        cudaLaunchAttribute sa[1];
        static const bool pdl = !getenv("VTI_PDL") || atoi(getenv("VTI_PDL")) != 0;
        if (pdl) {   // overlap this launch with the previous step's tail (see vti_small.cuh)
            sa[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            sa[0].val.programmaticStreamSerializationAllowed = 1;
            sl.attrs = sa;
            sl.numAttrs = 1;
        }
        void *sargs[] = {&S};
        const void *sfn = direct ? (io ? h->small->fn_direct_io : h->small->fn_direct)
                                 : (io ? h->small->fn_io : h->small->fn);
        CU(h, cudaLaunchKernelExC(&sl, sfn, sargs));
        return VTI_OK;
    }
    const int grid = std::min(P.items, cap > 0 ? std::min(cap, slots(h)) : slots(h));
    const int rounds = (P.items + grid - 1) / grid;
    P.sync_ctr = nullptr;
    P.sync_base = 0;
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(grid);
    lc.blockDim = dim3(h->K->threads);
    lc.dynamicSmemBytes = h->smem_bytes;
    lc.stream = h->stream;
    cudaLaunchAttribute attr[1];
    if (rounds > 1 && h->align_rounds) {
        // all CTAs must be co-resident for the in-kernel round barrier: cooperative launch
        P.sync_ctr = h->sync_ctr;
        P.sync_base = h->sync_value;
        h->sync_value += (unsigned long long)grid * (rounds - 1);
        attr[0].id = cudaLaunchAttributeCooperative;
        attr[0].val.cooperative = 1;
        lc.attrs = attr;
        lc.numAttrs = 1;
    }
    void *args[] = {&P};
    // only tile rows within R of the slab edges store into the neighbours (edge launches)
    const bool peer_rows = (P.peer_lo || P.peer_hi) && (tr0 * h->TY < h->R || (tr0 + ntr0) * h->TY > h->nyl - h->R ||
                                                        (ntr1 > 0 && (tr1 + ntr1) * h->TY > h->nyl - h->R));
    const void *fn = peer_rows ? (io ? h->K->fn_peer_io : h->K->fn_peer) : (io ? h->K->fn_io : h->K->fn);
    if (!fn) return fail(h, VTI_E_STATE, "step-kernel variant without the point-set (IO) instantiation");
    CU(h, cudaLaunchKernelExC(&lc, fn, args));
    return VTI_OK;
}

vti_status launch_fused(vti_s *h, unsigned int *const sig[4], const unsigned int sig_val[4])
{
    int e1, e2;
    edge_rows(h, e1, e2);
    FusedDesc fd;
    fd.tr2 = e1;
    fd.ntr2 = e2 - e1;
    for (int i = 0; i < 4; ++i) {
        fd.sig[i] = sig[i];
        fd.sig_val[i] = sig_val[i];
    }
    // one launch over every tile row: the full-launch plan (z-chunk, CTA cap)
    return h->es == 8 ? launch_rows_t<double>(h, 0, e1, e2, h->nty - e2, h->zchunk, h->cap, &fd)
                      : launch_rows_t<float>(h, 0, e1, e2, h->nty - e2, h->zchunk, h->cap, &fd);
}

// Tile rows [tr0, tr0+ntr0) then [tr1, tr1+ntr1) of this slab, z-chunks of zchunk planes.
static vti_status launch_rows(vti_s *h, int tr0, int ntr0, int tr1, int ntr1, int zchunk, int cap)
{
    if (ntr0 + ntr1 <= 0) return VTI_OK;
    return h->es == 8 ? launch_rows_t<double>(h, tr0, ntr0, tr1, ntr1, zchunk, cap)
                      : launch_rows_t<float>(h, tr0, ntr0, tr1, ntr1, zchunk, cap);
}

vti_status launch_edge(vti_s *h)
{
    int e1, e2;
    edge_rows(h, e1, e2);
    return launch_rows(h, 0, e1, e2, h->nty - e2, h->zchunk_edge, h->cap_edge);
}

vti_status launch_interior(vti_s *h)
{
    int e1, e2;
    edge_rows(h, e1, e2);
    return launch_rows(h, e1, e2 - e1, 0, 0, h->zchunk_inner, h->cap_inner);
}

vti_status check_finite(vti_s *h)
{
    CU(h, cudaMemsetAsync(h->flag, 0, sizeof(unsigned int), h->stream));
    if (h->es == 8)
        k_check_finite<double><<<launch_grid(h), 256, 0, h->stream>>>(
            (const double *)h->p_int(h->cur), (const double *)h->q_int(h->cur), h->nyl, h->cfg.nz, h->cfg.nx, h->ys,
            h->zs, h->flag);
    else
        k_check_finite<float><<<launch_grid(h), 256, 0, h->stream>>>(
            (const float *)h->p_int(h->cur), (const float *)h->q_int(h->cur), h->nyl, h->cfg.nz, h->cfg.nx, h->ys,
            h->zs, h->flag);
    CU(h, cudaGetLastError());
    unsigned int f = 0;
    CU(h, cudaMemcpyAsync(&f, h->flag, sizeof f, cudaMemcpyDeviceToHost, h->stream));
    CU(h, cudaStreamSynchronize(h->stream));
    if (f) return fail(h, VTI_E_INSTABILITY, "non-finite wavefield at time index %lld", (long long)h->n);
    return VTI_OK;
}

// Receiver rows written by `steps` steps (the gather itself is fused into the step kernel's
// store epilogue); recording stops silently at the capacity (vti_get_traces reports the count).
void advance_records(vti_s *h, int steps)
{
    if (h->rec_set.n == 0 || h->suppress_src) return;   // not during autotune probes
    h->rec_steps = std::min(h->rec_cap, h->rec_steps + steps);
}

// While a point set is active, the step kernel must be an IO instantiation: the small-grid
// kernel has one for every radius pair; otherwise switch to the pair's default variant (every
// variant computes the same bits, so only the speed can change).
vti_status prepare_io(vti_s *h)
{
    if (!h->io_active() || h->small || h->K->fn_io) return VTI_OK;
    const KernelEntry *K = find_io_kernel(h->es, h->R, h->RZ);
    if (!K) return fail(h, VTI_E_UNSUPPORTED, "no point-set (IO) step kernel for (%d, %d)", h->R, h->RZ);
    return select_variant(h, K);
}

// Build the device CSR of a point set: pts = (x, local row, plane, column).
static vti_status build_point_set(vti_s *h, DevPointSet &ps, std::vector<std::array<int, 4>> pts)
{
    cudaFree(ps.off);
    cudaFree(ps.ent);
    ps = DevPointSet{};
    if (pts.empty()) return VTI_OK;
    std::sort(pts.begin(), pts.end(), [](const std::array<int, 4> &a, const std::array<int, 4> &b) {
        return a[2] != b[2] ? a[2] < b[2] : a[1] != b[1] ? a[1] < b[1] : a[0] != b[0] ? a[0] < b[0] : a[3] < b[3];
    });
    const size_t rows = (size_t)h->cfg.nz * h->nyl;
    std::vector<int> off(rows + 1, 0);
    std::vector<int2> ent(pts.size());
    for (size_t e = 0; e < pts.size(); ++e) {
        off[(size_t)pts[e][2] * h->nyl + pts[e][1] + 1] += 1;
        ent[e] = make_int2(pts[e][0], pts[e][3]);
    }
    for (size_t r = 0; r < rows; ++r) off[r + 1] += off[r];
    CU(h, cudaMalloc((void **)&ps.off, off.size() * sizeof(int)));
    CU(h, cudaMemcpy(ps.off, off.data(), off.size() * sizeof(int), cudaMemcpyHostToDevice));
    CU(h, cudaMalloc((void **)&ps.ent, ent.size() * sizeof(int2)));
    CU(h, cudaMemcpy(ps.ent, ent.data(), ent.size() * sizeof(int2), cudaMemcpyHostToDevice));
    ps.n = (int)pts.size();
    return VTI_OK;
}

extern "C" {

vti_status vti_set_receivers(vti_t h, int32_t n, const int32_t *ijk, int32_t field_mask, int32_t capacity_steps)
{
    if (!h) return VTI_E_PARAM;
    if (n < 0 || capacity_steps < 0 || (n > 0 && !ijk)) return fail(h, VTI_E_PARAM, "bad receiver arguments");
    if (n > 0 && (field_mask < 1 || field_mask > 3)) return fail(h, VTI_E_PARAM, "field_mask must be 1, 2 or 3");
    std::vector<std::array<int, 4>> pts;   // (x, local row, plane, local receiver index)
    std::vector<int32_t> ids;
    for (int r = 0; r < n; ++r) {
        const int i = ijk[3 * r], j = ijk[3 * r + 1], k = ijk[3 * r + 2];
        if (i < 0 || i >= h->cfg.nx || j < 0 || j >= h->cfg.ny || k < 0 || k >= h->cfg.nz)
            return fail(h, VTI_E_INDEX, "receiver %d (%d,%d,%d) outside the grid", r, i, j, k);
        if (j < h->y0 || j >= h->y0 + h->nyl) continue;   // another rank's slab
        pts.push_back({i, j - h->y0, k, (int)ids.size()});
        ids.push_back(r);
    }
    CU(h, cudaSetDevice(h->cfg.device));
    CU(h, cudaStreamSynchronize(h->stream));
    CU(h, cudaStreamSynchronize(h->comm));
    invalidate_graphs(h);   // the point set is baked into graph nodes
    cudaFree(h->traces);
    h->traces = nullptr;
    h->nrec = (int)ids.size();
    h->rec_ids = ids;
    h->rec_mask = field_mask;
    h->rec_cap = capacity_steps;
    h->rec_steps = 0;
    vti_status s = build_point_set(h, h->rec_set, capacity_steps > 0 ? pts : std::vector<std::array<int, 4>>{});
    if (s != VTI_OK) return s;
    if (h->nrec > 0 && capacity_steps > 0) {
        const int nf = (field_mask & 1) + ((field_mask >> 1) & 1);
        CU(h, cudaMalloc(&h->traces, (size_t)capacity_steps * h->nrec * nf * h->es));
        CU(h, cudaMemset(h->traces, 0, (size_t)capacity_steps * h->nrec * nf * h->es));
    }
    return VTI_OK;
}

static vti_status set_injection(vti_s *h, int es, int32_t n, const int32_t *ijk, int32_t field_mask, int32_t nt,
                                int64_t t_first, const void *traces)
{
    if (!h) return VTI_E_PARAM;
    vti_status s = check_precision(h, es, "vti_set_injection");
    if (s != VTI_OK) return s;
    if (n < 0 || nt < 0 || (n > 0 && (!ijk || (nt > 0 && !traces))))
        return fail(h, VTI_E_PARAM, "bad injection arguments");
    if (n > 0 && (field_mask < 1 || field_mask > 3)) return fail(h, VTI_E_PARAM, "field_mask must be 1, 2 or 3");
    std::vector<std::array<int, 4>> pts;   // (x, local row, plane, column = caller's index r)
    std::vector<long long> keys;
    for (int r = 0; r < n; ++r) {
        const int i = ijk[3 * r], j = ijk[3 * r + 1], k = ijk[3 * r + 2];
        if (i < 0 || i >= h->cfg.nx || j < 0 || j >= h->cfg.ny || k < 0 || k >= h->cfg.nz)
            return fail(h, VTI_E_INDEX, "injection point %d (%d,%d,%d) outside the grid", r, i, j, k);
        keys.push_back(((long long)k * h->cfg.ny + j) * h->cfg.nx + i);
        if (j < h->y0 || j >= h->y0 + h->nyl) continue;   // another rank's slab
        pts.push_back({i, j - h->y0, k, r});
    }
    std::sort(keys.begin(), keys.end());
    if (std::adjacent_find(keys.begin(), keys.end()) != keys.end())
        return fail(h, VTI_E_PARAM, "injection points must be distinct");
    CU(h, cudaSetDevice(h->cfg.device));
    if (traces && is_device_ptr(traces) && (s = order_after_caller(h)) != VTI_OK) return s;
    CU(h, cudaStreamSynchronize(h->stream));
    CU(h, cudaStreamSynchronize(h->comm));
    invalidate_graphs(h);
    cudaFree(h->inj_tr);
    h->inj_tr = nullptr;
    h->inj_cols = n;
    h->inj_mask = field_mask;
    h->inj_nt = nt;
    h->inj_t_first = t_first;
    const bool any = !pts.empty() && nt > 0;
    if ((s = build_point_set(h, h->inj_set, any ? pts : std::vector<std::array<int, 4>>{})) != VTI_OK) return s;
    if (any) {
        const size_t bytes = (size_t)nt * n * h->es;
        CU(h, cudaMalloc(&h->inj_tr, bytes));
        CU(h, cudaMemcpy(h->inj_tr, traces, bytes, cudaMemcpyDefault));   // host or device source
    }
    return VTI_OK;
}

vti_status vti_set_injection(vti_t h, int32_t n, const int32_t *ijk, int32_t field_mask, int32_t nt,
                             int64_t t_first, const float *traces)
{
    return set_injection(h, 4, n, ijk, field_mask, nt, t_first, traces);
}

vti_status vti_set_injection_f64(vti_t h, int32_t n, const int32_t *ijk, int32_t field_mask, int32_t nt,
                                 int64_t t_first, const double *traces)
{
    return set_injection(h, 8, n, ijk, field_mask, nt, t_first, traces);
}

vti_status vti_receiver_info(vti_t h, int32_t *n_local, int32_t *steps_recorded, int32_t *ids)
{
    if (!h) return VTI_E_PARAM;
    if (n_local) *n_local = h->nrec;
    if (steps_recorded) *steps_recorded = h->rec_steps;
    if (ids)
        for (int r = 0; r < h->nrec; ++r) ids[r] = h->rec_ids[r];
    return VTI_OK;
}

static vti_status get_traces(vti_s *h, int es, void *out)
{
    if (!h) return VTI_E_PARAM;
    vti_status s = check_precision(h, es, "vti_get_traces");
    if (s != VTI_OK) return s;
    if (!out) return fail(h, VTI_E_PARAM, "NULL output");
    if (h->nrec == 0 || h->rec_steps == 0) return VTI_OK;
    const int nf = (h->rec_mask & 1) + ((h->rec_mask >> 1) & 1);
    CU(h, cudaSetDevice(h->cfg.device));
    CU(h, cudaStreamSynchronize(h->stream));
    CU(h, cudaMemcpy(out, h->traces, (size_t)h->rec_steps * h->nrec * nf * h->es, cudaMemcpyDefault));
    return VTI_OK;
}

vti_status vti_get_traces(vti_t h, float *out) { return get_traces(h, 4, out); }
vti_status vti_get_traces_f64(vti_t h, double *out) { return get_traces(h, 8, out); }

vti_status vti_reverse(vti_t h)
{
    if (!h) return VTI_E_PARAM;
    CU(h, cudaSetDevice(h->cfg.device));
    CU(h, cudaStreamSynchronize(h->stream));
    CU(h, cudaStreamSynchronize(h->comm));
    // the stored levels (u^n, u^{n-dir}) become (u^{n-dir}, u^n): the next step applies Eq. 3
    // at level n - dir and produces level n - 2 dir
    h->cur = 1 - h->cur;
    h->n -= h->dir;
    h->dir = -h->dir;
    h->halo_dirty = h->cfg.nranks > 1;   // re-exchange the new current level's halo rows
    return VTI_OK;
}

int32_t vti_direction(vti_t h) { return h ? h->dir : 0; }

vti_status vti_create(vti_t *out, const vti_config *cfg, const float *w_xy, const float *w_z)
{
    if (!out) return fail(nullptr, VTI_E_PARAM, "NULL output handle");
    *out = nullptr;
    vti_status st = check_cfg(cfg);
    if (st != VTI_OK) return fail(nullptr, st, "invalid configuration (%s)", vti_status_string(st));
    if (!w_xy || !w_z) return fail(nullptr, VTI_E_PARAM, "NULL weights");
    const int NQ = 2 * cfg->r_z + 1;
    std::vector<double> wxy(cfg->r_xy + 1), wz((size_t)cfg->nz * NQ);
    for (size_t i = 0; i < wxy.size(); ++i) wxy[i] = (double)w_xy[i];   // exact widening
    for (size_t i = 0; i < wz.size(); ++i) wz[i] = (double)w_z[i];
    return create_common(out, cfg, wxy.data(), wz.data());
}

vti_status vti_create_f64(vti_t *out, const vti_config *cfg, const double *w_xy, const double *w_z)
{
    if (!out) return fail(nullptr, VTI_E_PARAM, "NULL output handle");
    *out = nullptr;
    vti_status st = check_cfg(cfg);
    if (st != VTI_OK) return fail(nullptr, st, "invalid configuration (%s)", vti_status_string(st));
    if (precision_bits(cfg) != 64) return fail(nullptr, VTI_E_PARAM, "vti_create_f64 needs cfg->precision = 64");
    if (!w_xy || !w_z) return fail(nullptr, VTI_E_PARAM, "NULL weights");
    return create_common(out, cfg, w_xy, w_z);
}

const char *vti_last_error(vti_t h)
{
    if (h) return h->err.c_str();
    std::lock_guard<std::mutex> g(g_err_mu);
    return g_create_err.c_str();
}

vti_status vti_set_model_planes(vti_t h, int32_t k0, int32_t nk, const float *vx2, const float *vn2,
                                const float *vz2)
{
    return set_model_planes(h, 4, k0, nk, vx2, vn2, vz2);
}

vti_status vti_set_model_planes_f64(vti_t h, int32_t k0, int32_t nk, const double *vx2, const double *vn2,
                                    const double *vz2)
{
    return set_model_planes(h, 8, k0, nk, vx2, vn2, vz2);
}

vti_status vti_set_model(vti_t h, const float *vx2, const float *vn2, const float *vz2)
{
    if (!h) return VTI_E_PARAM;
    return set_model_planes(h, 4, 0, h->cfg.nz, vx2, vn2, vz2);
}

vti_status vti_set_model_f64(vti_t h, const double *vx2, const double *vn2, const double *vz2)
{
    if (!h) return VTI_E_PARAM;
    return set_model_planes(h, 8, 0, h->cfg.nz, vx2, vn2, vz2);
}

int64_t vti_model_warnings(vti_t h) { return h ? h->aniso_warn : -1; }

vti_status vti_add_source(vti_t h, int32_t i, int32_t j, int32_t k, double f, double t0, double amp,
                          int32_t field_mask)
{
    if (!h) return VTI_E_PARAM;
    if (field_mask < 1 || field_mask > 3) return fail(h, VTI_E_PARAM, "field_mask must be 1, 2 or 3");
    if (!std::isfinite(f) || !std::isfinite(t0) || !std::isfinite(amp))
        return fail(h, VTI_E_PARAM, "non-finite source parameter");
    if (i < 0 || i >= h->cfg.nx || j < 0 || j >= h->cfg.ny || k < 0 || k >= h->cfg.nz)
        return fail(h, VTI_E_INDEX, "source (%d,%d,%d) outside the %dx%dx%d grid", i, j, k, h->cfg.nx, h->cfg.ny,
                    h->cfg.nz);
    invalidate_graphs(h);   // the source position and mask are baked into graph nodes
    h->has_src = true;
    h->src_i = i;
    h->src_j = j;
    h->src_k = k;
    h->src_f = f;
    h->src_t0 = t0;
    h->src_amp = amp;
    h->src_mask = field_mask;
    return VTI_OK;
}

vti_status vti_set_fields_planes(vti_t h, int32_t k0, int32_t nk, const float *p, const float *q, const float *pm,
                                 const float *qm)
{
    return set_fields_planes(h, 4, k0, nk, p, q, pm, qm);
}

vti_status vti_set_fields_planes_f64(vti_t h, int32_t k0, int32_t nk, const double *p, const double *q,
                                     const double *pm, const double *qm)
{
    return set_fields_planes(h, 8, k0, nk, p, q, pm, qm);
}

vti_status vti_set_fields(vti_t h, const float *p, const float *q, const float *pm, const float *qm,
                          int64_t time_index)
{
    if (!h) return VTI_E_PARAM;
    vti_status s = set_fields_planes(h, 4, 0, h->cfg.nz, p, q, pm, qm);
    if (s == VTI_OK) h->n = time_index;
    return s;
}

vti_status vti_set_fields_f64(vti_t h, const double *p, const double *q, const double *pm, const double *qm,
                              int64_t time_index)
{
    if (!h) return VTI_E_PARAM;
    vti_status s = set_fields_planes(h, 8, 0, h->cfg.nz, p, q, pm, qm);
    if (s == VTI_OK) h->n = time_index;
    return s;
}

// A pointer the device can write directly: device / managed memory, or page-locked host memory
// with a device mapping (UVA).
static bool device_writable(const void *p)
{
    cudaPointerAttributes a;
    if (!p || cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged ||
           (a.type == cudaMemoryTypeHost && a.devicePointer != nullptr);
}

static vti_status snapshot_async(vti_s *h, int es, int32_t k0, int32_t nk, void *p, void *q, int32_t level)
{
    if (!h) return VTI_E_PARAM;
    vti_status s = check_precision(h, es, "vti_snapshot_async");
    if (s != VTI_OK) return s;
    if (level != 0 && level != 1) return fail(h, VTI_E_PARAM, "level must be 0 (u^n) or 1 (u^{n-1})");
    if (k0 < 0 || nk < 0 || k0 + nk > h->cfg.nz)
        return fail(h, VTI_E_INDEX, "planes [%d,%d) outside [0,%d)", k0, k0 + nk, h->cfg.nz);
    CU(h, cudaSetDevice(h->cfg.device));
    if ((p && !device_writable(p)) || (q && !device_writable(q)))
        return fail(h, VTI_E_PARAM, "snapshot buffers must be device memory or mapped page-locked host memory");
    const int b = level == 0 ? h->cur : 1 - h->cur;
    if (p) i2u(h, h->p_int(b), p, nk, k0);
    if (q) i2u(h, h->q_int(b), q, nk, k0);
    CU(h, cudaGetLastError());
    return VTI_OK;
}

vti_status vti_snapshot_async(vti_t h, int32_t k0, int32_t nk, float *p, float *q, int32_t level)
{
    return snapshot_async(h, 4, k0, nk, p, q, level);
}

vti_status vti_snapshot_async_f64(vti_t h, int32_t k0, int32_t nk, double *p, double *q, int32_t level)
{
    return snapshot_async(h, 8, k0, nk, p, q, level);
}

vti_status vti_get_fields_planes(vti_t h, int32_t k0, int32_t nk, float *p, float *q, int32_t level)
{
    return get_fields_planes(h, 4, k0, nk, p, q, level);
}

vti_status vti_get_fields_planes_f64(vti_t h, int32_t k0, int32_t nk, double *p, double *q, int32_t level)
{
    return get_fields_planes(h, 8, k0, nk, p, q, level);
}

vti_status vti_get_fields(vti_t h, float *p, float *q, int32_t level)
{
    if (!h) return VTI_E_PARAM;
    return get_fields_planes(h, 4, 0, h->cfg.nz, p, q, level);
}

vti_status vti_get_fields_f64(vti_t h, double *p, double *q, int32_t level)
{
    if (!h) return VTI_E_PARAM;
    return get_fields_planes(h, 8, 0, h->cfg.nz, p, q, level);
}

// ---- CUDA graphs for launch-bound small grids (single slab, one round per step)
// Two graph sizes (even: a replay returns to its starting parity): 128-step graphs while at
// least 128 steps remain, then 32-step ones; the source table and the N4 header are refilled
// before each replay, a stream-ordered copy that costs a bubble per replay (C1: 32-step
// replays 92.9, 128-step 95.8 Gpoints/s). Env VTI_GRAPH_STEPS (even, 2..256) sets the large size.
static constexpr int GRAPH_STEPS = 32;
static const int GRAPH_STEPS_BIG = [] {
    const int v = getenv("VTI_GRAPH_STEPS") ? atoi(getenv("VTI_GRAPH_STEPS")) : 128;
    return (v >= 2 && v <= 256 && v % 2 == 0) ? v : 128;
}();
static int graph_steps(int z) { return z ? GRAPH_STEPS_BIG : GRAPH_STEPS; }

static bool graph_eligible(const vti_s *h)
{
    if (!h->graph_enabled || h->cfg.nranks > 1 || h->cfg.check_every > 0 || h->suppress_src ||
        getenv("VTI_FORCE_SPLIT"))
        return false;
    const long items = (long)h->ntx * h->nty * h->nzc;
    if (items > (long)h->cap) return false;          // multi-round: cooperative launches
    const double pts = (double)h->cfg.nx * h->nyl * h->cfg.nz;
    return pts <= 64.0 * 1024 * 1024;   // beyond that a step is long enough that launch gaps do not matter
}

// Capture graph_steps(z) steps starting at parity c into h->gexec[z][c].
static vti_status build_graph(vti_s *h, int z, int c)
{
    const int n = graph_steps(z);
    if (!h->s_graph) CU(h, cudaMalloc(&h->s_graph, 256 * 8));
    if (!h->dyn) CU(h, cudaMalloc((void **)&h->dyn, 3 * sizeof(long long)));
    const int keep_cur = h->cur;
    cudaGraph_t g = nullptr;
    CU(h, cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
    h->capturing = true;
    vti_status s = VTI_OK;
    for (int i = 0; i < n && s == VTI_OK; ++i) {
        h->cur = (c + i) & 1;
        h->capture_index = i;
        s = launch_rows(h, 0, h->nty, 0, 0, h->zchunk, h->cap);
    }
    h->capturing = false;
    h->cur = keep_cur;
    cudaError_t e = cudaStreamEndCapture(h->stream, &g);
    if (s != VTI_OK) {
        if (g) cudaGraphDestroy(g);
        return s;
    }
    if (e != cudaSuccess) return fail(h, VTI_E_CUDA, "graph capture: %s", cudaGetErrorString(e));
    e = cudaGraphInstantiate(&h->gexec[z][c], g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return fail(h, VTI_E_CUDA, "graph instantiate: %s", cudaGetErrorString(e));
    return VTI_OK;
}

// Replay graph_steps(z) steps: refill the source table (stream-ordered, from pageable host
// memory so the host buffer is free on return), then launch the graph.
static vti_status replay_graph(vti_s *h, int z)
{
    vti_status s;
    const int n = graph_steps(z);
    if (!h->gexec[z][h->cur] && (s = build_graph(h, z, h->cur)) != VTI_OK) return s;
    const bool owned = h->has_src && h->src_j >= h->y0 && h->src_j < h->y0 + h->nyl;
    h->s_host.assign(n, 0.0);
    for (int i = 0; i < n && owned; ++i)
        h->s_host[i] = h->src_amp * ricker((double)(h->n + (int64_t)i * h->dir) * h->cfg.dt, h->src_f, h->src_t0);
    if (h->es == 8) {
        CU(h, cudaMemcpyAsync(h->s_graph, h->s_host.data(), n * 8, cudaMemcpyHostToDevice, h->stream));
    } else {
        std::vector<float> f(n);
        for (int i = 0; i < n; ++i) f[i] = (float)h->s_host[i];   // rounded once, as P.s
        CU(h, cudaMemcpyAsync(h->s_graph, f.data(), n * sizeof(float), cudaMemcpyHostToDevice, h->stream));
    }
    // N4 trace rows of the replay's first step: injection row n - t_first (then + i * dir),
    // receiver row rec_steps (then + i); the kernels skip rows outside their ranges
    const long long hdr[3] = {(long long)(h->n - h->inj_t_first), (long long)h->rec_steps, (long long)h->dir};
    CU(h, cudaMemcpyAsync(h->dyn, hdr, sizeof hdr, cudaMemcpyHostToDevice, h->stream));
    CU(h, cudaGraphLaunch(h->gexec[z][h->cur], h->stream));
    h->n += (int64_t)n * h->dir;   // parity (cur) is unchanged after an even number of steps
    advance_records(h, n);
    return VTI_OK;
}

}  // extern "C"

// ---- multi-step small-grid kernel (vti_small.cuh): one cooperative launch per chunk of steps
static constexpr int MULTI_MAX = 1024;

static bool multi_eligible(const vti_s *h)
{
    return h->multi_enabled && h->small && h->cfg.nranks == 1 && h->cfg.check_every == 0 && !h->suppress_src &&
           !h->capturing && !getenv("VTI_FORCE_SPLIT") && h->grid <= h->multi_slots && h->done;
}

template <typename T>
static vti_status launch_multi_t(vti_s *h, int nsteps)
{
    if (!h->s_multi) CU(h, cudaMalloc(&h->s_multi, MULTI_MAX * sizeof(double)));
    MultiParams<T> M;
    const int cur0 = h->cur;
    for (int c = 0; c < 2; ++c) {   // both buffer parities (fill_params reads h->cur)
        h->cur = c;
        fill_params<T>(h, M.P[c], 0, h->nty, 0, 0, 1);
        M.tm_qcol[c] = h->tm_qcol[c];
    }
    h->cur = cur0;
    M.done = h->done;
    M.epoch0 = h->multi_epoch;
    M.nsteps = nsteps;
    M.cur0 = cur0;
    M.dir = h->dir;
    static const int mode = getenv("VTI_MULTI_MODE") ? atoi(getenv("VTI_MULTI_MODE")) : 0;
    M.mode = mode;
    const bool owned = h->has_src && h->src_j >= h->y0 && h->src_j < h->y0 + h->nyl;
    std::vector<T> sv(nsteps);
    for (int i = 0; i < nsteps; ++i)   // s(t^n) per step: double on the host, rounded once (reading c7)
        sv[i] = owned ? (T)(h->src_amp * ricker((double)(h->n + (int64_t)i * h->dir) * h->cfg.dt, h->src_f,
                                                h->src_t0))
                      : T(0);
    CU(h, cudaMemcpyAsync(h->s_multi, sv.data(), nsteps * sizeof(T), cudaMemcpyHostToDevice, h->stream));
    M.s_table = (const T *)h->s_multi;
    const bool io = h->io_active();
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(h->grid);
    lc.blockDim = dim3(h->small->threads);
    lc.dynamicSmemBytes = h->small->smem;
    lc.stream = h->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;   // every item's CTA co-resident: the epoch waits need it
    attr[0].val.cooperative = 1;
    lc.attrs = attr;
    lc.numAttrs = 1;
    void *args[] = {&M};
    CU(h, cudaLaunchKernelExC(&lc, io ? h->small->fn_multi_io : h->small->fn_multi, args));
    h->multi_epoch += (unsigned int)nsteps;
    h->cur = (cur0 + nsteps) & 1;
    h->n += (int64_t)nsteps * h->dir;
    advance_records(h, nsteps);
    return VTI_OK;
}

static vti_status launch_multi(vti_s *h, int nsteps)
{
    for (int done = 0; done < nsteps;) {
        const int m = std::min(MULTI_MAX, nsteps - done);
        vti_status s = h->es == 8 ? launch_multi_t<double>(h, m) : launch_multi_t<float>(h, m);
        if (s != VTI_OK) return s;
        done += m;
    }
    return VTI_OK;
}

extern "C" {

vti_status vti_prepare(vti_t h)
{
    if (!h) return VTI_E_PARAM;
    if (!h->model_set) return fail(h, VTI_E_STATE, "model not set (vti_set_model)");
    CU(h, cudaSetDevice(h->cfg.device));
    vti_status s;
    if (graph_eligible(h) && !multi_eligible(h))   // capture only: nothing executes, the state is untouched
        for (int z = 0; z < 2; ++z)
            for (int c = 0; c < 2; ++c)
                if (!h->gexec[z][c] && (s = build_graph(h, z, c)) != VTI_OK) return s;
    return VTI_OK;
}

vti_status vti_step(vti_t h, int32_t nsteps)
{
    if (!h) return VTI_E_PARAM;
    if (nsteps < 0) return fail(h, VTI_E_PARAM, "nsteps < 0");
    if (!h->model_set) return fail(h, VTI_E_STATE, "model not set (vti_set_model)");
    if (h->group_mode) return fail(h, VTI_E_STATE, "local-group handle: use vti_group_step");
    if (h->cfg.nranks > 1 && !h->peer && !h->comm_nccl)
        return fail(h, VTI_E_STATE, "nranks > 1 needs an nccl_id at create time or vti_ipc_connect");
    CU(h, cudaSetDevice(h->cfg.device));
    const bool multi = h->cfg.nranks > 1;
    vti_status s;
    if ((s = prepare_io(h)) != VTI_OK) return s;
    if (multi && h->halo_dirty) {   // halos of a state set by the caller
        if (h->peer) {
            if ((s = peer_release(h)) != VTI_OK || (s = peer_publish(h)) != VTI_OK) return s;
        } else {
            if ((s = pack_send(h, h->cur)) != VTI_OK) return s;
            CU(h, cudaEventRecord(h->ev_edge, h->stream));
            if ((s = exchange_nccl(h, h->cur)) != VTI_OK) return s;
            CU(h, cudaStreamWaitEvent(h->stream, h->ev_comm, 0));
        }
        h->halo_dirty = false;
    }
    if (!multi && nsteps >= 2 && multi_eligible(h)) {   // small grids: one cooperative launch for the lot
        if ((s = launch_multi(h, nsteps)) != VTI_OK) return s;
        CU(h, cudaGetLastError());
        return VTI_OK;
    }
    int it = 0;
    if (!multi && nsteps >= GRAPH_STEPS && graph_eligible(h)) {
        for (int z = 1; z >= 0 && h->graph_enabled; --z)   // large graphs first, then 32-step ones
            for (; it + graph_steps(z) <= nsteps; it += graph_steps(z))
                if ((s = replay_graph(h, z)) != VTI_OK) {
                    // capture is not possible on this stream (e.g. the legacy default stream): launch directly
                    cudaGetLastError();
                    h->graph_enabled = false;
                    invalidate_graphs(h);
                    break;
                }
    }
    // diagnostic: VTI_FORCE_SPLIT=1 runs a single slab with the multi-GPU two-launch schedule
    // (edge tile rows, then interior; no transport) to time what one rank's GPU does per step
    static const bool force_split = getenv("VTI_FORCE_SPLIT") && atoi(getenv("VTI_FORCE_SPLIT")) != 0;
    for (; it < nsteps; ++it) {
        if (!multi && force_split) {
            if ((s = launch_edge(h)) != VTI_OK || (s = launch_interior(h)) != VTI_OK) return s;
        } else if (!multi) {
            if ((s = launch_rows(h, 0, h->nty, 0, 0, h->zchunk, h->cap)) != VTI_OK) return s;
        } else if (h->peer && h->fused()) {
            // one launch: edge items first (their PEER stores feed the neighbours' halos), the
            // last edge item raises the neighbours' flags from the device, the interior follows
            if ((s = peer_fused_step(h)) != VTI_OK) return s;
        } else if (h->peer) {
            // the edge launch stores the neighbours' halo rows itself; the interior overlaps their edges
            if ((s = peer_pre_step(h)) != VTI_OK) return s;
            if ((s = launch_edge(h)) != VTI_OK) return s;
            if ((s = peer_post_edge(h)) != VTI_OK) return s;
            if ((s = launch_interior(h)) != VTI_OK) return s;
        } else {
            const int o = 1 - h->cur;
            // edge tile rows first, so the rows the neighbours need are ready early
            if ((s = launch_edge(h)) != VTI_OK) return s;
            if ((s = pack_send(h, o)) != VTI_OK) return s;
            CU(h, cudaEventRecord(h->ev_edge, h->stream));
            if ((s = exchange_nccl(h, o)) != VTI_OK) return s;
            if ((s = launch_interior(h)) != VTI_OK) return s;   // overlaps the exchange
            CU(h, cudaStreamWaitEvent(h->stream, h->ev_comm, 0));
        }
        h->cur = 1 - h->cur;
        h->n += h->dir;
        advance_records(h, 1);
        if (h->cfg.check_every > 0 && h->n % h->cfg.check_every == 0)
            if ((s = check_finite(h)) != VTI_OK) return s;
    }
    CU(h, cudaGetLastError());
    return VTI_OK;
}

vti_status vti_step_timed(vti_t h, int32_t nsteps, float *ms)
{
    if (!h) return VTI_E_PARAM;
    if (!ms) return fail(h, VTI_E_PARAM, "NULL ms");
    CU(h, cudaSetDevice(h->cfg.device));
    CU(h, cudaEventRecord(h->ev_t0, h->stream));
    vti_status s = vti_step(h, nsteps);
    if (s != VTI_OK) return s;
    CU(h, cudaEventRecord(h->ev_t1, h->stream));
    CU(h, cudaEventSynchronize(h->ev_t1));
    CU(h, cudaEventElapsedTime(ms, h->ev_t0, h->ev_t1));
    return VTI_OK;
}

vti_status vti_sync(vti_t h)
{
    if (!h) return VTI_E_PARAM;
    CU(h, cudaSetDevice(h->cfg.device));
    CU(h, cudaStreamSynchronize(h->stream));
    CU(h, cudaStreamSynchronize(h->comm));
    CU(h, cudaGetLastError());
    return VTI_OK;
}

int64_t vti_time_index(vti_t h) { return h ? h->n : -1; }

void *vti_stream(vti_t h) { return h ? (void *)h->stream : nullptr; }

vti_status vti_query(vti_t h, vti_info *info)
{
    if (!h || !info) return VTI_E_PARAM;
    info->y0 = h->y0;
    info->ny_local = h->nyl;
    info->nx_pad = h->nxp;
    info->layout = h->layout_zyx ? 0 : 1;
    info->tile_x = TX;
    info->tile_y = h->TY;
    info->rows_per_thread = h->K->rpt;
    info->producer_warp = h->K->wp;
    info->points_per_thread = h->K->px;
    info->small_kernel = h->small != nullptr;
    info->zchunk = h->zchunk;
    info->grid = h->small ? h->ntx * h->nty * h->nzc : std::min(h->ntx * h->nty * h->nzc, h->cap);
    info->work_items = h->ntx * h->nty * h->nzc;
    if (h->cfg.nranks > 1) {   // edge + interior step kernels (+ pack and unpack per neighbour with NCCL)
        const int neighbours = (h->cfg.rank > 0) + (h->cfg.rank < h->cfg.nranks - 1);
        int e1, e2;
        edge_rows(h, e1, e2);
        const bool peer_path = h->peer || h->group_mode;
        info->launches_per_step = peer_path && h->fused() ? 1   // one fused launch per step
                                                          : 1 + (e2 > e1 ? 1 : 0) + (peer_path ? 0 : 2 * neighbours);
    } else {
        info->launches_per_step = 1;
    }
    info->device_bytes = h->device_bytes;
    info->time_index = h->n;
    info->steps_per_launch = multi_eligible(h) ? MULTI_MAX : 1;
    return VTI_OK;
}

vti_status vti_set_tuning(vti_t h, int32_t zchunk, int32_t ctas_per_sm)
{
    if (!h) return VTI_E_PARAM;
    if (zchunk < 0 || ctas_per_sm < 0) return fail(h, VTI_E_PARAM, "negative tuning value");
    h->tune_zchunk = zchunk;
    h->tune_ctas = ctas_per_sm;
    CU(h, cudaSetDevice(h->cfg.device));
    return select_variant(h, h->K);
}

vti_status vti_set_variant(vti_t h, int32_t tile_y, int32_t producer_warp, int32_t rows_per_thread,
                           int32_t points_per_thread)
{
    if (!h) return VTI_E_PARAM;
    const KernelEntry *K = find_kernel(h->es, h->R, h->RZ, tile_y, producer_warp, rows_per_thread, points_per_thread);
    if (!K)
        return fail(h, VTI_E_UNSUPPORTED,
                    "no compiled variant (fp%d, r_xy %d, r_z %d, tile_y %d, producer_warp %d, rpt %d, px %d)", 8 * h->es,
                    h->R, h->RZ, tile_y, producer_warp, rows_per_thread, points_per_thread);
    CU(h, cudaSetDevice(h->cfg.device));
    CU(h, cudaStreamSynchronize(h->stream));
    h->explicit_variant = true;   // the caller picked this kernel: no small-grid substitution
    return select_variant(h, K);
}

vti_status vti_autotune(vti_t h, int32_t probe_steps, vti_tune_result *out)
{
    if (!h) return VTI_E_PARAM;
    if (probe_steps < 1) return fail(h, VTI_E_PARAM, "probe_steps must be >= 1");
    if (!h->model_set) return fail(h, VTI_E_STATE, "model not set");
    if (h->group_mode) return fail(h, VTI_E_STATE, "autotune is per handle; not for local-group handles");
    if (h->n != 0 || h->fields_touched)
        return fail(h, VTI_E_STATE, "autotune needs the initial zero state (call it before stepping or set_fields)");
    CU(h, cudaSetDevice(h->cfg.device));
    const KernelEntry *keep = h->K;
    const int keep_zc = h->tune_zchunk;
    float best_ms = 1e30f;
    const KernelEntry *best_k = keep;
    int best_zc = 0, ncand = 0;
    h->suppress_src = true;   // zero state, no injection: every probe step leaves u == 0
    h->explicit_variant = true;   // autotune chooses among the compiled step-kernel variants
    for (const KernelEntry *K : all_kernels(h->es, h->R, h->RZ)) {
        h->tune_zchunk = 0;
        vti_status s = select_variant(h, K);
        if (s != VTI_OK) continue;   // e.g. not resident on this device
        std::vector<int> zcs = {0, h->cfg.nz, (h->cfg.nz + 1) / 2, (h->cfg.nz + 3) / 4};
        for (int zc : zcs) {
            if (zc != 0 && zc < 4 * h->RZ) continue;
            h->tune_zchunk = zc;
            choose_schedule(h);
            float ms = 0.f;
            if ((s = vti_step(h, 2)) != VTI_OK) break;                       // warm-up
            if ((s = vti_step_timed(h, probe_steps, &ms)) != VTI_OK) break;
            ++ncand;
            if (ms < best_ms) {
                best_ms = ms;
                best_k = K;
                best_zc = zc;
            }
        }
        if (s != VTI_OK) {
            h->suppress_src = false;
            return s;
        }
    }
    h->suppress_src = false;
    h->n = 0;   // probes stepped a zero state; restore the time origin
    h->tune_zchunk = best_zc;
    vti_status s = select_variant(h, best_k ? best_k : keep);
    if (s != VTI_OK) return s;
    (void)keep_zc;
    if (out) {
        out->tile_y = h->K->ty;
        out->producer_warp = h->K->wp;
        out->rows_per_thread = h->K->rpt;
        out->points_per_thread = h->K->px;
        out->zchunk = h->zchunk;
        out->ms_per_step = best_ms / probe_steps;
        out->candidates = ncand;
    }
    return VTI_OK;
}

}  // extern "C"
