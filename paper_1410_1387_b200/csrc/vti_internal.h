// vti_internal.h -- shared internals of the host runtime (not part of the C ABI).
//
// The runtime is split by concern:
//   vti_runtime.cu   handle lifecycle, model/field I/O, stepping, CUDA graphs,
//                    receivers, time reversal, tuning (and the auxiliary kernels);
//   vti_schedule.cu  host-side planning: tile rows, edge/interior split, z-chunks
//                    and the CTA cap (vti_plan, vti_slab);
//   vti_transport.cu the y-slab halo transports: fused peer stores (local group,
//                    CUDA IPC), NCCL send/recv (dlopen'ed), vti_group_step.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "vti.h"
#include "vti_kernel.cuh"
#include "vti_small.cuh"
#include "vti_variants.h"

using namespace vti;

// ============================================================ NCCL (dlopen'ed in vti_transport.cu)
typedef struct ncclComm *ncclComm_t;
typedef struct {
    char internal[128];
} ncclUniqueId;
typedef enum { ncclSuccess = 0 } ncclResult_t;
typedef enum { ncclFloat32 = 7, ncclFloat64 = 8 } ncclDataType_t;

struct NcclApi {
    bool ok = false;
    std::string err;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi &nccl();

// ============================================================ N4 point sets
// CSR over (plane k, local row yl) of (x, column) entries sorted by x (StepParams::inj_* / rec_*).
struct DevPointSet {
    int *off = nullptr;    // device [nz * nyl + 1]
    int2 *ent = nullptr;   // device [n]
    int n = 0;
};

// ============================================================ handle
struct vti_s {
    vti_config cfg{};
    std::string err;
    int es = 4;                               // element size: 4 (fp32) or 8 (fp64)
    int R = 0, RZ = 0, TY = 16;
    int y0 = 0, nyl = 0, nxp = 0, rows = 0;   // rows = nyl + 2R (halo'd)
    long long ys = 0, zs = 0;                 // row / plane strides (elements)
    bool layout_zyx = true;                   // [z][y][x] (default) or [y][z][x]
    int ntx = 0, nty = 0;
    const KernelEntry *K = nullptr;
    int smem_bytes = 0;
    int sms = 0, ctas_per_sm = 0;
    int zchunk = 0, nzc = 0, grid = 0;        // single-launch schedule
    int zchunk_edge = 0, zchunk_inner = 0;    // nranks > 1: per-launch chunking
    int cap = 0, cap_edge = 0, cap_inner = 0; // CTAs per launch at most (plan_sched)
    int tune_zchunk = 0, tune_ctas = 0;       // vti_set_tuning / vti_autotune overrides (0 = model)
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    cudaStream_t comm = nullptr;
    cudaEvent_t ev_edge = nullptr, ev_comm = nullptr, ev_t0 = nullptr, ev_t1 = nullptr;
    void *pbuf[2] = {nullptr, nullptr};       // halo'd arrays (base = first halo row)
    void *qbuf[2] = {nullptr, nullptr};
    void *vx2 = nullptr, *vn2 = nullptr, *vz2 = nullptr;
    void *sbuf[2] = {nullptr, nullptr};       // packed send rows: [0] to rank-1, [1] to rank+1
    void *rbuf[2] = {nullptr, nullptr};       // packed recv rows: [0] from rank-1, [1] from rank+1
    void *zrow = nullptr, *gx = nullptr, *gy = nullptr;
    void *staging = nullptr;
    size_t staging_bytes = 0;
    unsigned long long *counters = nullptr;
    unsigned int *flag = nullptr;
    unsigned long long *sync_ctr = nullptr;   // round-alignment counter (monotone across launches)
    unsigned long long sync_value = 0;        // its value once all launched work has finished
    unsigned long long *edge_ctr = nullptr;   // fused multi-GPU step: edge items completed (monotone)
    unsigned long long edge_value = 0;        // its value once all launched work has finished
    // peer transport schedule: one fused launch per step (edge items first, device-side flags) or
    // the edge + interior pair. Default: fused for a multi-process rank (one slab per GPU), the
    // pair for a local group (slabs sharing a GPU interleave better); env VTI_FUSED_STEP=1/0 forces.
    int fused_env = -1;
    bool fused() const { return fused_env >= 0 ? fused_env != 0 : !group_mode; }
    bool align_rounds = true;                 // env VTI_ALIGN=0 disables
    int64_t device_bytes = 0;
    CUtensorMap tm_ph[2], tm_pi[2], tm_q[2], tm_vx, tm_vn, tm_vz;
    CUtensorMap tm_qcol[2];                   // q^n column views (box depth 2 R_z + 1) for the small-grid kernel
    const SmallEntry *small = nullptr;        // small-grid kernel in use (single slab, 1-plane items), or NULL
    // multi-step small-grid kernel (vti_small_multi_kernel): one cooperative launch per vti_step
    // call (chunks of MULTI_MAX steps); done[] = per-item epoch counters, multi_epoch their value
    int multi_slots = 0;                      // co-resident multi-step CTAs on the device
    bool multi_enabled = false;               // env VTI_MULTI=1 enables (measured slower than graph
                                              // replays of the one-step kernel on C1)
    unsigned int *done = nullptr;
    int done_items = 0;
    unsigned int multi_epoch = 0;
    void *s_multi = nullptr;                  // device: s(t^n) of each step of a launch
    bool explicit_variant = false;            // env VTI_TY/WP/RPT/PX or vti_set_variant / vti_autotune chose K
    double cxy[MAX_R + 1] = {0};              // w^xy / h^2 in double; rounded to T at launch (reading c3)
    int cur = 0;                              // pbuf[cur], qbuf[cur] hold u^n
    int64_t n = 0;                            // time index
    bool model_set = false;
    std::vector<char> model_planes;           // per plane: uploaded by vti_set_model* (model_set = all)
    int64_t aniso_warn = 0;
    bool has_src = false;
    int src_i = 0, src_j = 0, src_k = 0, src_mask = 0;
    double src_f = 15.0, src_t0 = 0.0, src_amp = 1.0;
    ncclComm_t comm_nccl = nullptr;
    bool group_mode = false;
    // fused peer-memory halo transport (local group, or multi-process after vti_ipc_connect):
    // the edge launch stores p^{n+1}'s boundary rows straight into the neighbours' halo rows;
    // flags[] = {DATA_LO, DATA_HI, ACK_LO, ACK_HI} of p's halo, then the same four for the adjoint's
    // s1 rows (multi-process peer ranks), written by the neighbours
    bool peer = false;
    unsigned int *flags = nullptr;
    void *peer_p[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};   // [side][b]: neighbour's pbuf[b] at the
                                                                      // first halo row this rank writes
    long long peer_zs[2] = {0, 0};                    // the neighbours' plane strides (elements)
    unsigned int *peer_flags[2] = {nullptr, nullptr}; // the neighbours' flags
    void *ipc_opened[8] = {};                         // cudaIpcCloseMemHandle on destroy
    unsigned int xseq = 0;                            // halo publications so far (the flag values)
    void *peer_rbuf[2] = {nullptr, nullptr};          // [side]: the neighbour's receive buffer for our rows
    unsigned int adj_xseq = 0;                        // s1 row publications so far (peer adjoint)
    bool flush_remote = false;                        // CU_STREAM_WAIT_VALUE_FLUSH supported
    bool halo_dirty = false;
    bool suppress_src = false;                // autotune probes inject nothing
    bool fields_touched = false;              // vti_set_fields* called (state may be non-zero)
    int dir = 1;                              // +1 forward in time, -1 after vti_reverse
    // CUDA graphs of GRAPH_STEPS single-slab steps (launch-bound small grids)
    bool graph_enabled = true;                // env VTI_GRAPH=0 disables
    bool capturing = false;
    int capture_index = 0;
    cudaGraphExec_t gexec[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};   // [32 / large steps][starting parity]
    void *s_graph = nullptr;                  // device: GRAPH_STEPS source samples of T
    std::vector<double> s_host;
    // N4 point sets of this slab, gathered / injected inside the step
    // kernels' IO instantiations (StepParams::inj_* / rec_*)
    DevPointSet rec_set, inj_set;
    // receivers (this slab's subset, in the caller's order)
    int nrec = 0, rec_mask = 0, rec_cap = 0, rec_steps = 0;
    void *traces = nullptr;                   // device: [rec_cap][nrec][nf] of T
    std::vector<int32_t> rec_ids;             // global receiver index of each local receiver
    // trace injection: rows [0, inj_nt) of inj_tr = time indices inj_t_first.., inj_cols columns
    void *inj_tr = nullptr;                   // device: [inj_nt][inj_cols] of T
    int inj_cols = 0, inj_mask = 0, inj_nt = 0;
    int64_t inj_t_first = 0;
    long long *dyn = nullptr;                 // device: graph-replay header {inj row, rec row, dir}
    void *adj_s[2] = {nullptr, nullptr};      // vti_step_adjoint scratch: s1, s2 (vti_adjoint.cu)
    // the TMA adjoint kernel (vti_adjoint.cu): transposed z-weight rows [nz][zrow] and, per buffer
    // parity c of psi^m, its 9 tensor maps; adj_tma = 0 until built, -1 if setup failed, else the
    // kernel's grid cap (resident CTAs)
    void *adj_wt = nullptr;
    CUtensorMap adj_tm[2][9];
    CUtensorMap adj_tm_s1[2];                 // halo'd views of the two s1 scratch buffers (two-pass TMA form)
    int adj_tma = 0, adj_tma_ch = 0;          // grid caps of the plain and the chained kernel
    bool io_active() const { return (rec_set.n > 0 && rec_cap > 0) || inj_set.n > 0; }

    size_t total_elems() const { return (size_t)cfg.nz * rows * nxp; }
    char *in(void *base) const { return (char *)base + (long long)R * ys * es; }   // interior view
    char *p_int(int b) const { return in(pbuf[b]); }
    char *q_int(int b) const { return in(qbuf[b]); }
};


// ============================================================ shared helpers
// per-handle error text (h == NULL: the last create error); returns s
vti_status fail(vti_s *h, vti_status s, const char *fmt, ...);

#define CU(h, call)                                                                                   \
    do {                                                                                              \
        cudaError_t e_ = (call);                                                                      \
        if (e_ != cudaSuccess) return fail(h, VTI_E_CUDA, "%s failed: %s", #call, cudaGetErrorString(e_)); \
    } while (0)

// grid of the grid-stride auxiliary kernels
inline int launch_grid(const vti_s *h) { return 4 * h->sms; }

// vti_schedule.cu
int precision_bits(const vti_config *c);
vti_status check_cfg(const vti_config *c);
int slots(const vti_s *h);                      // CTA slots of a launch (resident CTAs, optionally capped)
void edge_rows(const vti_s *h, int &e1, int &e2);
void choose_schedule(vti_s *h);                 // z-chunks and CTA caps of the full / edge / interior launches

// vti_runtime.cu
vti_status launch_edge(vti_s *h);               // tile rows the neighbours receive (PEER kernel when connected)
vti_status launch_interior(vti_s *h);
void advance_records(vti_s *h, int steps);      // receiver rows written by `steps` steps (fused in the kernel)
// 3-D tensor map over (x, y, z) of an array with this handle's strides: rows of the view, box bx x by x bz
vti_status encode(vti_s *h, CUtensorMap *tm, void *base, int rows, int bx, int by,
                  CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_256B, int bz = 1);
vti_status prepare_io(vti_s *h);                // an IO-capable step kernel while a point set is active
vti_status check_finite(vti_s *h);              // check_every: INSTABILITY on a non-finite value

// vti_transport.cu
vti_status pack_send(vti_s *h, int b);          // NCCL: boundary rows of buffer b -> send buffers (main stream)
// R boundary rows of halo'd slab arrays bufs[i] into the neighbours' halo rows: NCCL (one
// handle of a multi-process job) or copies between a local group's send / recv buffers
vti_status rows_exchange(vti_s *const *hs, int n, void *const *bufs, bool nccl_path);
// the same over CUDA IPC for a multi-process peer rank: rows packed straight into the
// neighbours' receive buffers, ordered by flag words 4..7
vti_status rows_exchange_peer(vti_s *h, void *buf);
vti_status exchange_nccl(vti_s *h, int b);      // NCCL: send/recv + unpack on the comm stream, records ev_comm
vti_status peer_pre_step(vti_s *h);             // peer: wait for the halo this step reads
vti_status peer_post_edge(vti_s *h);            // peer: after the edge launch, ACK + DATA to the neighbours
vti_status peer_release(vti_s *h);              // peer re-publication (set_fields, reverse), first half
vti_status peer_publish(vti_s *h);              // ... second half
vti_status peer_fused_step(vti_s *h);           // peer: one launch (edge items first, device-side flags)

// vti_runtime.cu: the fused multi-GPU launch -- edge tile rows (items first, PEER stores)
// then the interior rows; the last edge item stores sig_val[i] to sig[i] (release, system)
vti_status launch_fused(vti_s *h, unsigned int *const sig[4], const unsigned int sig_val[4]);
