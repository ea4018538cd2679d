// vti_transport.cu -- the y-slab halo transports (see vti_internal.h and DESIGN.md 6).
#include <dlfcn.h>

#include "vti_internal.h"

// ============================================================ NCCL (dlopen'ed)
NcclApi &nccl()
{
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        const char *env = getenv("VTI_NCCL_LIB");
        const char *names[] = {env ? env : "libnccl.so.2", "libnccl.so.2", "libnccl.so"};
        void *h = nullptr;
        for (const char *n : names) {
            h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
            if (h) break;
        }
        if (!h) {
            api.err = std::string("cannot dlopen libnccl.so.2: ") + dlerror();
            return;
        }
#define LOADSYM(field, name)                                                   \
    api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name));        \
    if (!api.field) {                                                          \
        api.err = std::string("missing NCCL symbol ") + name;                  \
        return;                                                                \
    }
        LOADSYM(GetUniqueId, "ncclGetUniqueId");
        LOADSYM(CommInitRank, "ncclCommInitRank");
        LOADSYM(CommDestroy, "ncclCommDestroy");
        LOADSYM(Send, "ncclSend");
        LOADSYM(Recv, "ncclRecv");
        LOADSYM(GroupStart, "ncclGroupStart");
        LOADSYM(GroupEnd, "ncclGroupEnd");
        LOADSYM(GetErrorString, "ncclGetErrorString");
#undef LOADSYM
        api.ok = true;
    });
    return api;
}


// ============================================================ stream memory operations (peer flags)
typedef CUresult (*PFN_streamValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

struct StreamMemOps {
    PFN_streamValue32 wait = nullptr, write = nullptr;
};

static const StreamMemOps &stream_mem_ops()
{
    static StreamMemOps ops;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            ops.wait = reinterpret_cast<PFN_streamValue32>(p);
        if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            ops.write = reinterpret_cast<PFN_streamValue32>(p);
    });
    return ops;
}

// ============================================================ pack / unpack (NCCL transport)
// Internal element (x, y, k) of a buffer lives at base[y * ys + k * zs + x].
template <typename T>
__global__ void k_pack_rows(const T *__restrict__ buf, T *__restrict__ out, int row0, int R, int nz, int nx,
                            long long ys, long long zs)
{
    const int64_t n = (int64_t)nz * R * nx;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const int x = (int)(t % nx);
        const int64_t r = t / nx;
        const int y = (int)(r % R);
        const int k = (int)(r / R);
        out[t] = buf[(row0 + y) * ys + k * zs + x];
    }
}

template <typename T>
__global__ void k_unpack_rows(const T *__restrict__ in, T *__restrict__ buf, int row0, int R, int nz, int nx,
                              long long ys, long long zs)
{
    const int64_t n = (int64_t)nz * R * nx;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const int x = (int)(t % nx);
        const int64_t r = t / nx;
        const int y = (int)(r % R);
        const int k = (int)(r / R);
        buf[(row0 + y) * ys + k * zs + x] = in[t];
    }
}

template <typename T>
static void launch_pack(vti_s *h, const void *buf, void *out, int row0, cudaStream_t st)
{
    k_pack_rows<T><<<launch_grid(h), 256, 0, st>>>((const T *)buf, (T *)out, row0, h->R, h->cfg.nz, h->cfg.nx, h->ys,
                                                   h->zs);
}
template <typename T>
static void launch_unpack(vti_s *h, const void *in, void *buf, int row0, cudaStream_t st)
{
    k_unpack_rows<T><<<launch_grid(h), 256, 0, st>>>((const T *)in, (T *)buf, row0, h->R, h->cfg.nz, h->cfg.nx, h->ys,
                                                     h->zs);
}
static void pack(vti_s *h, const void *buf, void *out, int row0, cudaStream_t st)
{
    if (h->es == 8) launch_pack<double>(h, buf, out, row0, st);
    else launch_pack<float>(h, buf, out, row0, st);
}
static void unpack(vti_s *h, const void *in, void *buf, int row0, cudaStream_t st)
{
    if (h->es == 8) launch_unpack<double>(h, in, buf, row0, st);
    else launch_unpack<float>(h, in, buf, row0, st);
}

// ---- halo transport of p (y-slab decomposition)
// Halo'd row index: [0, R) rows from rank-1, [R, R+nyl) own rows, [R+nyl, 2R+nyl) rows from rank+1.
static size_t halo_elems(const vti_s *h) { return (size_t)h->cfg.nz * h->R * h->cfg.nx; }

// On the main stream: pack this rank's boundary rows of buffer b into sbuf[0] (-> rank-1) and sbuf[1] (-> rank+1).
vti_status pack_send(vti_s *h, int b)
{
    const int r = h->cfg.rank, nr = h->cfg.nranks;
    if (r > 0) pack(h, h->pbuf[b], h->sbuf[0], h->R, h->stream);
    if (r < nr - 1) pack(h, h->pbuf[b], h->sbuf[1], h->nyl, h->stream);
    CU(h, cudaGetLastError());
    return VTI_OK;
}

// On the comm stream: unpack rbuf[0] (from rank-1) and rbuf[1] (from rank+1) into the halo rows
// of the halo'd slab array buf (p: pbuf[b]; the adjoint's s1).
static vti_status unpack_recv_buf(vti_s *h, void *buf)
{
    const int r = h->cfg.rank, nr = h->cfg.nranks;
    if (r > 0) unpack(h, h->rbuf[0], buf, 0, h->comm);
    if (r < nr - 1) unpack(h, h->rbuf[1], buf, h->nyl + h->R, h->comm);
    CU(h, cudaGetLastError());
    return VTI_OK;
}
static vti_status unpack_recv(vti_s *h, int b) { return unpack_recv_buf(h, h->pbuf[b]); }

// Staged local-group transport (vti_group_step_staged): the NCCL branch of vti_step for
// handle i of a local group, with device copies from the neighbours' packed send buffers
// standing in for ncclSend/ncclRecv. Comm stream: after this rank's and the neighbours'
// ev_edge (their packs of buffer b), copy, unpack into the halo rows, record ev_comm.
static vti_status exchange_staged_buf(vti_s *const *hs, int n, int i, void *buf)
{
    vti_s *h = hs[i];
    const size_t bytes = halo_elems(h) * h->es;
    CU(h, cudaStreamWaitEvent(h->comm, h->ev_edge, 0));
    if (i > 0) {   // rank-1's last rows (its sbuf[1]) -> our bottom halo
        CU(h, cudaStreamWaitEvent(h->comm, hs[i - 1]->ev_edge, 0));
        CU(h, cudaMemcpyAsync(h->rbuf[0], hs[i - 1]->sbuf[1], bytes, cudaMemcpyDefault, h->comm));
    }
    if (i < n - 1) {   // rank+1's first rows (its sbuf[0]) -> our top halo
        CU(h, cudaStreamWaitEvent(h->comm, hs[i + 1]->ev_edge, 0));
        CU(h, cudaMemcpyAsync(h->rbuf[1], hs[i + 1]->sbuf[0], bytes, cudaMemcpyDefault, h->comm));
    }
    vti_status s = unpack_recv_buf(h, buf);
    if (s != VTI_OK) return s;
    CU(h, cudaEventRecord(h->ev_comm, h->comm));
    return VTI_OK;
}

static vti_status exchange_staged(vti_s *const *hs, int n, int i, int b)
{
    return exchange_staged_buf(hs, n, i, hs[i]->pbuf[b]);
}

// The main stream of handle i waits for its own and its neighbours' exchanges: its halo rows
// are complete, and the neighbours' copies out of its send buffers are done before the next
// pack overwrites them (what ncclSend's completion guarantees on the NCCL path).
static vti_status wait_staged(vti_s *const *hs, int n, int i)
{
    vti_s *h = hs[i];
    CU(h, cudaStreamWaitEvent(h->stream, h->ev_comm, 0));
    if (i > 0) CU(h, cudaStreamWaitEvent(h->stream, hs[i - 1]->ev_comm, 0));
    if (i < n - 1) CU(h, cudaStreamWaitEvent(h->stream, hs[i + 1]->ev_comm, 0));
    return VTI_OK;
}

// NCCL transport on the comm stream after ev_edge, then unpack into buf; records ev_comm.
static vti_status exchange_nccl_buf(vti_s *h, void *buf)
{
    NcclApi &api = nccl();
    CU(h, cudaStreamWaitEvent(h->comm, h->ev_edge, 0));
    const size_t cnt = halo_elems(h);
    const ncclDataType_t dt = h->es == 8 ? ncclFloat64 : ncclFloat32;
    const int r = h->cfg.rank, nr = h->cfg.nranks;
    ncclResult_t e = api.GroupStart();
    if (e == ncclSuccess && r > 0) {
        e = api.Send(h->sbuf[0], cnt, dt, r - 1, h->comm_nccl, h->comm);
        if (e == ncclSuccess) e = api.Recv(h->rbuf[0], cnt, dt, r - 1, h->comm_nccl, h->comm);
    }
    if (e == ncclSuccess && r < nr - 1) {
        e = api.Send(h->sbuf[1], cnt, dt, r + 1, h->comm_nccl, h->comm);
        if (e == ncclSuccess) e = api.Recv(h->rbuf[1], cnt, dt, r + 1, h->comm_nccl, h->comm);
    }
    ncclResult_t e2 = api.GroupEnd();
    if (e != ncclSuccess || e2 != ncclSuccess)
        return fail(h, VTI_E_COMM, "NCCL halo exchange: %s", api.GetErrorString(e != ncclSuccess ? e : e2));
    vti_status s = unpack_recv_buf(h, buf);
    if (s != VTI_OK) return s;
    CU(h, cudaEventRecord(h->ev_comm, h->comm));
    return VTI_OK;
}
vti_status exchange_nccl(vti_s *h, int b) { return exchange_nccl_buf(h, h->pbuf[b]); }

// The R boundary rows of an arbitrary halo'd slab array (the adjoint's s1, vti_adjoint.cu) into
// the neighbours' halo rows with the same pack / exchange / unpack as p's NCCL path: packs on each
// main stream (ev_edge), then over NCCL (nccl: one handle of a multi-process job, n = 1) or, in a
// local group, as copies from the neighbours' send buffers; every main stream then waits for the
// exchanges that read its send buffers and fill its halo rows.
vti_status rows_exchange(vti_s *const *hs, int n, void *const *bufs, bool nccl_path)
{
    vti_status s;
    for (int i = 0; i < n; ++i) {
        vti_s *h = hs[i];
        CU(h, cudaSetDevice(h->cfg.device));
        const int r = h->cfg.rank, nr = h->cfg.nranks;
        if (r > 0) pack(h, bufs[i], h->sbuf[0], h->R, h->stream);
        if (r < nr - 1) pack(h, bufs[i], h->sbuf[1], h->nyl, h->stream);
        CU(h, cudaGetLastError());
        CU(h, cudaEventRecord(h->ev_edge, h->stream));
    }
    for (int i = 0; i < n; ++i) {
        CU(hs[i], cudaSetDevice(hs[i]->cfg.device));
        if ((s = nccl_path ? exchange_nccl_buf(hs[i], bufs[i]) : exchange_staged_buf(hs, n, i, bufs[i])) != VTI_OK)
            return s;
    }
    for (int i = 0; i < n; ++i) {
        CU(hs[i], cudaSetDevice(hs[i]->cfg.device));
        if (nccl_path) CU(hs[i], cudaStreamWaitEvent(hs[i]->stream, hs[i]->ev_comm, 0));
        else if ((s = wait_staged(hs, n, i)) != VTI_OK) return s;
    }
    return VTI_OK;
}

// Fused peer-memory transport (no NCCL, no pack/copy/unpack): the edge launch
// itself stores p^{n+1} of this slab's first / last R rows into rank-1's top /
// rank+1's bottom halo rows through peer pointers (NVLink; the neighbours' own
// buffers in a local group, CUDA-IPC mappings across processes), so the halo
// travels tile by tile while the edge tiles are computed. Publication j is the
// halo of the level the next step reads; flags[] are monotone counters written
// by the neighbours with cuStreamWriteValue32 (which fences the kernel's peer
// stores before the flag) and waited on with cuStreamWaitValue32, all on the
// main stream:
//   before the edge launch that consumes publication j:
//     DATA >= j    the neighbours' rows of this level are in our halo
//     ACK  >= j-1  the neighbours have read the halo we are about to overwrite
//                  (publication j+1 lands in the buffer parity of j-1)
//   after it: the neighbours' ACK = j (only the edge launch reads halo rows)
//             and DATA = j+1.
// Enqueue-order rule: streams share a small pool of in-order hardware channels,
// so a value-wait may only wait on a write ENQUEUED EARLIER (the rule that makes
// event waits safe); a local group therefore enqueues every handle's step j
// writes before any handle's step j+1 waits, and splits a re-publication into
// a release half and a publish half.
enum { F_DATA_LO = 0, F_DATA_HI = 1, F_ACK_LO = 2, F_ACK_HI = 3 };
// the adjoint's s1 rows between multi-process peer ranks (rows_exchange_peer)
enum { F_S1DATA_LO = 4, F_S1DATA_HI = 5, F_S1ACK_LO = 6, F_S1ACK_HI = 7 };

static CUdeviceptr dev_ptr(const void *p) { return (CUdeviceptr)(uintptr_t)p; }
static bool has_side(const vti_s *h, int side) { return side == 0 ? h->cfg.rank > 0 : h->cfg.rank < h->cfg.nranks - 1; }

static vti_status flag_wait(vti_s *h, int idx, unsigned int v, bool remote_data)
{
    const StreamMemOps &ops = stream_mem_ops();
    if (!ops.wait) return fail(h, VTI_E_COMM, "stream memory operations unavailable");
    unsigned fl = CU_STREAM_WAIT_VALUE_GEQ;
    if (remote_data && h->flush_remote) fl |= CU_STREAM_WAIT_VALUE_FLUSH;
    if (ops.wait((CUstream)h->stream, dev_ptr(h->flags + idx), v, fl) != CUDA_SUCCESS)
        return fail(h, VTI_E_COMM, "cuStreamWaitValue32 failed");
    return VTI_OK;
}

// the neighbour on `side` sees flag `idx` (its own numbering) become v
static vti_status flag_write(vti_s *h, int side, int idx, unsigned int v)
{
    const StreamMemOps &ops = stream_mem_ops();
    if (!ops.write) return fail(h, VTI_E_COMM, "stream memory operations unavailable");
    if (ops.write((CUstream)h->stream, dev_ptr(h->peer_flags[side] + idx), v, CU_STREAM_WRITE_VALUE_DEFAULT) !=
        CUDA_SUCCESS)
        return fail(h, VTI_E_COMM, "cuStreamWriteValue32 failed");
    return VTI_OK;
}

// Multi-process peer ranks (CUDA IPC): publication j of buf's boundary rows, all on the main
// stream. Per side: once the neighbour has unpacked publication j-1 (S1ACK >= j-1), pack our rows
// straight into its receive buffer and raise its S1DATA to j; then, once its rows are in our
// receive buffer (S1DATA >= j), unpack them into buf's halo rows and raise its S1ACK to j.
// Every rank publishes in the same order, so the waits are always on writes the neighbour
// makes before its own waits.
vti_status rows_exchange_peer(vti_s *h, void *buf)
{
    const unsigned int j = ++h->adj_xseq;
    vti_status s;
    for (int side = 0; side < 2; ++side) {
        if (!has_side(h, side)) continue;
        if (j >= 2 && (s = flag_wait(h, side == 0 ? F_S1ACK_LO : F_S1ACK_HI, j - 1, false)) != VTI_OK) return s;
        pack(h, buf, h->peer_rbuf[side], side == 0 ? h->R : h->nyl, h->stream);
        CU(h, cudaGetLastError());
        if ((s = flag_write(h, side, side == 0 ? F_S1DATA_HI : F_S1DATA_LO, j)) != VTI_OK) return s;
    }
    for (int side = 0; side < 2; ++side) {
        if (!has_side(h, side)) continue;
        if ((s = flag_wait(h, side == 0 ? F_S1DATA_LO : F_S1DATA_HI, j, true)) != VTI_OK) return s;
        unpack(h, h->rbuf[side], buf, side == 0 ? 0 : h->nyl + h->R, h->stream);
        CU(h, cudaGetLastError());
        if ((s = flag_write(h, side, side == 0 ? F_S1ACK_HI : F_S1ACK_LO, j)) != VTI_OK) return s;
    }
    return VTI_OK;
}

vti_status peer_pre_step(vti_s *h)
{
    const unsigned int j = h->xseq;
    vti_status s;
    for (int side = 0; side < 2; ++side) {
        if (!has_side(h, side)) continue;
        if ((s = flag_wait(h, side == 0 ? F_DATA_LO : F_DATA_HI, j, true)) != VTI_OK) return s;
        if (j >= 1 && (s = flag_wait(h, side == 0 ? F_ACK_LO : F_ACK_HI, j - 1, false)) != VTI_OK) return s;
    }
    return VTI_OK;
}

vti_status peer_post_edge(vti_s *h)
{
    const unsigned int j = h->xseq;
    vti_status s;
    for (int side = 0; side < 2; ++side) {
        if (!has_side(h, side)) continue;
        if ((s = flag_write(h, side, side == 0 ? F_ACK_HI : F_ACK_LO, j)) != VTI_OK) return s;
        if ((s = flag_write(h, side, side == 0 ? F_DATA_HI : F_DATA_LO, j + 1)) != VTI_OK) return s;
    }
    h->xseq = j + 1;
    return VTI_OK;
}

// The same protocol in one launch: after the pre-step waits, the fused launch's last edge
// item stores ACK = j and DATA = j + 1 into the neighbours' flag words from the device.
vti_status peer_fused_step(vti_s *h)
{
    const unsigned int j = h->xseq;
    vti_status s = peer_pre_step(h);
    if (s != VTI_OK) return s;
    unsigned int *sig[4] = {nullptr, nullptr, nullptr, nullptr};
    unsigned int val[4] = {0, 0, 0, 0};
    if (has_side(h, 0)) {
        sig[0] = h->peer_flags[0] + F_ACK_HI;
        val[0] = j;
        sig[1] = h->peer_flags[0] + F_DATA_HI;
        val[1] = j + 1;
    }
    if (has_side(h, 1)) {
        sig[2] = h->peer_flags[1] + F_ACK_LO;
        val[2] = j;
        sig[3] = h->peer_flags[1] + F_DATA_LO;
        val[3] = j + 1;
    }
    if ((s = launch_fused(h, sig, val)) != VTI_OK) return s;
    h->xseq = j + 1;
    return VTI_OK;
}

// Re-publication of the current level (state set by the caller, vti_reverse). Release
// half: everything published so far is consumed or abandoned (stream-ordered after
// this rank's last read of its halo).
vti_status peer_release(vti_s *h)
{
    vti_status s;
    for (int side = 0; side < 2; ++side)
        if (has_side(h, side) && (s = flag_write(h, side, side == 0 ? F_ACK_HI : F_ACK_LO, h->xseq)) != VTI_OK)
            return s;
    return VTI_OK;
}

// Publish half: once the neighbours released every earlier publication, copy this
// rank's boundary rows of the current level into their halo rows (R contiguous
// rows per plane on both sides: one 2-D copy per neighbour), then DATA.
vti_status peer_publish(vti_s *h)
{
    const unsigned int j = ++h->xseq;
    vti_status s;
    // [z][y][x]: R rows are contiguous within each plane; [y][z][x]: the R rows of every plane are one block
    const size_t width = (size_t)h->R * h->ys * h->es;
    const size_t height = h->layout_zyx ? (size_t)h->cfg.nz : 1;
    for (int side = 0; side < 2; ++side) {
        if (!has_side(h, side)) continue;
        if ((s = flag_wait(h, side == 0 ? F_ACK_LO : F_ACK_HI, j - 1, false)) != VTI_OK) return s;
        const char *src = (const char *)h->pbuf[h->cur] + (size_t)(side == 0 ? h->R : h->nyl) * h->ys * h->es;
        const size_t spitch = h->layout_zyx ? (size_t)h->zs * h->es : width;
        const size_t dpitch = h->layout_zyx ? (size_t)h->peer_zs[side] * h->es : width;
        CU(h, cudaMemcpy2DAsync(h->peer_p[side][h->cur], dpitch, src, spitch, width, height, cudaMemcpyDefault,
                                h->stream));
        if ((s = flag_write(h, side, side == 0 ? F_DATA_HI : F_DATA_LO, j)) != VTI_OK) return s;
    }
    return VTI_OK;
}


extern "C" {

vti_status vti_nccl_unique_id(void *out128)
{
    if (!out128) return fail(nullptr, VTI_E_PARAM, "NULL output");
    NcclApi &api = nccl();
    if (!api.ok) return fail(nullptr, VTI_E_COMM, "%s", api.err.c_str());
    ncclUniqueId id;
    ncclResult_t r = api.GetUniqueId(&id);
    if (r != ncclSuccess) return fail(nullptr, VTI_E_COMM, "ncclGetUniqueId: %s", api.GetErrorString(r));
    memcpy(out128, &id, sizeof id);
    return VTI_OK;
}

// ---- multi-process fused peer transport over CUDA IPC
struct IpcBlob {
    uint32_t magic, version;
    int32_t rank, nranks, nyl, nxp, R, es, zyx;
    cudaIpcMemHandle_t pbuf[2], flags, rbuf[2];
};
static_assert(sizeof(IpcBlob) <= VTI_IPC_BYTES, "IPC blob too large");
static const uint32_t IPC_MAGIC = 0x56544932u;   // "VTI2"

vti_status vti_ipc_export(vti_t h, void *out)
{
    if (!h || !out) return VTI_E_PARAM;
    if (h->cfg.nranks < 2 || !h->flags) return fail(h, VTI_E_STATE, "vti_ipc_export needs nranks > 1");
    CU(h, cudaSetDevice(h->cfg.device));
    IpcBlob b;
    memset(&b, 0, sizeof b);
    b.magic = IPC_MAGIC;
    b.version = VTI_ABI_VERSION;
    b.rank = h->cfg.rank;
    b.nranks = h->cfg.nranks;
    b.nyl = h->nyl;
    b.nxp = h->nxp;
    b.R = h->R;
    b.es = h->es;
    b.zyx = h->layout_zyx;
    CU(h, cudaIpcGetMemHandle(&b.pbuf[0], h->pbuf[0]));
    CU(h, cudaIpcGetMemHandle(&b.pbuf[1], h->pbuf[1]));
    CU(h, cudaIpcGetMemHandle(&b.flags, h->flags));
    CU(h, cudaIpcGetMemHandle(&b.rbuf[0], h->rbuf[0]));
    CU(h, cudaIpcGetMemHandle(&b.rbuf[1], h->rbuf[1]));
    memset(out, 0, VTI_IPC_BYTES);
    memcpy(out, &b, sizeof b);
    return VTI_OK;
}

vti_status vti_ipc_connect(vti_t h, const void *lo, const void *hi)
{
    if (!h) return VTI_E_PARAM;
    const int r = h->cfg.rank, nr = h->cfg.nranks;
    if (nr < 2) return fail(h, VTI_E_STATE, "vti_ipc_connect needs nranks > 1");
    if ((r > 0) != (lo != nullptr) || (r < nr - 1) != (hi != nullptr))
        return fail(h, VTI_E_PARAM, "pass the blob of rank-1 (lo) and rank+1 (hi), NULL at the ends");
    const StreamMemOps &ops = stream_mem_ops();
    if (!ops.wait || !ops.write) return fail(h, VTI_E_COMM, "stream memory operations unavailable");
    CU(h, cudaSetDevice(h->cfg.device));
    const void *blobs[2] = {lo, hi};
    for (int side = 0; side < 2; ++side) {
        if (!blobs[side]) continue;
        IpcBlob b;
        memcpy(&b, blobs[side], sizeof b);
        if (b.magic != IPC_MAGIC || b.version != (uint32_t)VTI_ABI_VERSION || b.nranks != nr ||
            b.rank != (side == 0 ? r - 1 : r + 1) || b.nxp != h->nxp || b.R != h->R || b.es != h->es ||
            b.zyx != (int32_t)h->layout_zyx)
            return fail(h, VTI_E_PARAM, "IPC blob of the wrong rank, job, geometry or library version");
        void *pb[2] = {nullptr, nullptr}, *fl = nullptr;
        for (int k = 0; k < 2; ++k) {
            cudaError_t e = cudaIpcOpenMemHandle(&pb[k], b.pbuf[k], cudaIpcMemLazyEnablePeerAccess);
            if (e != cudaSuccess) return fail(h, VTI_E_COMM, "cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
            h->ipc_opened[3 * side + k] = pb[k];
        }
        cudaError_t e = cudaIpcOpenMemHandle(&fl, b.flags, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) return fail(h, VTI_E_COMM, "cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
        h->ipc_opened[3 * side + 2] = fl;
        // the neighbour's receive buffer for our rows: rank-1's rbuf[1] (from its rank+1), rank+1's rbuf[0]
        void *rb = nullptr;
        e = cudaIpcOpenMemHandle(&rb, b.rbuf[side == 0 ? 1 : 0], cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) return fail(h, VTI_E_COMM, "cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
        h->ipc_opened[6 + side] = rb;
        h->peer_rbuf[side] = rb;
        // rank-1: our first rows go to its top halo (row R + nyl); rank+1: our last rows to its row 0.
        // Same layout on both sides, so the row stride is ours (h->ys); the plane stride is theirs.
        const size_t row0 = side == 0 ? (size_t)b.R + b.nyl : 0;
        for (int k = 0; k < 2; ++k) h->peer_p[side][k] = (char *)pb[k] + row0 * h->ys * (size_t)b.es;
        h->peer_zs[side] = b.zyx ? (long long)(b.nyl + 2 * b.R) * b.nxp : (long long)b.nxp;
        h->peer_flags[side] = (unsigned int *)fl;
    }
    h->peer = true;
    h->group_mode = false;   // created with nccl_id = NULL; now a multi-process peer rank stepped by vti_step
    return VTI_OK;
}

int32_t vti_halo_transport(vti_t h) { return !h ? -1 : h->cfg.nranks < 2 ? 0 : h->peer ? 2 : h->comm_nccl ? 1 : 0; }

vti_status vti_debug_flags(vti_t h, uint32_t *get8, const uint32_t *set8)
{
    if (!h) return VTI_E_PARAM;
    if (!h->flags) return fail(h, VTI_E_STATE, "no flag words (nranks < 2)");
    CU(h, cudaSetDevice(h->cfg.device));
    CU(h, cudaStreamSynchronize(h->stream));
    if (get8) CU(h, cudaMemcpy(get8, h->flags, 8 * sizeof(unsigned int), cudaMemcpyDeviceToHost));
    if (set8) CU(h, cudaMemcpy(h->flags, set8, 8 * sizeof(unsigned int), cudaMemcpyHostToDevice));
    return VTI_OK;
}

vti_status vti_debug_rows(vti_t h, int32_t what, void *out)
{
    if (!h || !out || what < 0 || what > 5) return VTI_E_PARAM;
    CU(h, cudaSetDevice(h->cfg.device));
    CU(h, cudaStreamSynchronize(h->stream));
    const size_t row = (size_t)h->cfg.nx * h->es;
    if (what >= 4) {   // receive buffer [nz][R][nx], packed
        if (!h->rbuf[what - 4]) return fail(h, VTI_E_STATE, "no receive buffers (nranks < 2)");
        CU(h, cudaMemcpy(out, h->rbuf[what - 4], (size_t)h->cfg.nz * h->R * row, cudaMemcpyDeviceToHost));
        return VTI_OK;
    }
    if (!h->adj_s[what >> 1]) return fail(h, VTI_E_STATE, "no adjoint scratch buffers yet");
    // own rows [0, R) (what & 1 == 0) or [nyl - R, nyl) of scratch buffer what >> 1 -> out[nz][R][nx]
    const char *src = h->in(h->adj_s[what >> 1]) + (size_t)((what & 1) ? h->nyl - h->R : 0) * h->ys * h->es;
    for (int k = 0; k < h->cfg.nz; ++k)
        CU(h, cudaMemcpy2D((char *)out + (size_t)k * h->R * row, row, src + (size_t)k * h->zs * h->es,
                           (size_t)h->ys * h->es, row, h->R, cudaMemcpyDeviceToHost));
    return VTI_OK;
}

vti_status vti_debug_halo(vti_t h, int32_t level, int32_t side, void *out)
{
    if (!h || !out || (level != 0 && level != 1) || (side != 0 && side != 1)) return VTI_E_PARAM;
    CU(h, cudaSetDevice(h->cfg.device));
    CU(h, cudaStreamSynchronize(h->stream));
    const int b = level == 0 ? h->cur : 1 - h->cur;
    // halo'd rows [0, R) (side 0) or [nyl + R, nyl + 2R) (side 1) of p buffer b -> out[nz][R][nx]
    const char *src = (const char *)h->pbuf[b] + (size_t)(side == 0 ? 0 : h->nyl + h->R) * h->ys * h->es;
    const size_t row = (size_t)h->cfg.nx * h->es;
    for (int k = 0; k < h->cfg.nz; ++k)
        CU(h, cudaMemcpy2D((char *)out + (size_t)k * h->R * row, row, src + (size_t)k * h->zs * h->es,
                           (size_t)h->ys * h->es, row, h->R, cudaMemcpyDeviceToHost));
    return VTI_OK;
}

// Local group: the fused peer-memory transport between handles of one process
// (peer pointers are the neighbours' own device buffers), the same protocol as the
// multi-process CUDA-IPC form.
static void group_connect(vti_t *hs, int n)
{
    for (int i = 0; i < n; ++i) {
        vti_s *h = hs[i];
        h->peer = true;
        for (int side = 0; side < 2; ++side) {
            const vti_s *nb = side == 0 ? (i > 0 ? hs[i - 1] : nullptr) : (i < n - 1 ? hs[i + 1] : nullptr);
            for (int b = 0; b < 2; ++b)
                h->peer_p[side][b] = !nb ? nullptr
                                         : (char *)nb->pbuf[b] + (size_t)(side == 0 ? nb->R + nb->nyl : 0) * nb->ys * nb->es;
            h->peer_zs[side] = nb ? nb->zs : 0;
            h->peer_flags[side] = nb ? nb->flags : nullptr;
        }
    }
}

vti_status vti_group_step(vti_t *hs, int32_t n, int32_t nsteps)
{
    if (!hs || n < 1 || nsteps < 0) return VTI_E_PARAM;
    for (int i = 0; i < n; ++i) {
        if (!hs[i]) return VTI_E_PARAM;
        if (hs[i]->cfg.nranks != n || hs[i]->cfg.rank != i)
            return fail(hs[i], VTI_E_STATE, "group handle %d has rank %d / nranks %d", i, hs[i]->cfg.rank,
                        hs[i]->cfg.nranks);
        if (n > 1 && !hs[i]->group_mode) return fail(hs[i], VTI_E_STATE, "handle not created for local-group mode");
        if (!hs[i]->model_set) return fail(hs[i], VTI_E_STATE, "model not set");
        if (hs[i]->n != hs[0]->n) return fail(hs[i], VTI_E_STATE, "time indices differ inside the group");
    }
    if (n == 1) return vti_step(hs[0], nsteps);
    vti_status s;
    for (int i = 0; i < n; ++i) {
        CU(hs[i], cudaSetDevice(hs[i]->cfg.device));
        if ((s = prepare_io(hs[i])) != VTI_OK) return s;
    }
    for (int i = 0; i < n; ++i)
        if (hs[i]->xseq != hs[0]->xseq || hs[i]->cur != hs[0]->cur)
            return fail(hs[i], VTI_E_STATE, "halo publications or buffer parity differ inside the group");
    group_connect(hs, n);
    bool dirty = false;
    for (int i = 0; i < n; ++i) dirty |= hs[i]->halo_dirty;
    if (dirty) {   // every release before any publish (enqueue-order rule)
        for (int i = 0; i < n; ++i) {
            CU(hs[i], cudaSetDevice(hs[i]->cfg.device));
            if ((s = peer_release(hs[i])) != VTI_OK) return s;
        }
        for (int i = 0; i < n; ++i) {
            CU(hs[i], cudaSetDevice(hs[i]->cfg.device));
            if ((s = peer_publish(hs[i])) != VTI_OK) return s;
            hs[i]->halo_dirty = false;
        }
    }
    for (int it = 0; it < nsteps; ++it) {
        for (int i = 0; i < n; ++i) {   // waits on the previous step's writes only
            vti_s *h = hs[i];
            CU(h, cudaSetDevice(h->cfg.device));
            if (h->fused()) {
                if ((s = peer_fused_step(h)) != VTI_OK) return s;
                continue;
            }
            if ((s = peer_pre_step(h)) != VTI_OK) return s;
            if ((s = launch_edge(h)) != VTI_OK) return s;
            if ((s = peer_post_edge(h)) != VTI_OK) return s;
        }
        for (int i = 0; i < n; ++i) {
            vti_s *h = hs[i];
            CU(h, cudaSetDevice(h->cfg.device));
            if (!h->fused() && (s = launch_interior(h)) != VTI_OK) return s;
            h->cur = 1 - h->cur;
            h->n += h->dir;
            advance_records(h, 1);
            if (h->cfg.check_every > 0 && h->n % h->cfg.check_every == 0 && (s = check_finite(h)) != VTI_OK)
                return s;
        }
    }
    return VTI_OK;
}

vti_status vti_group_step_staged(vti_t *hs, int32_t n, int32_t nsteps)
{
    if (!hs || n < 2 || nsteps < 0) return VTI_E_PARAM;
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
        if ((s = prepare_io(hs[i])) != VTI_OK) return s;
        CU(hs[i], cudaStreamSynchronize(hs[i]->comm));
    }
    bool dirty = false;
    for (int i = 0; i < n; ++i) dirty |= hs[i]->halo_dirty;
    if (dirty) {   // halos of the current level (state set by the caller, vti_reverse)
        for (int i = 0; i < n; ++i) {
            CU(hs[i], cudaSetDevice(hs[i]->cfg.device));
            if ((s = pack_send(hs[i], hs[i]->cur)) != VTI_OK) return s;
            CU(hs[i], cudaEventRecord(hs[i]->ev_edge, hs[i]->stream));
        }
        for (int i = 0; i < n; ++i) {
            CU(hs[i], cudaSetDevice(hs[i]->cfg.device));
            if ((s = exchange_staged(hs, n, i, hs[i]->cur)) != VTI_OK) return s;
        }
        for (int i = 0; i < n; ++i) {
            CU(hs[i], cudaSetDevice(hs[i]->cfg.device));
            if ((s = wait_staged(hs, n, i)) != VTI_OK) return s;
            hs[i]->halo_dirty = false;
        }
    }
    for (int it = 0; it < nsteps; ++it) {
        for (int i = 0; i < n; ++i) {   // edge tile rows first, then pack the rows the neighbours need
            vti_s *h = hs[i];
            CU(h, cudaSetDevice(h->cfg.device));
            if ((s = launch_edge(h)) != VTI_OK) return s;
            if ((s = pack_send(h, 1 - h->cur)) != VTI_OK) return s;
            CU(h, cudaEventRecord(h->ev_edge, h->stream));
        }
        for (int i = 0; i < n; ++i) {   // exchange on the comm streams, overlapped with the interiors
            CU(hs[i], cudaSetDevice(hs[i]->cfg.device));
            if ((s = exchange_staged(hs, n, i, 1 - hs[i]->cur)) != VTI_OK) return s;
        }
        for (int i = 0; i < n; ++i) {
            vti_s *h = hs[i];
            CU(h, cudaSetDevice(h->cfg.device));
            if ((s = launch_interior(h)) != VTI_OK) return s;
        }
        for (int i = 0; i < n; ++i) {
            vti_s *h = hs[i];
            CU(h, cudaSetDevice(h->cfg.device));
            if ((s = wait_staged(hs, n, i)) != VTI_OK) return s;
        }
        for (int i = 0; i < n; ++i) {
            vti_s *h = hs[i];
            CU(h, cudaSetDevice(h->cfg.device));
            h->cur = 1 - h->cur;
            h->n += h->dir;
            advance_records(h, 1);
            if (h->cfg.check_every > 0 && h->n % h->cfg.check_every == 0 && (s = check_finite(h)) != VTI_OK)
                return s;
        }
    }
    return VTI_OK;
}

}  // extern "C"
