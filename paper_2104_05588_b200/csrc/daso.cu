// libdaso.so runtime: the DASO context, its NCCL communicators and the per-batch
// step (Fig. 2-5).  Host C++; all arithmetic runs in the fused
// kernels of kernels.cu, all communication in NCCL over NVLink / NVSwitch.
//
// Communicators (Fig. 1): the world comm is split into
//   node  comm: color = node,  key = local  -> rank in node comm  == local id
//   group comm: color = local, key = node   -> rank in group comm == node id
// The node comm is only ever used on the caller's (compute) stream and the group
// comm only on the library's side stream, so no communicator is driven from two
// streams; every rank issues the same sequence of collectives on each comm because
// every rank runs the same deterministic schedule.
//
// Data layout in HBM: caller-owned flat fp32 x, g, v [n_pad];
// library-owned ring slot [P][seg] wire elements (seg = n_pad in the faithful mode,
// n_pad / G in the sharded mode); 4-byte non-finite flag.
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "daso_internal.h"

struct daso_vcluster;

struct daso_ctx {
    int world = 0, G = 0, P = 0, rank = 0, node = 0, local = 0;
    int device = 0;
    daso_config cfg{};
    daso_sched_config scfg{};
    daso::Schedule* sched = nullptr;

    ncclComm_t world_comm = nullptr, node_comm = nullptr, group_comm = nullptr;
    ncclComm_t bucket_comm = nullptr;   // node comm for backward-overlapped bucket all-reduces (N2)
    cudaStream_t side = nullptr;
    cudaEvent_t ev_packed = nullptr, ev_exchanged = nullptr;

    bool bound = false;
    float *x = nullptr, *g = nullptr, *v = nullptr;
    int64_t n = 0, n_pad = 0, seg = 0;
    void* slot = nullptr;
    size_t wire_bytes = 2;
    uint32_t* d_flag = nullptr;

    bool inflight = false;
    int infl_group = -1, infl_S = 0;
    bool exch_enabled = true;   // daso_set_exchange(0): timing knob, the group all-gather is skipped

    // copy-engine group exchange (cfg.exchange == DASO_EXCH_CE): every member pushes its packed row
    // into row `node` of every group member's slot with cudaMemcpyAsync (copy engines over NVLink,
    // CUDA IPC mappings), then raises a flag there with cuStreamWriteValue64; receivers wait with
    // cuStreamWaitValue64.  xs = own [2P] u64: [0,P) epoch of the last row received from member i,
    // [P,2P) epoch of the last exchange member i has consumed (merged / averaged) — flow control
    // before a row of i's slot is overwritten.
    bool ce = false;
    std::vector<void*> peer_slot;                 // [P] group members' slot bases (own = slot)
    std::vector<unsigned long long*> peer_xs;     // [P] group members' xs arrays
    unsigned long long* xs = nullptr;
    unsigned long long exch_epoch = 0;            // exchanges this rank has issued
    std::vector<void*> ipc_group;                 // opened group mappings
    std::vector<cudaStream_t> ce_streams;         // one per other member: the pushes run on parallel copy engines
    std::vector<cudaEvent_t> ce_done;             // [P-1] fork/join events

    // fused mode: node peers' buffers mapped through CUDA IPC (NVLink peer memory)
    float* peer_x[daso::kMaxPeers] = {};
    float* peer_g[daso::kMaxPeers] = {};
    unsigned long long* peer_sig[daso::kMaxPeers] = {};
    unsigned long long* sig = nullptr;   // own [2][G] signals followed by the CTA counter
    unsigned long long epoch = 0;
    std::vector<void*> ipc_opened;

    // library-owned buckets (daso_alloc_bind, cudaMalloc)
    void* own_cuda[3] = {};

    // virtual cluster (daso_vcluster_*): this ctx is one of W virtual ranks on ONE GPU; the
    // group all-gather and the blocking tail are run by the cluster driver after every rank's
    // batch (loopback transport), the node tier's peers are the sibling ranks' buffers
    daso_vcluster* vc = nullptr;
    bool vc_sent = false, vc_blocking = false;
    int vc_group = -1;
    unsigned long long* vc_node_sig = nullptr;   // the node's [G][2G+2] signal block (local 0 pre-sets it)

    daso_record last{};
    std::string err;

    // tracing (daso_trace_enable / daso_trace_read)
    struct SpanRec { cudaEvent_t a, b; int phase; double bytes, nvl; };
    bool tracing = false;
    std::vector<cudaEvent_t> pool;
    size_t pool_used = 0;
    std::vector<SpanRec> spans;
    daso_trace acc{};

    daso_status fail(daso_status s, const char* fmt, ...) {
        char buf[512];
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(buf, sizeof buf, fmt, ap);
        va_end(ap);
        err = buf;
        return s;
    }
};

#define CUDA_TRY(c, expr)                                                                          \
    do {                                                                                           \
        cudaError_t e_ = (expr);                                                                   \
        if (e_ != cudaSuccess) return (c)->fail(DASO_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(e_)); \
    } while (0)
#define KERN_TRY(c, expr)                                                                          \
    do {                                                                                           \
        int e_ = (expr);                                                                           \
        if (e_ != 0) return (c)->fail(DASO_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(cudaError_t(e_))); \
    } while (0)
#define NCCL_TRY(c, expr)                                                                          \
    do {                                                                                           \
        ncclResult_t r_ = (expr);                                                                  \
        if (r_ != ncclSuccess) return (c)->fail(DASO_ERR_NCCL, "%s: %s", #expr, ncclGetErrorString(r_)); \
    } while (0)
#define STATUS_TRY(expr)                  \
    do {                                  \
        daso_status s_ = (expr);          \
        if (s_ != DASO_OK) return s_;     \
    } while (0)

namespace {

ncclDataType_t wire_nccl(int wire) { return wire == DASO_WIRE_BF16 ? ncclBfloat16 : ncclFloat32; }

// ---- state checks -----------------------------------------------------------
daso_status poll_async(daso_ctx* c) {
    cudaError_t e = cudaPeekAtLastError();
    if (e != cudaSuccess) return c->fail(DASO_ERR_CUDA, "asynchronous CUDA error: %s", cudaGetErrorString(e));
    ncclComm_t comms[4] = {c->world_comm, c->node_comm, c->group_comm, c->bucket_comm};
    for (ncclComm_t m : comms) {
        if (!m) continue;
        ncclResult_t a = ncclSuccess;
        ncclCommGetAsyncError(m, &a);
        if (a != ncclSuccess && a != ncclInProgress)
            return c->fail(DASO_ERR_NCCL, "asynchronous NCCL error: %s", ncclGetErrorString(a));
    }
    return DASO_OK;
}

daso_status require_bound(daso_ctx* c) {
    if (!c->bound) return c->fail(DASO_ERR_PROTOCOL, "daso_bind has not been called");
    return poll_async(c);
}

// ---- kernel argument builders --------------------------------------------------
daso::KernelArgs base_args(daso_ctx* c, int64_t off, int64_t len, float lr) {
    daso::KernelArgs a;
    a.x = c->x + off;
    a.v = c->v + off;
    a.g = c->g + off;
    a.n = len;
    a.lr = lr;
    a.mu = c->cfg.momentum;
    a.wd = c->cfg.weight_decay;
    a.gscale = 1.0f / float(c->G);      // Fig. 2 average = node sum x 1/G (R4)
    a.slot = c->slot;
    a.slot_stride = c->seg;
    a.P = c->P;
    a.flag = c->cfg.check_finite ? c->d_flag : nullptr;
    a.err = c->d_flag;
    return a;
}

void* own_segment(daso_ctx* c) {
    return static_cast<char*>(c->slot) + size_t(c->node) * size_t(c->seg) * c->wire_bytes;
}

// ---- tracing ---------------------------------------------------------------------
enum Phase { PH_KERNEL = 0, PH_LOCAL = 1, PH_NODE = 2, PH_WAIT = 3, PH_EXCH = 4 };

cudaEvent_t next_event(daso_ctx* c) {
    if (c->pool_used == c->pool.size()) {
        cudaEvent_t e = nullptr;
        if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
        c->pool.push_back(e);
    }
    return c->pool[c->pool_used++];
}

struct Span {   // RAII event pair around one phase on one stream
    daso_ctx* c;
    cudaStream_t s;
    int phase;
    double bytes, nvl;
    cudaEvent_t a = nullptr;
    Span(daso_ctx* c_, cudaStream_t s_, int ph, double b, double nvl_ = 0.0) : c(c_), s(s_), phase(ph), bytes(b), nvl(nvl_) {
        if (c->tracing && (a = next_event(c)) != nullptr) cudaEventRecord(a, s);
    }
    ~Span() {
        if (!a) return;
        cudaEvent_t b = next_event(c);
        if (!b) return;
        cudaEventRecord(b, s);
        c->spans.push_back({a, b, phase, bytes, nvl});
    }
};

// algorithmic HBM bytes per element of a fused launch
double kernel_bytes_per_elem(int ops, int P, double wb) {
    double b = 0;
    if (ops & daso::OP_UPDATE) b += 20;                                  // x, v read+write, g read
    else if (ops & daso::OP_MERGE) b += 8;                               // x read+write
    else if (ops & daso::OP_PACK) b += 4;                                // x read
    if (ops & daso::OP_MERGE) b += P * wb;                               // P slot rows
    if (ops & daso::OP_AVERAGE) b += P * wb + 4;                         // P slot rows, x write
    if (ops & daso::OP_PACK) b += wb;                                    // own slot segment
    return b;
}

int launch(daso_ctx* c, int ops, const daso::KernelArgs& a, cudaStream_t s) {
    // NVLink bytes per direction of a kernel push (blocking sync, below): the packed row to each member
    Span sp(c, s, PH_KERNEL, kernel_bytes_per_elem(ops, a.P, double(c->wire_bytes)) * double(a.n),
            double(a.npush) * double(c->wire_bytes) * double(a.n));
    return daso::launch_fused(ops, c->cfg.wire, a, s);
}

// ---- stream memory operations (driver API, resolved at run time) -----------------------
typedef CUresult (*PfnWriteValue64)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
typedef CUresult (*PfnWaitValue64)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
typedef CUresult (*PfnDevAttr)(int*, CUdevice_attribute, CUdevice);

template <typename F>
F driver_fn(const char* name) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) == cudaSuccess && q == cudaDriverEntryPointSuccess)
        return reinterpret_cast<F>(p);
    return nullptr;
}
PfnWriteValue64 write_value64() {
    static PfnWriteValue64 f = driver_fn<PfnWriteValue64>("cuStreamWriteValue64");
    return f;
}
PfnWaitValue64 wait_value64() {
    static PfnWaitValue64 f = driver_fn<PfnWaitValue64>("cuStreamWaitValue64");
    return f;
}
int wait_flags(int device) {   // GEQ, plus a flush of remote writes where the device supports it
    static int flags = -1;
    if (flags < 0) {
        flags = CU_STREAM_WAIT_VALUE_GEQ;
        PfnDevAttr attr = driver_fn<PfnDevAttr>("cuDeviceGetAttribute");
        int can = 0;
        if (attr && attr(&can, CU_DEVICE_ATTRIBUTE_CAN_FLUSH_REMOTE_WRITES, CUdevice(device)) == CUDA_SUCCESS && can)
            flags |= CU_STREAM_WAIT_VALUE_FLUSH;
    }
    return flags;
}

// ---- collectives ---------------------------------------------------------------
daso_status push_exchange(daso_ctx* c, cudaStream_t s);

// Non-blocking global exchange: after the packing kernel on the compute
// stream, the side stream runs the in-place group all-gather of the slot.
daso_status start_exchange(daso_ctx* c, cudaStream_t s) {
    if (c->vc) {   // virtual cluster: the driver issues the exchange after every rank's batch (see there)
        c->vc_sent = true;
        return DASO_OK;
    }
    return push_exchange(c, s);
}

// The send itself: after the pack on `s`, the group all-gather (NCCL) or the copy-engine pushes.
daso_status push_exchange(daso_ctx* c, cudaStream_t s) {
    CUDA_TRY(c, cudaEventRecord(c->ev_packed, s));
    CUDA_TRY(c, cudaStreamWaitEvent(c->side, c->ev_packed, 0));
    if (c->ce) {   // copy-engine pushes into every group member's slot (no SMs), one stream per member
        const unsigned long long e = ++c->exch_epoch;
        const size_t row = size_t(c->seg) * c->wire_bytes;
        Span sp(c, c->side, PH_EXCH, double(c->P - 1) * double(row));
        for (int k = 1; k < c->P; ++k) {
            const int i = (c->node + k) % c->P;             // start with the next member: spread the links
            cudaStream_t cs = c->ce_streams[size_t(k - 1)];
            CUDA_TRY(c, cudaStreamWaitEvent(cs, c->ev_packed, 0));
            if (c->exch_enabled) {
                // member i has consumed exchange e-1, so row `node` of its slot is free
                if (wait_value64()(cs, CUdeviceptr(c->xs + c->P + i), e - 1, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
                    return c->fail(DASO_ERR_CUDA, "cuStreamWaitValue64 (exchange flow control) failed");
                CUDA_TRY(c, cudaMemcpyAsync(static_cast<char*>(c->peer_slot[i]) + size_t(c->node) * row,
                                            own_segment(c), row, cudaMemcpyDeviceToDevice, cs));
            }   // else timing knob: flags only, no data
            if (write_value64()(cs, CUdeviceptr(c->peer_xs[i] + c->node), e, 0) != CUDA_SUCCESS)
                return c->fail(DASO_ERR_CUDA, "cuStreamWriteValue64 (exchange flag) failed");
            CUDA_TRY(c, cudaEventRecord(c->ce_done[size_t(k - 1)], cs));
            CUDA_TRY(c, cudaStreamWaitEvent(c->side, c->ce_done[size_t(k - 1)], 0));   // join
        }
    } else if (c->exch_enabled) {
        Span sp(c, c->side, PH_EXCH, double(c->P - 1) * double(c->seg) * double(c->wire_bytes));
        NCCL_TRY(c, ncclAllGather(own_segment(c), c->slot, size_t(c->seg), wire_nccl(c->cfg.wire), c->group_comm,
                                  c->side));
    }
    CUDA_TRY(c, cudaEventRecord(c->ev_exchanged, c->side));
    return DASO_OK;
}

// ---- kernel push (blocking syncs, copy-engine transport) ---------------------------------
// In a blocking batch (Fig. 3) the exchange is on the critical path.  With the CE transport's
// IPC mappings of the group members' slots in place, the update + pack kernel stores the packed row
// straight into row `node` of every member's slot over NVLink (one pass, no separate copy phase);
// the same flow control and arrival flags as the copy-engine pushes, issued on the compute stream:
// before the kernel, wait until every member has consumed exchange e-1 (its row `node` is free);
// after it, raise the arrival flag e in every member's xs (cuStreamWriteValue64 orders it after the
// kernel's stores).  Not in a batch that also merges: there this rank's acknowledgement of e-1
// follows the kernel, and the members wait for it before their own kernel pushes.
// Where: by default from the local pack kernel (G = 1, or the sharded mode), whose links are
// otherwise idle — 4x1 blocking batch 0.468 -> 0.332 ms.  Inside the fused node-tier kernel (G > 1)
// the push shares the links with the peer gradient reads; with a group of two it measured slower
// than the copy-engine push after the kernel (2x2: 0.309 vs 0.292 ms, profiles/r02/multi4_k), but
// the copy engines' all-to-all reaches only 0.57 of the link for groups of four (probe,
// profiles/r02/multi4_r) against 0.86 for SM bulk traffic, so for P >= 3 the node-tier kernel
// pushes too (4x2: ~194 vs ~255 us of link time by the probe rates; 8 GPUs, so not measured here).
// DASO_BLOCKING_PUSH: 0 never, 1 default (as above), 2 always (also P = 2 node-tier kernels).
int kernel_push_mode() {   // read per blocking batch, so a test can compare the transports
    const char* e = getenv("DASO_BLOCKING_PUSH");
    if (e && strcmp(e, "0") == 0) return 0;
    if (e && strcmp(e, "2") == 0) return 2;
    return 1;
}

bool kernel_push_ok(daso_ctx* c, bool merge) {
    const bool node_tier_kernel_p2 = c->cfg.mode == DASO_MODE_FUSED && c->G > 1 && c->P <= 2;
    return c->ce && c->exch_enabled && !merge && c->P > 1 && c->P - 1 <= daso::kMaxPush &&
           kernel_push_mode() >= (node_tier_kernel_p2 ? 2 : 1);
}

daso_status kernel_push_prepare(daso_ctx* c, daso::KernelArgs& a, cudaStream_t s) {
    const unsigned long long e = ++c->exch_epoch;
    const size_t row = size_t(c->seg) * c->wire_bytes;
    Span sp(c, s, PH_WAIT, 0.0);
    a.npush = 0;
    for (int k = 1; k < c->P; ++k) {
        const int i = (c->node + k) % c->P;
        if (wait_value64()(s, CUdeviceptr(c->xs + c->P + i), e - 1, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
            return c->fail(DASO_ERR_CUDA, "cuStreamWaitValue64 (exchange flow control) failed");
        a.push[a.npush++] = static_cast<char*>(c->peer_slot[i]) + size_t(c->node) * row;
    }
    return DASO_OK;
}

daso_status kernel_push_publish(daso_ctx* c, cudaStream_t s) {
    for (int k = 1; k < c->P; ++k) {
        const int i = (c->node + k) % c->P;
        if (write_value64()(s, CUdeviceptr(c->peer_xs[i] + c->node), c->exch_epoch, 0) != CUDA_SUCCESS)
            return c->fail(DASO_ERR_CUDA, "cuStreamWriteValue64 (exchange flag) failed");
    }
    CUDA_TRY(c, cudaEventRecord(c->ev_exchanged, s));   // wait_exchange's event wait: already in order
    return DASO_OK;
}

daso_status wait_exchange(daso_ctx* c, cudaStream_t s) {
    if (c->vc && !c->ce) return DASO_OK;   // virtual cluster, loopback: the copies precede on the same stream
    Span sp(c, s, PH_WAIT, 0.0);
    CUDA_TRY(c, cudaStreamWaitEvent(s, c->ev_exchanged, 0));   // own outgoing copies / all-gather done
    if (c->ce)   // every other member's row of this exchange has landed in the slot (flush once, at the last)
        for (int k = 1; k < c->P; ++k) {
            const int i = (c->node + k) % c->P;
            const unsigned flags = k == c->P - 1 ? wait_flags(c->device) : unsigned(CU_STREAM_WAIT_VALUE_GEQ);
            if (wait_value64()(s, CUdeviceptr(c->xs + i), c->exch_epoch, flags) != CUDA_SUCCESS)
                return c->fail(DASO_ERR_CUDA, "cuStreamWaitValue64 (exchange arrival) failed");
        }
    return DASO_OK;
}

// The slot rows of the current exchange have been read (merge / blocking average issued on s):
// tell every member its row in this rank's slot may be overwritten (copy-engine exchange only).
daso_status exchange_consumed(daso_ctx* c, cudaStream_t s) {
    if (!c->ce) return DASO_OK;
    for (int i = 0; i < c->P; ++i)
        if (i != c->node && write_value64()(s, CUdeviceptr(c->peer_xs[i] + c->P + c->node), c->exch_epoch, 0) != CUDA_SUCCESS)
            return c->fail(DASO_ERR_CUDA, "cuStreamWriteValue64 (exchange ack) failed");
    return DASO_OK;
}

// Fig. 4 local update: the group member's parameters replace the node's.
daso_status node_bcast(daso_ctx* c, int root, cudaStream_t s) {
    if (c->G == 1) return DASO_OK;
    Span sp(c, s, PH_NODE, 4.0 * double(c->n));
    NCCL_TRY(c, ncclBroadcast(c->x, c->x, size_t(c->n), ncclFloat32, root, c->node_comm, s));
    return DASO_OK;
}

// ---- blocking tails (Fig. 3 average + Fig. 4 re-publish, on the critical path) ------------
// Split out of the step functions so the virtual-cluster driver can run them after its
// loopback all-gather (daso_vcluster_step).
daso_status faithful_blocking_tail(daso_ctx* c, int group, cudaStream_t s) {
    if (c->local == group) {
        STATUS_TRY(wait_exchange(c, s));
        daso::KernelArgs av = base_args(c, 0, c->n, 0.f);
        av.den = float(c->P);
        KERN_TRY(c, launch(c, daso::OP_AVERAGE, av, s));
        STATUS_TRY(exchange_consumed(c, s));
    }
    return node_bcast(c, group, s);
}

daso_status shard_blocking_tail(daso_ctx* c, cudaStream_t s) {   // sharded / fused with G = 1
    const int64_t off = int64_t(c->local) * c->seg;
    STATUS_TRY(wait_exchange(c, s));
    daso::KernelArgs av = base_args(c, off, c->seg, 0.f);
    av.den = float(c->P);
    KERN_TRY(c, launch(c, daso::OP_AVERAGE, av, s));
    return exchange_consumed(c, s);
}

// Node-tier kernel arguments common to the fused batch and the fused blocking tail: peer
// pointer tables at this rank's shard, signal arrays, a fresh barrier epoch.
daso_status fused_peer_args(daso_ctx* c, daso::PeerArgs& pa, int64_t off, int64_t sh, float lr, cudaStream_t s) {
    pa.a = base_args(c, off, sh, lr);
    for (int q = 0; q < c->G; ++q) {
        pa.xp[q] = c->peer_x[q] + off;
        pa.gp[q] = c->peer_g[q] + off;
        pa.sig_peer[q] = c->peer_sig[q];
    }
    pa.sig_me = c->sig;
    pa.done = reinterpret_cast<unsigned*>(c->sig + 2 * c->G);
    pa.err = c->d_flag;
    pa.epoch = ++c->epoch;
    if (c->vc) {
        // Virtual cluster: the node's G kernels run one after another on one stream, so no
        // launch may wait for a later one (B200 guide: never launch kernels that wait on each
        // other on one GPU).  The first rank of the node pre-sets every start and end signal
        // of the node to this epoch, so every barrier wait is satisfied at its first poll;
        // the kernels' own signal stores write the same values.  Stream order provides what
        // the barriers provide across GPUs (all g complete before any read; all x stores
        // complete before the next batch), and shards are disjoint, so the sequential
        // execution computes exactly what G concurrent GPUs compute.
        if (c->local == 0) KERN_TRY(c, daso::launch_fill_u64(c->vc_node_sig, c->G, 2 * c->G + 2, 2 * c->G, pa.epoch, s));
        pa.timeout_ns = 1000ull * 1000 * 1000;
    }
    pa.G = c->G;
    pa.me = c->local;
    return DASO_OK;
}

// Fig. 3 average + Fig. 4 re-publish in one kernel (launch_avg_publish): the averaged shard goes
// straight into every node peer's x over NVLink, and the kernel's end barrier (which also
// covers the preceding OP_NOX node-tier kernel's gradient reads) orders it before any rank's
// next read of x.
daso_status fused_blocking_tail(daso_ctx* c, cudaStream_t s) {
    const int64_t sh = c->seg, off = int64_t(c->local) * sh;
    STATUS_TRY(wait_exchange(c, s));
    daso::PeerArgs pa;
    STATUS_TRY(fused_peer_args(c, pa, off, sh, 0.f, s));
    pa.a.den = float(c->P);
    {
        // HBM bytes on THIS GPU per shard element: P slot rows read, own x written, and the G-1
        // peers' stores into this GPU's x (symmetric); NVLink per direction (G-1) * 4.
        Span sp(c, s, PH_KERNEL, (double(c->P) * double(c->wire_bytes) + 4.0 * c->G) * double(sh),
                4.0 * (c->G - 1) * double(sh));
        KERN_TRY(c, daso::launch_avg_publish(c->cfg.wire, pa, s));
    }
    return exchange_consumed(c, s);
}

daso_status finish_blocking(daso_ctx* c, cudaStream_t s) {   // virtual cluster, after the loopback exchange
    c->vc_blocking = false;
    if (c->cfg.mode == DASO_MODE_FAITHFUL) return faithful_blocking_tail(c, c->vc_group, s);
    if (c->cfg.mode == DASO_MODE_FUSED && c->G > 1) return fused_blocking_tail(c, s);
    return shard_blocking_tail(c, s);
}

// ---- faithful (v1) batch ---------------------------------------------------------
daso_status step_faithful(daso_ctx* c, const daso_record& r, float lr, cudaStream_t s, bool reduced) {
    const bool global = c->P > 1;
    if (c->G > 1 && !reduced) {   // Fig. 2: node-local gradient sum (x 1/G in the kernel)
        Span sp(c, s, PH_LOCAL, 2.0 * (c->G - 1) / c->G * 4.0 * double(c->n));
        NCCL_TRY(c, ncclAllReduce(c->g, c->g, size_t(c->n), ncclFloat32, ncclSum, c->node_comm, s));
    }

    const bool merge = global && r.merge;
    const bool merge_here = merge && c->local == r.merge_group;
    const bool send = global && r.send;
    const bool send_here = send && c->local == r.send_group;
    // pack fuses into this batch's kernel unless a broadcast from another GPU
    // replaces x in between (R11)
    const bool fuse_pack = send_here && (!merge || r.merge_group == r.send_group);

    daso::KernelArgs a = base_args(c, 0, c->n, lr);
    int ops = daso::OP_UPDATE;
    if (merge_here) {
        STATUS_TRY(wait_exchange(c, s));
        ops |= daso::OP_MERGE;
        a.den = float(2 * r.merge_S + c->P);     // Eq. (1) denominator 2S + P
    }
    if (fuse_pack) {
        ops |= daso::OP_PACK;
        a.pack_out = own_segment(c);
    }
    KERN_TRY(c, launch(c, ops, a, s));
    if (merge_here) STATUS_TRY(exchange_consumed(c, s));
    if (merge) {
        STATUS_TRY(node_bcast(c, int(r.merge_group), s));
        c->inflight = false;
    }
    if (send_here && !fuse_pack) {
        daso::KernelArgs p = base_args(c, 0, c->n, 0.f);
        p.pack_out = own_segment(c);
        p.flag = nullptr;
        KERN_TRY(c, launch(c, daso::OP_PACK, p, s));
    }
    if (send) {
        if (send_here) STATUS_TRY(start_exchange(c, s));
        if (r.blocking) {   // Fig. 3 average + Fig. 4 broadcast on the critical path
            if (c->vc) {
                c->vc_blocking = true;
                c->vc_group = int(r.send_group);
                return DASO_OK;
            }
            STATUS_TRY(faithful_blocking_tail(c, int(r.send_group), s));
        } else {
            c->inflight = true;
            c->infl_group = int(r.send_group);
            c->infl_S = int(r.S);
        }
    }
    return DASO_OK;
}

// ---- sharded (v2) batch ----------------------------------------------------------
// Node replicas are bitwise identical between syncs, so the update, the Eq. (1)
// merge and the exchange are element-sharded over the node's G GPUs: reduce-scatter
// of g, shard kernel, every group exchanges its own shard, all-gather of x.
daso_status step_sharded(daso_ctx* c, const daso_record& r, float lr, cudaStream_t s) {
    const bool global = c->P > 1;
    const int64_t sh = c->seg;
    const int64_t off = int64_t(c->local) * sh;
    if (c->G > 1) {
        Span sp(c, s, PH_LOCAL, double(c->G - 1) / c->G * 4.0 * double(c->n_pad));
        NCCL_TRY(c, ncclReduceScatter(c->g, c->g + off, size_t(sh), ncclFloat32, ncclSum, c->node_comm, s));
    }
    const bool merge = global && r.merge;
    const bool send = global && r.send;
    daso::KernelArgs a = base_args(c, off, sh, lr);
    int ops = daso::OP_UPDATE;
    if (merge) {
        STATUS_TRY(wait_exchange(c, s));
        ops |= daso::OP_MERGE;
        a.den = float(2 * r.merge_S + c->P);
        c->inflight = false;
    }
    bool kpush = false;
    if (send) {
        ops |= daso::OP_PACK;
        a.pack_out = own_segment(c);
        if (r.blocking && kernel_push_ok(c, merge)) {
            STATUS_TRY(kernel_push_prepare(c, a, s));
            ops |= daso::OP_PUSH;
            kpush = true;
        }
    }
    KERN_TRY(c, launch(c, ops, a, s));
    if (merge) STATUS_TRY(exchange_consumed(c, s));
    if (send) {
        STATUS_TRY(kpush ? kernel_push_publish(c, s) : start_exchange(c, s));
        if (r.blocking) {
            if (c->vc) {   // G == 1 in a virtual cluster: nothing follows the tail
                c->vc_blocking = true;
                return DASO_OK;
            }
            STATUS_TRY(shard_blocking_tail(c, s));
        } else {
            c->inflight = true;
            c->infl_group = int(r.send_group);
            c->infl_S = int(r.S);
        }
    }
    if (c->G > 1) {
        Span sp(c, s, PH_NODE, double(c->G - 1) / c->G * 4.0 * double(c->n_pad));
        NCCL_TRY(c, ncclAllGather(c->x + off, c->x, size_t(sh), ncclFloat32, c->node_comm, s));
    }
    return DASO_OK;
}

// ---- fused (v3) batch: the sharded batch with the node tier inside one kernel ----------
daso_status step_fused(daso_ctx* c, const daso_record& r, float lr, cudaStream_t s) {
    if (c->G == 1) return step_sharded(c, r, lr, s);   // no node tier
    const bool global = c->P > 1;
    const int64_t sh = c->seg;
    const int64_t off = int64_t(c->local) * sh;
    const bool merge = global && r.merge;
    const bool send = global && r.send;
    daso::PeerArgs pa;
    STATUS_TRY(fused_peer_args(c, pa, off, sh, lr, s));
    int ops = daso::OP_UPDATE;
    if (merge) {
        STATUS_TRY(wait_exchange(c, s));
        ops |= daso::OP_MERGE;
        pa.a.den = float(2 * r.merge_S + c->P);
        c->inflight = false;
    }
    if (send) {
        ops |= daso::OP_PACK;
        pa.a.pack_out = own_segment(c);
        // blocking batch: the average of the tail replaces x, so the node-tier kernel only
        // packs (no x stores to the peers, no end barrier: the tail's end barrier covers it)
        if (r.blocking) ops |= daso::OP_NOX;
    }
    const bool kpush = send && r.blocking && kernel_push_ok(c, merge);
    if (kpush) {
        STATUS_TRY(kernel_push_prepare(c, pa.a, s));
        ops |= daso::OP_PUSH;
    }
    {
        // HBM bytes on THIS GPU per shard element: own x r + w, v r + w, own g r
        // (20) + the G-1 peers reading this GPU's g and writing its x (8 (G-1)) + slot rows / pack.
        // NVLink per direction: (G-1) * 4 B per shard element (bench.py reports it separately).
        const double wb = double(c->wire_bytes);
        double per = ((ops & daso::OP_NOX) ? 16.0 + 4.0 * (c->G - 1) : 20.0 + 8.0 * (c->G - 1)) +
                     ((ops & daso::OP_MERGE) ? c->P * wb : 0) + ((ops & daso::OP_PACK) ? wb : 0);
        const double nvl = ((ops & daso::OP_NOX) ? 1.0 : 2.0) * 4.0 * (c->G - 1) * double(sh) +
                           double(pa.a.npush) * wb * double(sh);
        Span sp(c, s, PH_KERNEL, per * double(sh), nvl);
        KERN_TRY(c, daso::launch_peer(ops, c->cfg.wire, pa, s));
    }
    if (merge) STATUS_TRY(exchange_consumed(c, s));
    if (send) {
        STATUS_TRY(kpush ? kernel_push_publish(c, s) : start_exchange(c, s));
        if (r.blocking) {
            if (c->vc) {
                c->vc_blocking = true;
                return DASO_OK;
            }
            STATUS_TRY(fused_blocking_tail(c, s));
        } else {
            c->inflight = true;
            c->infl_group = int(r.send_group);
            c->infl_S = int(r.S);
        }
    }
    return DASO_OK;
}

typedef CUresult (*PfnAddressRange)(CUdeviceptr*, size_t*, CUdeviceptr);

PfnAddressRange address_range_fn() {
    static PfnAddressRange fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PfnAddressRange>(p);
    }
    return fn;
}

// Exchange CUDA IPC handles of x, g and the signal array over the node communicator and
// map every node peer's buffers into this process (peer access over NVLink).
struct IpcExport {
    cudaIpcMemHandle_t h[3];
    uint64_t base[3];
    uint64_t off[3];
};

daso_status setup_peers(daso_ctx* c) {
    PfnAddressRange range = address_range_fn();
    if (!range) return c->fail(DASO_ERR_CUDA, "cuMemGetAddressRange unavailable");
    const size_t sig_bytes = (2 * size_t(c->G) + 2) * sizeof(unsigned long long);
    CUDA_TRY(c, cudaMalloc(&c->sig, sig_bytes));
    CUDA_TRY(c, cudaMemset(c->sig, 0, sig_bytes));
    void* bufs[3] = {c->x, c->g, c->sig};
    IpcExport mine{};
    for (int b = 0; b < 3; ++b) {
        CUdeviceptr base = 0;
        size_t size = 0;
        if (range(&base, &size, CUdeviceptr(bufs[b])) != CUDA_SUCCESS)
            return c->fail(DASO_ERR_ARGUMENT, "buffer %d is not a device allocation", b);
        const cudaError_t e = cudaIpcGetMemHandle(&mine.h[b], reinterpret_cast<void*>(base));
        if (e != cudaSuccess)
            return c->fail(DASO_ERR_ARGUMENT,
                           "buffer %d cannot be exported by CUDA IPC (%s): the fused mode needs cudaMalloc-backed "
                           "buckets (not cuMem / expandable_segments memory); use daso_alloc_bind",
                           b, cudaGetErrorString(e));
        mine.base[b] = uint64_t(base);
        mine.off[b] = uint64_t(CUdeviceptr(bufs[b]) - base);
    }
    std::vector<IpcExport> all(c->G);
    void* dbuf = nullptr;
    CUDA_TRY(c, cudaMalloc(&dbuf, sizeof(IpcExport) * c->G));
    CUDA_TRY(c, cudaMemcpy(static_cast<char*>(dbuf) + sizeof(IpcExport) * c->local, &mine, sizeof mine,
                           cudaMemcpyHostToDevice));
    NCCL_TRY(c, ncclAllGather(static_cast<char*>(dbuf) + sizeof(IpcExport) * c->local, dbuf, sizeof(IpcExport),
                              ncclUint8, c->node_comm, c->side));
    CUDA_TRY(c, cudaStreamSynchronize(c->side));
    CUDA_TRY(c, cudaMemcpy(all.data(), dbuf, sizeof(IpcExport) * c->G, cudaMemcpyDeviceToHost));
    cudaFree(dbuf);
    for (int q = 0; q < c->G; ++q) {
        void* mapped[3] = {nullptr, nullptr, nullptr};
        if (q == c->local) {
            for (int b = 0; b < 3; ++b) mapped[b] = reinterpret_cast<char*>(bufs[b]) - all[q].off[b];
        } else {
            for (int b = 0; b < 3; ++b) {
                for (int e = 0; e < b; ++e)   // one mapping per distinct allocation of the peer
                    if (all[q].base[e] == all[q].base[b]) mapped[b] = mapped[e];
                if (!mapped[b]) {
                    CUDA_TRY(c, cudaIpcOpenMemHandle(&mapped[b], all[q].h[b], cudaIpcMemLazyEnablePeerAccess));
                    c->ipc_opened.push_back(mapped[b]);
                }
            }
        }
        c->peer_x[q] = reinterpret_cast<float*>(static_cast<char*>(mapped[0]) + all[q].off[0]);
        c->peer_g[q] = reinterpret_cast<float*>(static_cast<char*>(mapped[1]) + all[q].off[1]);
        c->peer_sig[q] = reinterpret_cast<unsigned long long*>(static_cast<char*>(mapped[2]) + all[q].off[2]);
    }
    return DASO_OK;
}

// Copy-engine group exchange: map every group member's slot and flag array (CUDA IPC handles
// exchanged over the group communicator at bind time).
struct GroupExport {
    cudaIpcMemHandle_t slot, xs;
};

daso_status setup_group_ce(daso_ctx* c) {
    PfnDevAttr attr = driver_fn<PfnDevAttr>("cuDeviceGetAttribute");
    int can = 0;
    if (!write_value64() || !wait_value64() || !attr ||
        attr(&can, CU_DEVICE_ATTRIBUTE_CAN_USE_64_BIT_STREAM_MEM_OPS, CUdevice(c->device)) != CUDA_SUCCESS || !can)
        return c->fail(DASO_ERR_CONFIG, "DASO_EXCH_CE needs 64-bit stream memory operations (cuStreamWaitValue64)");
    const size_t xs_bytes = (2 * size_t(c->P) + 1) * sizeof(unsigned long long);   // + barrier scratch
    CUDA_TRY(c, cudaMalloc(&c->xs, xs_bytes));
    CUDA_TRY(c, cudaMemset(c->xs, 0, xs_bytes));
    GroupExport mine{};
    CUDA_TRY(c, cudaIpcGetMemHandle(&mine.slot, c->slot));
    CUDA_TRY(c, cudaIpcGetMemHandle(&mine.xs, c->xs));
    std::vector<GroupExport> all(c->P);
    void* dbuf = nullptr;
    CUDA_TRY(c, cudaMalloc(&dbuf, sizeof(GroupExport) * c->P));
    CUDA_TRY(c, cudaMemcpy(static_cast<char*>(dbuf) + sizeof(GroupExport) * c->node, &mine, sizeof mine,
                           cudaMemcpyHostToDevice));
    NCCL_TRY(c, ncclAllGather(static_cast<char*>(dbuf) + sizeof(GroupExport) * c->node, dbuf, sizeof(GroupExport),
                              ncclUint8, c->group_comm, c->side));
    CUDA_TRY(c, cudaStreamSynchronize(c->side));
    CUDA_TRY(c, cudaMemcpy(all.data(), dbuf, sizeof(GroupExport) * c->P, cudaMemcpyDeviceToHost));
    cudaFree(dbuf);
    c->peer_slot.assign(size_t(c->P), nullptr);
    c->peer_xs.assign(size_t(c->P), nullptr);
    for (int i = 0; i < c->P; ++i) {
        if (i == c->node) {
            c->peer_slot[i] = c->slot;
            c->peer_xs[i] = c->xs;
            continue;
        }
        void* ms = nullptr;
        void* mx = nullptr;
        CUDA_TRY(c, cudaIpcOpenMemHandle(&ms, all[i].slot, cudaIpcMemLazyEnablePeerAccess));
        c->ipc_group.push_back(ms);
        CUDA_TRY(c, cudaIpcOpenMemHandle(&mx, all[i].xs, cudaIpcMemLazyEnablePeerAccess));
        c->ipc_group.push_back(mx);
        c->peer_slot[i] = ms;
        c->peer_xs[i] = static_cast<unsigned long long*>(mx);
    }
    int lo = 0, hi = 0;
    CUDA_TRY(c, cudaDeviceGetStreamPriorityRange(&lo, &hi));
    for (int k = 1; k < c->P; ++k) {
        cudaStream_t st = nullptr;
        cudaEvent_t ev = nullptr;
        CUDA_TRY(c, cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking, hi));
        c->ce_streams.push_back(st);
        CUDA_TRY(c, cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        c->ce_done.push_back(ev);
    }
    c->ce = true;
    return DASO_OK;
}

}  // namespace

extern "C" {

const char* daso_status_string(daso_status s) {
    switch (s) {
        case DASO_OK: return "ok";
        case DASO_ERR_CONFIG: return "config error";
        case DASO_ERR_RANGE: return "range error";
        case DASO_ERR_PROTOCOL: return "protocol error";
        case DASO_ERR_ARGUMENT: return "argument error";
        case DASO_ERR_CUDA: return "CUDA error";
        case DASO_ERR_NCCL: return "NCCL error";
        case DASO_ERR_NONFINITE: return "non-finite parameters";
    }
    return "unknown status";
}

const char* daso_version(void) { return "daso-b200 0.1 (sm_100a)"; }

size_t daso_padded_numel(size_t n, int gpus_per_node) {
    const size_t q = 64 * size_t(gpus_per_node < 1 ? 1 : gpus_per_node);
    return (n + q - 1) / q * q;
}

daso_status daso_get_unique_id(void* out128) {
    if (!out128) return DASO_ERR_ARGUMENT;
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId must be 128 bytes");
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return DASO_ERR_NCCL;
    std::memcpy(out128, &id, sizeof id);
    return DASO_OK;
}

}  // extern "C"

namespace {

// Validate the configuration and create a ctx with its streams, events and flag word, but
// no communicators (daso_init adds them; a virtual cluster's ranks have none).
daso_status make_ctx(daso_ctx** out, int world, int gpus_per_node, int B, int S, const daso_config* cfg) {
    *out = nullptr;
    if (world < 1 || gpus_per_node < 1 || world % gpus_per_node != 0 || B < 1) return DASO_ERR_CONFIG;
    if (cfg->rank < 0 || cfg->rank >= world) return DASO_ERR_RANGE;
    if (cfg->wire != DASO_WIRE_BF16 && cfg->wire != DASO_WIRE_FP32) return DASO_ERR_ARGUMENT;
    if (cfg->exchange != DASO_EXCH_NCCL && cfg->exchange != DASO_EXCH_CE) return DASO_ERR_ARGUMENT;
    if (cfg->mode != DASO_MODE_FAITHFUL && cfg->mode != DASO_MODE_SHARDED && cfg->mode != DASO_MODE_FUSED)
        return DASO_ERR_ARGUMENT;
    if (cfg->mode == DASO_MODE_FUSED && gpus_per_node > daso::kMaxPeers)
        return DASO_ERR_CONFIG;
    daso_sched_config sc{};
    sc.B_init = B;
    sc.S_init = S;
    sc.warmup_epochs = cfg->warmup_epochs;
    sc.cooldown_epochs = cfg->cooldown_epochs;
    sc.total_epochs = cfg->total_epochs;
    sc.steps_per_epoch = cfg->steps_per_epoch;
    sc.gpus_per_node = gpus_per_node;
    if (daso::validate_sched(sc)) return DASO_ERR_CONFIG;

    daso_ctx* c = new (std::nothrow) daso_ctx;
    if (!c) return DASO_ERR_ARGUMENT;
    c->world = world;
    c->G = gpus_per_node;
    c->P = world / gpus_per_node;
    c->rank = cfg->rank;
    c->node = cfg->rank / gpus_per_node;
    c->local = cfg->rank % gpus_per_node;
    c->cfg = *cfg;
    c->scfg = sc;
    c->sched = new daso::Schedule(sc);
    c->wire_bytes = cfg->wire == DASO_WIRE_BF16 ? 2 : 4;
    *out = c;   // returned even on failure so daso_last_error can be read

    CUDA_TRY(c, cudaGetDevice(&c->device));
    int lo = 0, hi = 0;
    CUDA_TRY(c, cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CUDA_TRY(c, cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, hi));
    CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_packed, cudaEventDisableTiming));
    CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_exchanged, cudaEventDisableTiming));
    CUDA_TRY(c, cudaMalloc(&c->d_flag, sizeof(uint32_t)));
    CUDA_TRY(c, cudaMemset(c->d_flag, 0, sizeof(uint32_t)));
    return DASO_OK;
}

}  // namespace

extern "C" {

daso_status daso_init(daso_ctx** out, int world, int gpus_per_node, int B, int S, const daso_config* cfg,
                      const void* uid) {
    if (!out || !cfg || !uid) return DASO_ERR_ARGUMENT;
    STATUS_TRY(make_ctx(out, world, gpus_per_node, B, S, cfg));
    daso_ctx* c = *out;
    ncclUniqueId id;
    std::memcpy(&id, uid, sizeof id);
    ncclConfig_t wc = NCCL_CONFIG_INITIALIZER;
    wc.blocking = 1;
    NCCL_TRY(c, ncclCommInitRankConfig(&c->world_comm, world, id, c->rank, &wc));
    ncclConfig_t nc = NCCL_CONFIG_INITIALIZER;
    nc.blocking = 1;
    NCCL_TRY(c, ncclCommSplit(c->world_comm, c->node, c->local, &c->node_comm, &nc));
    ncclConfig_t gc = NCCL_CONFIG_INITIALIZER;
    gc.blocking = 1;
    if (cfg->nccl_max_ctas > 0) {
        gc.maxCTAs = cfg->nccl_max_ctas;
        gc.minCTAs = 1;
    }
    NCCL_TRY(c, ncclCommSplit(c->world_comm, c->local, c->node, &c->group_comm, &gc));
    ncclConfig_t bc = NCCL_CONFIG_INITIALIZER;
    bc.blocking = 1;
    NCCL_TRY(c, ncclCommSplit(c->world_comm, c->node, c->local, &c->bucket_comm, &bc));
    return DASO_OK;
}

daso_status bind_impl(daso_ctx* c, float* x, float* g, float* v, size_t n);

daso_status daso_bind(daso_ctx* c, float* x, float* g, float* v, size_t n) {
    if (!c) return DASO_ERR_ARGUMENT;
    return bind_impl(c, x, g, v, n);
}

daso_status daso_alloc_bind(daso_ctx* c, size_t n, float** x, float** g, float** v) {
    if (!c || !x || !g || !v || n == 0) return DASO_ERR_ARGUMENT;
    if (c->bound) return c->fail(DASO_ERR_PROTOCOL, "daso_bind called twice");
    const size_t n_pad = daso_padded_numel(n, c->G);
    const size_t bytes = (n_pad * sizeof(float) + (size_t(2) << 20) - 1) / (size_t(2) << 20) * (size_t(2) << 20);
    void* p[3] = {nullptr, nullptr, nullptr};
    for (int b = 0; b < 3; ++b) {   // cudaMalloc: what the fused mode's CUDA IPC export needs
        CUDA_TRY(c, cudaMalloc(&p[b], bytes));
        c->own_cuda[b] = p[b];
        CUDA_TRY(c, cudaMemset(p[b], 0, bytes));
    }
    c->x = static_cast<float*>(p[0]);
    c->g = static_cast<float*>(p[1]);
    c->v = static_cast<float*>(p[2]);
    STATUS_TRY(bind_impl(c, c->x, c->g, c->v, n));
    *x = c->x;
    *g = c->g;
    *v = c->v;
    return DASO_OK;
}

daso_status bind_impl(daso_ctx* c, float* x, float* g, float* v, size_t n) {
    if (c->bound) return c->fail(DASO_ERR_PROTOCOL, "daso_bind called twice");
    if (!x || !g || !v || n == 0) return c->fail(DASO_ERR_ARGUMENT, "null buffer or n == 0");
    if (((uintptr_t(x) | uintptr_t(g) | uintptr_t(v)) & 15u) != 0)
        return c->fail(DASO_ERR_ARGUMENT, "x, g, v must be 16-byte aligned");
    const int64_t q = 64 * int64_t(c->G);
    c->x = x;
    c->g = g;
    c->v = v;
    c->n = int64_t(n);
    c->n_pad = (int64_t(n) + q - 1) / q * q;
    c->seg = c->cfg.mode == DASO_MODE_FAITHFUL ? c->n_pad : c->n_pad / c->G;
    if (c->P > 1) {
        const size_t bytes = size_t(c->P) * size_t(c->seg) * c->wire_bytes;
        CUDA_TRY(c, cudaMalloc(&c->slot, bytes));
        CUDA_TRY(c, cudaMemset(c->slot, 0, bytes));
    }
    if (c->cfg.mode == DASO_MODE_FUSED && c->G > 1 && !c->vc) STATUS_TRY(setup_peers(c));
    if (c->cfg.exchange == DASO_EXCH_CE && c->P > 1 && !c->vc) STATUS_TRY(setup_group_ce(c));
    CUDA_TRY(c, cudaDeviceSynchronize());
    c->bound = true;
    return DASO_OK;
}

daso_status daso_local_sync(daso_ctx* c, void* stream) {
    if (!c) return DASO_ERR_ARGUMENT;
    STATUS_TRY(require_bound(c));
    if (c->cfg.mode != DASO_MODE_FAITHFUL) return c->fail(DASO_ERR_PROTOCOL, "split API requires DASO_MODE_FAITHFUL");
    if (c->G > 1) {
        Span sp(c, static_cast<cudaStream_t>(stream), PH_LOCAL, 2.0 * (c->G - 1) / c->G * 4.0 * double(c->n));
        NCCL_TRY(c, ncclAllReduce(c->g, c->g, size_t(c->n), ncclFloat32, ncclSum, c->node_comm,
                                  static_cast<cudaStream_t>(stream)));
    }
    return DASO_OK;
}

daso_status daso_local_update(daso_ctx* c, float lr, void* stream) {
    if (!c) return DASO_ERR_ARGUMENT;
    STATUS_TRY(require_bound(c));
    if (c->cfg.mode != DASO_MODE_FAITHFUL) return c->fail(DASO_ERR_PROTOCOL, "split API requires DASO_MODE_FAITHFUL");
    KERN_TRY(c, launch(c, daso::OP_UPDATE, base_args(c, 0, c->n, lr), static_cast<cudaStream_t>(stream)));
    return DASO_OK;
}

daso_status daso_global_send(daso_ctx* c, int group, int S, void* stream) {
    if (!c) return DASO_ERR_ARGUMENT;
    STATUS_TRY(require_bound(c));
    if (c->cfg.mode != DASO_MODE_FAITHFUL) return c->fail(DASO_ERR_PROTOCOL, "split API requires DASO_MODE_FAITHFUL");
    if (c->inflight) return c->fail(DASO_ERR_PROTOCOL, "an exchange is already in flight");
    if (group < 0 || group >= c->G) return c->fail(DASO_ERR_RANGE, "group %d outside [0, %d)", group, c->G);
    if (S < 0) return c->fail(DASO_ERR_ARGUMENT, "S must be >= 0");
    if (c->P == 1) return DASO_OK;   // global tier disabled (R12)
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const bool member = c->local == group;
    if (member) {
        daso::KernelArgs p = base_args(c, 0, c->n, 0.f);
        p.pack_out = own_segment(c);
        p.flag = nullptr;
        KERN_TRY(c, launch(c, daso::OP_PACK, p, s));
        STATUS_TRY(start_exchange(c, s));
    }
    if (S == 0) {
        if (member) {
            STATUS_TRY(wait_exchange(c, s));
            daso::KernelArgs av = base_args(c, 0, c->n, 0.f);
            av.den = float(c->P);
            KERN_TRY(c, launch(c, daso::OP_AVERAGE, av, s));
            STATUS_TRY(exchange_consumed(c, s));
        }
        STATUS_TRY(node_bcast(c, group, s));
    } else {
        c->inflight = true;
        c->infl_group = group;
        c->infl_S = S;
    }
    return DASO_OK;
}

daso_status daso_global_merge(daso_ctx* c, void* stream) {
    if (!c) return DASO_ERR_ARGUMENT;
    STATUS_TRY(require_bound(c));
    if (c->cfg.mode != DASO_MODE_FAITHFUL) return c->fail(DASO_ERR_PROTOCOL, "split API requires DASO_MODE_FAITHFUL");
    if (!c->inflight) return c->fail(DASO_ERR_PROTOCOL, "no exchange in flight to merge");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (c->local == c->infl_group) {
        STATUS_TRY(wait_exchange(c, s));
        daso::KernelArgs m = base_args(c, 0, c->n, 0.f);
        m.den = float(2 * c->infl_S + c->P);
        KERN_TRY(c, launch(c, daso::OP_MERGE, m, s));
        STATUS_TRY(exchange_consumed(c, s));
    }
    STATUS_TRY(node_bcast(c, c->infl_group, s));
    c->inflight = false;
    return DASO_OK;
}

daso_status daso_local_sync_bucket(daso_ctx* c, size_t offset, size_t count, void* stream) {
    if (!c) return DASO_ERR_ARGUMENT;
    STATUS_TRY(require_bound(c));
    if (c->cfg.mode != DASO_MODE_FAITHFUL)
        return c->fail(DASO_ERR_PROTOCOL, "bucketed local sync requires DASO_MODE_FAITHFUL");
    if (offset > size_t(c->n) || count > size_t(c->n) - offset)
        return c->fail(DASO_ERR_RANGE, "bucket [%zu, %zu) outside [0, %lld)", offset, offset + count, (long long)c->n);
    if (c->G == 1 || count == 0) return DASO_OK;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    Span sp(c, s, PH_LOCAL, 2.0 * (c->G - 1) / c->G * 4.0 * double(count));
    NCCL_TRY(c, ncclAllReduce(c->g + offset, c->g + offset, count, ncclFloat32, ncclSum, c->bucket_comm, s));
    return DASO_OK;
}

daso_status daso_step_ex(daso_ctx* c, float lr, int plateau, int flags, void* stream, daso_record* out) {
    if (!c) return DASO_ERR_ARGUMENT;
    STATUS_TRY(require_bound(c));
    const bool reduced = (flags & DASO_STEP_GRADS_REDUCED) != 0;
    if (reduced && c->cfg.mode != DASO_MODE_FAITHFUL)
        return c->fail(DASO_ERR_PROTOCOL, "DASO_STEP_GRADS_REDUCED requires DASO_MODE_FAITHFUL");
    const daso_record r = c->sched->next(plateau);
    c->last = r;
    if (c->tracing) c->acc.steps += 1;
    if (out) *out = r;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (r.merge && c->P > 1 && !c->inflight)
        return c->fail(DASO_ERR_PROTOCOL, "schedule merge at step %lld but nothing in flight", (long long)r.step);
    if (c->cfg.mode == DASO_MODE_SHARDED) return step_sharded(c, r, lr, s);
    if (c->cfg.mode == DASO_MODE_FUSED) return step_fused(c, r, lr, s);
    return step_faithful(c, r, lr, s, reduced);
}

daso_status daso_step(daso_ctx* c, float lr, int plateau, void* stream, daso_record* out) {
    return daso_step_ex(c, lr, plateau, 0, stream, out);
}

daso_status daso_step_host(daso_ctx* c, const float* host_grads, float lr, int plateau, void* stream,
                           daso_record* out, uint32_t* host_flag) {
    if (!c || !host_grads) return DASO_ERR_ARGUMENT;
    STATUS_TRY(require_bound(c));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    CUDA_TRY(c, cudaMemcpyAsync(c->g, host_grads, size_t(c->n) * sizeof(float), cudaMemcpyHostToDevice, s));
    STATUS_TRY(daso_step(c, lr, plateau, stream, out));
    if (host_flag) {
        CUDA_TRY(c, cudaMemcpyAsync(host_flag, c->d_flag, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
        CUDA_TRY(c, cudaMemsetAsync(c->d_flag, 0, sizeof(uint32_t), s));
    }
    CUDA_TRY(c, cudaStreamSynchronize(s));
    return DASO_OK;
}

daso_status daso_trace_enable(daso_ctx* c, int on) {
    if (!c) return DASO_ERR_ARGUMENT;
    c->tracing = on != 0;
    return DASO_OK;
}

daso_status daso_trace_read(daso_ctx* c, daso_trace* out, int reset) {
    if (!c || !out) return DASO_ERR_ARGUMENT;
    CUDA_TRY(c, cudaDeviceSynchronize());
    for (const auto& sp : c->spans) {
        float ms = 0.f;
        CUDA_TRY(c, cudaEventElapsedTime(&ms, sp.a, sp.b));
        switch (sp.phase) {
            case PH_KERNEL:
                c->acc.kernel_launches++; c->acc.kernel_ms += ms; c->acc.kernel_bytes += sp.bytes;
                c->acc.kernel_nvl_bytes += sp.nvl;
                break;
            case PH_LOCAL: c->acc.local_ops++; c->acc.local_ms += ms; c->acc.local_bytes += sp.bytes; break;
            case PH_NODE: c->acc.node_ops++; c->acc.node_ms += ms; c->acc.node_bytes += sp.bytes; break;
            case PH_WAIT: c->acc.wait_ops++; c->acc.wait_ms += ms; break;
            case PH_EXCH: c->acc.exch_ops++; c->acc.exch_ms += ms; c->acc.exch_bytes += sp.bytes; break;
        }
    }
    c->spans.clear();
    c->pool_used = 0;
    *out = c->acc;
    if (reset) c->acc = daso_trace{};
    return DASO_OK;
}

daso_status daso_query(const daso_ctx* c, daso_record* last) {
    if (!c || !last) return DASO_ERR_ARGUMENT;
    *last = c->last;
    return DASO_OK;
}

daso_status daso_check_finite(daso_ctx* c, void* stream) {
    if (!c) return DASO_ERR_ARGUMENT;
    if (!c->d_flag) return c->fail(DASO_ERR_PROTOCOL, "not initialised");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    uint32_t h = 0;
    CUDA_TRY(c, cudaMemcpyAsync(&h, c->d_flag, sizeof h, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(c, cudaMemsetAsync(c->d_flag, 0, sizeof(uint32_t), s));
    CUDA_TRY(c, cudaStreamSynchronize(s));
    if (h & 2u) return c->fail(DASO_ERR_PROTOCOL, "node barrier timed out in the fused kernel (a peer never arrived)");
    if (h & 4u) return c->fail(DASO_ERR_CUDA, "a TMA bulk-copy wait timed out (transfer never completed)");
    if (h & 1u) return c->fail(DASO_ERR_NONFINITE, "non-finite parameter written");
    return DASO_OK;
}

daso_status daso_topology(const daso_ctx* c, int* P, int* G, int* node, int* local) {
    if (!c) return DASO_ERR_ARGUMENT;
    if (P) *P = c->P;
    if (G) *G = c->G;
    if (node) *node = c->node;
    if (local) *local = c->local;
    return DASO_OK;
}

int daso_set_exchange(daso_ctx* c, int enabled) {
    if (!c) return -1;
    const int prev = c->exch_enabled ? 1 : 0;
    if (enabled == 0 || enabled == 1) c->exch_enabled = enabled == 1;
    return prev;
}

daso_status daso_exchange_alone(daso_ctx* c, int iters, double* ms_out) {
    if (!c || !ms_out || iters < 1) return DASO_ERR_ARGUMENT;
    STATUS_TRY(require_bound(c));
    if (c->vc) return c->fail(DASO_ERR_PROTOCOL, "no group communicator in a virtual cluster");
    if (c->P == 1) {
        *ms_out = 0.0;
        return DASO_OK;
    }
    if (c->inflight) return c->fail(DASO_ERR_PROTOCOL, "an exchange is in flight");
    CUDA_TRY(c, cudaDeviceSynchronize());
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    CUDA_TRY(c, cudaEventCreate(&e0));
    CUDA_TRY(c, cudaEventCreate(&e1));
    const size_t row = size_t(c->seg) * c->wire_bytes;
    auto one = [&]() -> daso_status {
        if (!c->ce) {
            NCCL_TRY(c, ncclAllGather(own_segment(c), c->slot, size_t(c->seg), wire_nccl(c->cfg.wire), c->group_comm,
                                      c->side));
            return DASO_OK;
        }
        CUDA_TRY(c, cudaEventRecord(c->ev_packed, c->side));
        for (int k = 1; k < c->P; ++k) {   // the copy-engine pushes of one exchange (parallel streams), no flags
            const int i = (c->node + k) % c->P;
            cudaStream_t cs = c->ce_streams[size_t(k - 1)];
            CUDA_TRY(c, cudaStreamWaitEvent(cs, c->ev_packed, 0));
            CUDA_TRY(c, cudaMemcpyAsync(static_cast<char*>(c->peer_slot[i]) + size_t(c->node) * row, own_segment(c),
                                        row, cudaMemcpyDeviceToDevice, cs));
            CUDA_TRY(c, cudaEventRecord(c->ce_done[size_t(k - 1)], cs));
            CUDA_TRY(c, cudaStreamWaitEvent(c->side, c->ce_done[size_t(k - 1)], 0));
        }
        return DASO_OK;
    };
    if (c->ce) {   // align the members: nobody starts pushing before everybody is idle
        unsigned long long* scratch = c->xs + 2 * c->P;
        NCCL_TRY(c, ncclAllReduce(scratch, scratch, 1, ncclUint64, ncclSum, c->group_comm, c->side));
    }
    STATUS_TRY(one());
    CUDA_TRY(c, cudaEventRecord(e0, c->side));
    for (int i = 0; i < iters; ++i) STATUS_TRY(one());
    CUDA_TRY(c, cudaEventRecord(e1, c->side));
    CUDA_TRY(c, cudaEventSynchronize(e1));
    float ms = 0.f;
    CUDA_TRY(c, cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *ms_out = double(ms) / iters;
    return DASO_OK;
}

daso_status daso_finalize(daso_ctx* c) {
    if (!c) return DASO_OK;
    daso_status st = DASO_OK;
    if (c->side) cudaStreamSynchronize(c->side);   // drain an in-flight exchange
    cudaDeviceSynchronize();
    if (!c->ipc_opened.empty() || c->sig) {
        // no node peer may still touch this rank's memory: node barrier before unmapping
        if (c->node_comm && c->sig && c->side) {
            ncclAllReduce(c->sig + 2 * c->G + 1, c->sig + 2 * c->G + 1, 1, ncclUint64, ncclSum, c->node_comm, c->side);
            cudaStreamSynchronize(c->side);
        }
        for (void* p : c->ipc_opened) cudaIpcCloseMemHandle(p);
        if (c->sig) cudaFree(c->sig);
    }
    for (cudaStream_t st : c->ce_streams) {
        cudaStreamSynchronize(st);
        cudaStreamDestroy(st);
    }
    for (cudaEvent_t ev : c->ce_done) cudaEventDestroy(ev);
    if (!c->ipc_group.empty() || c->xs) {
        // no group member may still push into this rank's slot: group barrier before unmapping
        if (c->group_comm && c->xs && c->side) {
            unsigned long long* scratch = c->xs + 2 * c->P;
            ncclAllReduce(scratch, scratch, 1, ncclUint64, ncclSum, c->group_comm, c->side);
            cudaStreamSynchronize(c->side);
        }
        for (void* p : c->ipc_group) cudaIpcCloseMemHandle(p);
        if (c->xs) cudaFree(c->xs);
    }
    cudaDeviceSynchronize();
    for (int b = 0; b < 3; ++b)
        if (c->own_cuda[b]) cudaFree(c->own_cuda[b]);
    ncclComm_t comms[4] = {c->bucket_comm, c->group_comm, c->node_comm, c->world_comm};
    for (ncclComm_t m : comms) {
        if (!m) continue;
        if (ncclCommFinalize(m) != ncclSuccess) st = DASO_ERR_NCCL;
        if (ncclCommDestroy(m) != ncclSuccess) st = DASO_ERR_NCCL;
    }
    for (cudaEvent_t e : c->pool) cudaEventDestroy(e);
    if (c->ev_packed) cudaEventDestroy(c->ev_packed);
    if (c->ev_exchanged) cudaEventDestroy(c->ev_exchanged);
    if (c->side) cudaStreamDestroy(c->side);
    if (c->slot) cudaFree(c->slot);
    if (c->d_flag) cudaFree(c->d_flag);
    delete c->sched;
    delete c;
    return st;
}

const char* daso_last_error(const daso_ctx* c) { return c ? c->err.c_str() : "null context"; }

// ---------------------------------------------------------------- virtual cluster (one GPU)
// W = P x G virtual ranks, each a full daso_ctx running the product step path (daso_step_ex
// -> step_fused / step_sharded / step_faithful -> the same kernels), on one device and one
// stream.  Only the transport differs: the node tier's peers are the sibling ranks' buffers
// on the same GPU (the fused kernel's barriers are pre-satisfied, see step_fused), and the
// group all-gather (a4) is a device-to-device copy of every packed row into every group
// member's slot, issued after all ranks ran their batch.  This lets the multi-rank path be
// parity-tested against the oracle at any topology on a one-GPU box.
struct daso_vcluster {
    int world = 0, G = 0, P = 0;
    std::vector<daso_ctx*> rank;
    std::vector<void*> owned;   // device allocations (buckets, signal blocks)
    std::string err;
    daso_status fail(daso_status s, const std::string& m) {
        err = m;
        return s;
    }
};

daso_status daso_vcluster_create(daso_vcluster** out, int world, int gpus_per_node, int B, int S,
                                 const daso_config* cfg, size_t n) {
    if (!out || !cfg || n == 0) return DASO_ERR_ARGUMENT;
    *out = nullptr;
    const bool fused = cfg->mode == DASO_MODE_FUSED;
    if (!fused && gpus_per_node != 1) return DASO_ERR_CONFIG;   // NCCL node collectives cannot loop back
    daso_vcluster* v = new (std::nothrow) daso_vcluster;
    if (!v) return DASO_ERR_ARGUMENT;
    *out = v;
    v->world = world;
    v->G = gpus_per_node;
    v->P = gpus_per_node > 0 ? world / gpus_per_node : 0;
    for (int r = 0; r < world; ++r) {
        daso_config rc = *cfg;
        rc.rank = r;
        daso_ctx* c = nullptr;
        const daso_status st = make_ctx(&c, world, gpus_per_node, B, S, &rc);
        if (c) v->rank.push_back(c);
        if (st != DASO_OK) return v->fail(st, c ? c->err : "invalid virtual-cluster configuration");
        c->vc = v;
    }
    const size_t n_pad = daso_padded_numel(n, gpus_per_node);
    for (daso_ctx* c : v->rank) {
        void* p[3] = {nullptr, nullptr, nullptr};
        for (int b = 0; b < 3; ++b) {
            if (cudaMalloc(&p[b], n_pad * sizeof(float)) != cudaSuccess ||
                cudaMemset(p[b], 0, n_pad * sizeof(float)) != cudaSuccess)
                return v->fail(DASO_ERR_CUDA, "virtual cluster: bucket allocation failed");
            v->owned.push_back(p[b]);
        }
        const daso_status st = bind_impl(c, static_cast<float*>(p[0]), static_cast<float*>(p[1]),
                                         static_cast<float*>(p[2]), n);
        if (st != DASO_OK) return v->fail(st, c->err);
    }
    if (fused && gpus_per_node > 1) {   // node tier over the siblings' buffers + one signal block per node
        const int G = gpus_per_node, row = 2 * G + 2;
        for (int j = 0; j < v->P; ++j) {
            void* blk = nullptr;
            if (cudaMalloc(&blk, size_t(G) * row * sizeof(unsigned long long)) != cudaSuccess ||
                cudaMemset(blk, 0, size_t(G) * row * sizeof(unsigned long long)) != cudaSuccess)
                return v->fail(DASO_ERR_CUDA, "virtual cluster: signal allocation failed");
            v->owned.push_back(blk);
            auto* sig = static_cast<unsigned long long*>(blk);
            for (int l = 0; l < G; ++l) {
                daso_ctx* c = v->rank[size_t(j) * G + l];
                c->sig = sig + size_t(l) * row;
                c->vc_node_sig = sig;
                for (int q = 0; q < G; ++q) {
                    daso_ctx* peer = v->rank[size_t(j) * G + q];
                    c->peer_x[q] = peer->x;
                    c->peer_g[q] = peer->g;
                    c->peer_sig[q] = sig + size_t(q) * row;
                }
            }
        }
    }
    if (cfg->exchange == DASO_EXCH_CE && v->P > 1) {
        // the real copy-engine exchange between sibling ranks on this GPU: same-device copies and the same
        // stream memory-op flags / acks as across GPUs (no kernel waits on another: the waits are stream waits)
        if (!write_value64() || !wait_value64()) return v->fail(DASO_ERR_CONFIG, "stream memory operations unavailable");
        const size_t xs_bytes = (2 * size_t(v->P) + 1) * sizeof(unsigned long long);
        for (daso_ctx* c : v->rank) {
            if (cudaMalloc(&c->xs, xs_bytes) != cudaSuccess || cudaMemset(c->xs, 0, xs_bytes) != cudaSuccess)
                return v->fail(DASO_ERR_CUDA, "virtual cluster: flag allocation failed");
        }
        for (daso_ctx* c : v->rank) {
            c->peer_slot.assign(size_t(v->P), nullptr);
            c->peer_xs.assign(size_t(v->P), nullptr);
            for (int i = 0; i < v->P; ++i) {
                daso_ctx* m = v->rank[size_t(i) * v->G + c->local];   // group member on node i
                c->peer_slot[i] = m->slot;
                c->peer_xs[i] = m->xs;
            }
            for (int k = 1; k < v->P; ++k) {
                cudaStream_t st = nullptr;
                cudaEvent_t ev = nullptr;
                if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess ||
                    cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess)
                    return v->fail(DASO_ERR_CUDA, "virtual cluster: stream creation failed");
                c->ce_streams.push_back(st);
                c->ce_done.push_back(ev);
            }
            c->ce = true;
        }
    }
    if (cudaDeviceSynchronize() != cudaSuccess) return v->fail(DASO_ERR_CUDA, "virtual cluster: setup failed");
    return DASO_OK;
}

daso_status daso_vcluster_buffers(daso_vcluster* v, int rank, float** x, float** g, float** vb) {
    if (!v || rank < 0 || rank >= int(v->rank.size())) return DASO_ERR_RANGE;
    daso_ctx* c = v->rank[size_t(rank)];
    if (x) *x = c->x;
    if (g) *g = c->g;
    if (vb) *vb = c->v;
    return DASO_OK;
}

daso_ctx* daso_vcluster_rank(daso_vcluster* v, int rank) {
    if (!v || rank < 0 || rank >= int(v->rank.size())) return nullptr;
    return v->rank[size_t(rank)];
}

daso_status daso_vcluster_step(daso_vcluster* v, float lr, int plateau, void* stream, daso_record* out) {
    if (!v || v->rank.empty()) return DASO_ERR_ARGUMENT;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    daso_record r0{};
    bool sent = false, blocking = false;
    for (size_t i = 0; i < v->rank.size(); ++i) {   // every rank's batch, in rank order
        daso_ctx* c = v->rank[i];
        c->vc_sent = c->vc_blocking = false;
        daso_record r{};
        const daso_status st = daso_step_ex(c, lr, plateau, 0, stream, &r);
        if (st != DASO_OK) return v->fail(st, "rank " + std::to_string(i) + ": " + c->err);
        if (i == 0) r0 = r;
        else if (std::memcmp(&r, &r0, sizeof r) != 0) return v->fail(DASO_ERR_PROTOCOL, "ranks disagree on the schedule");
        if (out) out[i] = r;
        sent |= c->vc_sent;
        blocking |= c->vc_blocking;
    }
    if (sent && v->rank[0]->ce) {
        // the real copy-engine exchange, issued only now: every rank's merge and its consumed acks are
        // already enqueued, so every stream wait (flow control on the copy streams, arrival at a later
        // merge) depends only on earlier work — within one process streams share hardware queues, and a
        // wait on a flag that later work of the same process writes could block that very work
        for (size_t i = 0; i < v->rank.size(); ++i) {
            daso_ctx* c = v->rank[i];
            if (!c->vc_sent) continue;
            const daso_status st = push_exchange(c, s);
            if (st != DASO_OK) return v->fail(st, "rank " + std::to_string(i) + ": " + c->err);
        }
    } else if (sent) {   // loopback group all-gather: member (i, l)'s packed row -> row i of every member (j, l)
        const size_t wb = v->rank[0]->wire_bytes, seg = size_t(v->rank[0]->seg);
        for (int l = 0; l < v->G; ++l)
            for (int i = 0; i < v->P; ++i) {
                daso_ctx* src = v->rank[size_t(i) * v->G + l];
                if (!src->vc_sent) continue;
                for (int j = 0; j < v->P; ++j) {
                    if (j == i) continue;
                    daso_ctx* dst = v->rank[size_t(j) * v->G + l];
                    if (cudaMemcpyAsync(static_cast<char*>(dst->slot) + size_t(i) * seg * wb, own_segment(src),
                                        seg * wb, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
                        return v->fail(DASO_ERR_CUDA, "virtual cluster: loopback all-gather copy failed");
                }
            }
    }
    if (blocking)
        for (size_t i = 0; i < v->rank.size(); ++i) {
            daso_ctx* c = v->rank[i];
            if (!c->vc_blocking) continue;
            const daso_status st = finish_blocking(c, s);
            if (st != DASO_OK) return v->fail(st, "rank " + std::to_string(i) + ": " + c->err);
        }
    return DASO_OK;
}

daso_status daso_vcluster_destroy(daso_vcluster* v) {
    if (!v) return DASO_OK;
    cudaDeviceSynchronize();
    daso_status st = DASO_OK;
    for (daso_ctx* c : v->rank) {
        c->sig = nullptr;   // owned by the cluster's signal blocks
        if (daso_finalize(c) != DASO_OK) st = DASO_ERR_CUDA;
    }
    for (void* p : v->owned) cudaFree(p);
    delete v;
    return st;
}

const char* daso_vcluster_last_error(const daso_vcluster* v) { return v ? v->err.c_str() : "null cluster"; }

// ---------------------------------------------------------------- kernel entry points
static bool aligned16(const void* p) { return (uintptr_t(p) & 15u) == 0; }

static daso_status kstatus(int e) { return e == 0 ? DASO_OK : DASO_ERR_CUDA; }

daso_status daso_k_update(float* x, float* v, const float* g, size_t n, float lr, float mu, float wd, float gscale,
                          void* pack_out, int wire, uint32_t* flag, void* stream) {
    if (n == 0) return DASO_OK;   // empty bucket: nothing to do
    if (!x || !v || !g || !aligned16(x) || !aligned16(v) || !aligned16(g)) return DASO_ERR_ARGUMENT;
    if (pack_out && !aligned16(pack_out)) return DASO_ERR_ARGUMENT;
    if (wire != DASO_WIRE_BF16 && wire != DASO_WIRE_FP32) return DASO_ERR_ARGUMENT;
    daso::KernelArgs a;
    a.x = x; a.v = v; a.g = g; a.n = int64_t(n);
    a.lr = lr; a.mu = mu; a.wd = wd; a.gscale = gscale;
    a.pack_out = pack_out; a.flag = flag;
    return kstatus(daso::launch_fused(daso::OP_UPDATE | (pack_out ? daso::OP_PACK : 0), wire, a, stream));
}

static bool slot_ok(const void* slot, size_t stride, int P, int wire) {
    const size_t eb = wire == DASO_WIRE_BF16 ? 2 : 4;
    return slot && P >= 1 && aligned16(slot) && (stride * eb) % 16 == 0;
}

daso_status daso_k_update_merge(float* x, float* v, const float* g, size_t n, float lr, float mu, float wd,
                                float gscale, const void* slot, size_t slot_stride, int P, int S, void* pack_out,
                                int wire, uint32_t* flag, void* stream) {
    if (n == 0) return DASO_OK;
    if (!x || !v || !g || !aligned16(x) || !aligned16(v) || !aligned16(g)) return DASO_ERR_ARGUMENT;
    if (wire != DASO_WIRE_BF16 && wire != DASO_WIRE_FP32) return DASO_ERR_ARGUMENT;
    if (!slot_ok(slot, slot_stride, P, wire) || slot_stride < n || S < 1) return DASO_ERR_ARGUMENT;
    if (pack_out && !aligned16(pack_out)) return DASO_ERR_ARGUMENT;
    daso::KernelArgs a;
    a.x = x; a.v = v; a.g = g; a.n = int64_t(n);
    a.lr = lr; a.mu = mu; a.wd = wd; a.gscale = gscale;
    a.slot = slot; a.slot_stride = int64_t(slot_stride); a.P = P; a.den = float(2 * S + P);
    a.pack_out = pack_out; a.flag = flag;
    return kstatus(daso::launch_fused(daso::OP_UPDATE | daso::OP_MERGE | (pack_out ? daso::OP_PACK : 0), wire, a,
                                      stream));
}

daso_status daso_k_merge(float* x, size_t n, const void* slot, size_t slot_stride, int P, int S, void* pack_out,
                         int wire, uint32_t* flag, void* stream) {
    if (n == 0) return DASO_OK;
    if (!x || !aligned16(x)) return DASO_ERR_ARGUMENT;
    if (wire != DASO_WIRE_BF16 && wire != DASO_WIRE_FP32) return DASO_ERR_ARGUMENT;
    if (!slot_ok(slot, slot_stride, P, wire) || slot_stride < n || S < 1) return DASO_ERR_ARGUMENT;
    if (pack_out && !aligned16(pack_out)) return DASO_ERR_ARGUMENT;
    daso::KernelArgs a;
    a.x = x; a.n = int64_t(n);
    a.slot = slot; a.slot_stride = int64_t(slot_stride); a.P = P; a.den = float(2 * S + P);
    a.pack_out = pack_out; a.flag = flag;
    return kstatus(daso::launch_fused(daso::OP_MERGE | (pack_out ? daso::OP_PACK : 0), wire, a, stream));
}

daso_status daso_k_average(float* x, size_t n, const void* slot, size_t slot_stride, int P, int wire, uint32_t* flag,
                           void* stream) {
    if (n == 0) return DASO_OK;
    if (!x || !aligned16(x)) return DASO_ERR_ARGUMENT;
    if (wire != DASO_WIRE_BF16 && wire != DASO_WIRE_FP32) return DASO_ERR_ARGUMENT;
    if (!slot_ok(slot, slot_stride, P, wire) || slot_stride < n) return DASO_ERR_ARGUMENT;
    daso::KernelArgs a;
    a.x = x; a.n = int64_t(n);
    a.slot = slot; a.slot_stride = int64_t(slot_stride); a.P = P; a.den = float(P);
    a.flag = flag;
    return kstatus(daso::launch_fused(daso::OP_AVERAGE, wire, a, stream));
}

daso_status daso_k_pack(const float* x, size_t n, void* pack_out, int wire, void* stream) {
    if (n == 0) return DASO_OK;
    if (!x || !pack_out || !aligned16(x) || !aligned16(pack_out)) return DASO_ERR_ARGUMENT;
    if (wire != DASO_WIRE_BF16 && wire != DASO_WIRE_FP32) return DASO_ERR_ARGUMENT;
    daso::KernelArgs a;
    a.x = const_cast<float*>(x); a.n = int64_t(n);
    a.pack_out = pack_out;
    return kstatus(daso::launch_fused(daso::OP_PACK, wire, a, stream));
}

daso_status daso_flat_layout(const size_t* numel, int count, size_t align_elems, size_t* offsets, size_t* total) {
    if (!numel || !offsets || !total || count < 0 || align_elems == 0) return DASO_ERR_ARGUMENT;
    size_t off = 0;
    for (int i = 0; i < count; ++i) {
        offsets[i] = off;
        off += (numel[i] + align_elems - 1) / align_elems * align_elems;
    }
    *total = off;
    return DASO_OK;
}

daso_status daso_k_gather(const float* const* src, const size_t* numel, const size_t* offsets, int count, float* dst,
                          void* stream) {
    if (!src || !numel || !offsets || !dst || count < 0) return DASO_ERR_ARGUMENT;
    return kstatus(daso::launch_gather(src, numel, offsets, count, dst, stream));
}

daso_status daso_k_scatter(const float* src, float* const* dst, const size_t* numel, const size_t* offsets, int count,
                           void* stream) {
    if (!src || !numel || !offsets || !dst || count < 0) return DASO_ERR_ARGUMENT;
    return kstatus(daso::launch_scatter(src, dst, numel, offsets, count, stream));
}

int daso_kernel_impl(int impl) { return daso::set_kernel_impl(impl); }

daso_status daso_k_checksum(const float* x, size_t n, uint64_t* out_dev, void* stream) {
    if (!x || !out_dev) return DASO_ERR_ARGUMENT;
    return kstatus(daso::launch_checksum(x, int64_t(n), out_dev, stream));
}

}  // extern "C"
