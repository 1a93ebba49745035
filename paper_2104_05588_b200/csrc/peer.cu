// Fused node-local tier over NVLink peer memory (DASO_MODE_FUSED).
//
// One kernel per rank and batch replaces [node reduce-scatter of g -> shard update
// (+ Eq. (1) merge) (+ bf16 pack) -> node all-gather of x]:
//   1. start barrier: each rank signals every node peer "my g is ready" (system-scope
//      release store into the peer's signal array) and waits for all peers' signals;
//   2. each rank owns shard `me` of the parameters: it loads that shard of every node
//      peer's gradient through NVLink (Fig. 2 "gradients from each GPU are
//      averaged"; summed in ascending local id — the oracle's order, R18), applies the
//      momentum-SGD update and, if due, the Eq. (1) merge and the bf16
//      pack, and stores the new shard into every peer's x (Fig. 4 "replace the
//      old parameters on those GPUs") — the node all-gather as direct NVLink stores;
//   3. end barrier: the last CTA to finish signals every peer "done" after a
//      system-scope fence and waits for all peers, so when the kernel completes every
//      GPU of the node holds the full new x and no peer still reads this rank's g.
// Node replicas stay bitwise identical; the arithmetic per element is K1/K3's.
// Blocking batches (Fig. 3) run the kernel as OP_NOX (pack only: no x stores, no end
// barrier) and finish with avg_publish_[tma_]kernel: the group average of the shard stored into
// every peer's x, then the end barrier (Fig. 4 re-publish).
// Each rank is its own GPU (one process per GPU), so the spin-waits never wait on a
// kernel of the same GPU; the grid leaves room on every SM for the side-stream NCCL
// exchange kernels to run concurrently.
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>

#include "daso_internal.h"
#include "device_common.cuh"

namespace daso {
namespace {
using namespace dev;

constexpr int kPeerThreads = 256;
constexpr int kPV = 8;   // parameters per thread per iteration (two 128-bit accesses per stream)

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}


// Spin until *p >= v.  A peer that never arrives (crashed process, protocol bug) must not
// hang the GPU: after `timeout_ns` the wait gives up, raises bit 1 of the error word
// (daso_check_finite reports it) and returns false; the kernel then skips its body, so
// it never reads or writes unsynchronised peer memory.
__device__ __forceinline__ bool wait_geq(const unsigned long long* p, unsigned long long v, uint32_t* flag,
                                         unsigned long long timeout_ns) {
    if (ld_acquire_sys(p) >= v) return true;
    const unsigned long long t0 = globaltimer_ns();
    while (ld_acquire_sys(p) < v) {
        if (globaltimer_ns() - t0 > timeout_ns) {
            if (flag) atomicOr(flag, 2u);
            return false;
        }
        __nanosleep(64);
    }
    return true;
}

// Start barrier: CTA 0 signals every node peer "my g is ready" (slot `me` of their
// start row); thread 0 of every CTA waits for all G start signals.  Returns false (in
// every thread of the CTA) if a wait timed out.
__device__ __forceinline__ bool start_barrier(const PeerArgs& pa, int G) {
    __shared__ int s_ok;
    if (blockIdx.x == 0 && threadIdx.x < G) {
        __threadfence_system();
        st_release_sys(pa.sig_peer[threadIdx.x] + pa.me, pa.epoch);
    }
    if (threadIdx.x == 0) {
        bool ok = true;
        for (int q = 0; q < G && ok; ++q) ok = wait_geq(pa.sig_me + q, pa.epoch, pa.err, pa.timeout_ns);
        s_ok = ok;
    }
    __syncthreads();
    return s_ok != 0;
}

// End barrier: the last CTA to finish (CTA counter `done`) signals every peer "my x
// stores and g reads are complete" after a system fence and waits for all peers, so when
// the kernel completes the node holds the full new x and no peer still reads this g.
__device__ __forceinline__ void end_barrier(const PeerArgs& pa, int G) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        const unsigned prev = atomicAdd(pa.done, 1u);
        if (prev == gridDim.x - 1) {
            *reinterpret_cast<volatile unsigned*>(pa.done) = 0u;
            __threadfence_system();
            for (int q = 0; q < G; ++q) st_release_sys(pa.sig_peer[q] + G + pa.me, pa.epoch);
            for (int q = 0; q < G; ++q)
                if (!wait_geq(pa.sig_me + G + q, pa.epoch, pa.err, pa.timeout_ns)) break;
        }
    }
}

template <int OPS, int WIRE, int G, int N>
__device__ __forceinline__ void peer_body(const PeerArgs& pa, int64_t i, bool& bad) {
    const KernelArgs& a = pa.a;
    float x[N], v[N], g[N];
    float gq[G][N];
#pragma unroll
    for (int q = 0; q < G; ++q) ld_f32<N>(pa.gp[q] + i, gq[q]);   // all peer loads in flight first
    ld_f32<N>(a.x + i, x);
    ld_f32<N>(a.v + i, v);
#pragma unroll
    for (int j = 0; j < N; ++j) g[j] = gq[0][j];
#pragma unroll
    for (int q = 1; q < G; ++q) {
#pragma unroll
        for (int j = 0; j < N; ++j) g[j] += gq[q][j];                // ascending local id (R18)
    }
#pragma unroll
    for (int j = 0; j < N; ++j) {
        const float d = fmaf(a.wd, x[j], g[j] * a.gscale);
        v[j] = fmaf(a.mu, v[j], d);
        x[j] = fmaf(-a.lr, v[j], x[j]);
    }
    st_f32<N>(a.v + i, v);
    if constexpr ((OPS & OP_MERGE) != 0) {
        float acc[N];
#pragma unroll
        for (int j = 0; j < N; ++j) acc[j] = 0.f;
#pragma unroll 4
        for (int p = 0; p < a.P; ++p) {
            float s[N];
            Wire<WIRE>::template load<N>(a.slot, p * a.slot_stride + i, s);
#pragma unroll
            for (int j = 0; j < N; ++j) acc[j] += s[j] - x[j];
        }
#pragma unroll
        for (int j = 0; j < N; ++j) x[j] = x[j] + acc[j] / a.den;
    }
    if constexpr ((OPS & OP_NOX) == 0) {
#pragma unroll
        for (int q = 0; q < G; ++q) st_f32<N>(pa.xp[q] + i, x);
    }
#pragma unroll
    for (int j = 0; j < N; ++j) bad |= !isfinite(x[j]);
    if constexpr ((OPS & OP_PACK) != 0) {
        Wire<WIRE>::template store<N>(a.pack_out, i, x);
        if constexpr ((OPS & OP_PUSH) != 0) {   // group members' slots (a separate instantiation: the
#pragma unroll                                        // push code costs the plain pack kernels registers)
            for (int k = 0; k < kMaxPush; ++k)
                if (k < a.npush) Wire<WIRE>::template store<N>(a.push[k], i, x);
        }
    }
}

template <int OPS, int WIRE, int G>
__global__ void __launch_bounds__(kPeerThreads) peer_kernel(const PeerArgs pa) {
    if (!start_barrier(pa, G)) return;   // 1. start barrier (timed out: error bit raised, do nothing)
    // 2. shard update over NVLink
    bool bad = false;
    const int64_t n = pa.a.n;
    const int64_t nch = n / kPV;
    const int64_t stride = int64_t(gridDim.x) * kPeerThreads;
    for (int64_t c = int64_t(blockIdx.x) * kPeerThreads + threadIdx.x; c < nch; c += stride)
        peer_body<OPS, WIRE, G, kPV>(pa, c * kPV, bad);
    if (blockIdx.x == gridDim.x - 1) {
        const int64_t i = nch * kPV + threadIdx.x;
        if (i < n) peer_body<OPS, WIRE, G, 1>(pa, i, bad);
    }
    if (pa.a.flag != nullptr) {
        const unsigned any = __ballot_sync(0xffffffffu, bad);
        if (any != 0u && (threadIdx.x & 31) == 0) atomicOr(pa.a.flag, 1u);
    }
    if constexpr ((OPS & OP_NOX) == 0) end_barrier(pa, G);   // 3. end barrier
}

int peer_blocks_per_sm() {   // grid = SMs x this (DASO_PEER_BPSM, default 2 (measured best)); one-shot if larger
    static int v = 0;
    if (v == 0) {
        const char* e = getenv("DASO_PEER_BPSM");
        v = e ? atoi(e) : 2;
        if (v < 1) v = 1;
    }
    return v;
}

template <int OPS, int WIRE, int G>
int launch_peer_t(const PeerArgs& pa, cudaStream_t s, int sms) {
    const int64_t nch = pa.a.n / kPV;
    int64_t blocks = (nch + kPeerThreads - 1) / kPeerThreads;
    blocks = std::max<int64_t>(1, std::min<int64_t>(blocks, int64_t(sms) * peer_blocks_per_sm()));
    peer_kernel<OPS, WIRE, G><<<dim3(unsigned(blocks)), dim3(kPeerThreads), 0, s>>>(pa);
    return int(cudaGetLastError());
}


// ---- TMA-staged variant (daso_kernel_impl(1)): the same batch with the peer gradient
// loads and the peer parameter stores done by the bulk-copy engine (cp.async.bulk on
// NVLink-mapped global addresses) through an mbarrier ring of shared-memory stages, one
// persistent CTA per SM.  Per tile: own x, v + G gradient tiles (G-1 remote) in; x out
// to G peers (G-1 remote), v and the packed row out locally.
constexpr int kPT = 2048;

struct PeerTmaLayout {   // byte offsets: NS input stages, then NO output buffers, then NS mbarriers
    uint32_t x, v, g, slot, in_bytes;    // inside an input stage
    uint32_t ox, ov, opack, out_bytes;   // inside an output buffer
};
__host__ __device__ inline PeerTmaLayout peer_tma_layout(int ops, int G, int P, int wb) {
    PeerTmaLayout L{};
    uint32_t o = 0;
    L.x = o; o += kPT * 4;
    L.v = o; o += kPT * 4;
    L.g = o; o += uint32_t(G) * kPT * 4;
    L.slot = o; if (ops & OP_MERGE) o += uint32_t(P) * kPT * wb;
    L.in_bytes = (o + 127) / 128 * 128;
    o = 0;
    L.ox = o; o += kPT * 4;
    L.ov = o; o += kPT * 4;
    L.opack = o; if (ops & OP_PACK) o += kPT * wb;
    L.out_bytes = (o + 127) / 128 * 128;
    return L;
}
constexpr int kPeerOut = 2;   // output buffers (double-buffered bulk stores)

__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

// Input stage s is refilled as soon as its tile has been computed (outputs go to a separate
// double-buffered output area), so the loads never wait for the NVLink stores to drain.
template <int OPS, int WIRE, int G>
__global__ void __launch_bounds__(kPeerThreads, 1) peer_tma_kernel(const PeerArgs pa, int NS) {
    extern __shared__ __align__(128) unsigned char smem[];
    constexpr int wb = WIRE == DASO_WIRE_BF16 ? 2 : 4;
    const KernelArgs& a = pa.a;
    const PeerTmaLayout L = peer_tma_layout(OPS, G, a.P, wb);
    unsigned char* outs = smem + size_t(NS) * L.in_bytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(outs + size_t(kPeerOut) * L.out_bytes);
    const bool leader = threadIdx.x == 0;
    if (!start_barrier(pa, G)) return;   // 1. start barrier (timed out: error bit raised, do nothing)
    if (leader) {
        for (int s = 0; s < NS; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        fence_proxy_async_global();
    }
    __syncthreads();

    const int64_t ntiles = a.n / kPT;
    const int64_t my = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    auto issue_load = [&](int64_t k) {
        const int s = int(k % NS);
        unsigned char* st = smem + size_t(s) * L.in_bytes;
        const int64_t e0 = (int64_t(blockIdx.x) + k * gridDim.x) * kPT;
        uint32_t tx = (2u + G) * kPT * 4u;
        if constexpr ((OPS & OP_MERGE) != 0) tx += uint32_t(a.P) * kPT * wb;
        mbar_expect_tx(&full[s], tx);
#pragma unroll
        for (int q = 0; q < G; ++q) bulk_g2s(st + L.g + uint32_t(q) * kPT * 4, pa.gp[q] + e0, kPT * 4, &full[s]);
        bulk_g2s(st + L.x, a.x + e0, kPT * 4, &full[s]);
        bulk_g2s(st + L.v, a.v + e0, kPT * 4, &full[s]);
        if constexpr ((OPS & OP_MERGE) != 0) {
            for (int p = 0; p < a.P; ++p)
                bulk_g2s(st + L.slot + uint32_t(p) * kPT * wb,
                         static_cast<const unsigned char*>(a.slot) + (p * a.slot_stride + e0) * wb, kPT * wb, &full[s]);
        }
    };
    if (leader)
        for (int64_t k = 0; k < my && k < NS; ++k) issue_load(k);

    bool bad = false;
    for (int64_t k = 0; k < my; ++k) {
        const int s = int(k % NS);
        unsigned char* st = smem + size_t(s) * L.in_bytes;
        unsigned char* ob = outs + size_t(k % kPeerOut) * L.out_bytes;
        if (leader && k >= kPeerOut) bulk_wait_read<kPeerOut - 1>();   // output buffer ob drained
        if (!mbar_wait(&full[s], uint32_t((k / NS) & 1), pa.err)) break;   // timed out: bit 2 raised, stop
        __syncthreads();                                                 // also publishes the drain
        const int i = threadIdx.x * 8;
        float x[8], v[8], g[8];
        Wire<DASO_WIRE_FP32>::template load_smem<8>(st + L.x, i, x);
        Wire<DASO_WIRE_FP32>::template load_smem<8>(st + L.v, i, v);
        Wire<DASO_WIRE_FP32>::template load_smem<8>(st + L.g, i, g);
#pragma unroll
        for (int q = 1; q < G; ++q) {
            float t[8];
            Wire<DASO_WIRE_FP32>::template load_smem<8>(st + L.g + uint32_t(q) * kPT * 4, i, t);
#pragma unroll
            for (int j = 0; j < 8; ++j) g[j] += t[j];                        // ascending local id (R18)
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const float d = fmaf(a.wd, x[j], g[j] * a.gscale);
            v[j] = fmaf(a.mu, v[j], d);
            x[j] = fmaf(-a.lr, v[j], x[j]);
        }
        if constexpr ((OPS & OP_MERGE) != 0) {
            float acc[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[j] = 0.f;
            for (int p = 0; p < a.P; ++p) {
                float sv[8];
                Wire<WIRE>::template load_smem<8>(st + L.slot + uint32_t(p) * kPT * wb, i, sv);
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[j] += sv[j] - x[j];
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) x[j] = x[j] + acc[j] / a.den;
        }
        if constexpr ((OPS & OP_NOX) == 0) Wire<DASO_WIRE_FP32>::template store_smem<8>(ob + L.ox, i, x);
        Wire<DASO_WIRE_FP32>::template store_smem<8>(ob + L.ov, i, v);
        if constexpr ((OPS & OP_PACK) != 0) Wire<WIRE>::template store_smem<8>(ob + L.opack, i, x);
#pragma unroll
        for (int j = 0; j < 8; ++j) bad |= !isfinite(x[j]);
        fence_async_smem();
        __syncthreads();                                                 // stage s consumed, ob written
        if (leader) {
            if (k + NS < my) issue_load(k + NS);                         // refill stage s right away
            const int64_t e0 = (int64_t(blockIdx.x) + k * gridDim.x) * kPT;
            if constexpr ((OPS & OP_NOX) == 0) {
#pragma unroll
                for (int q = 0; q < G; ++q) {                            // start with the next peer: spread links
                    const int qq = (pa.me + 1 + q) % G;
                    bulk_s2g(pa.xp[qq] + e0, ob + L.ox, kPT * 4);
                }
            }
            bulk_s2g(a.v + e0, ob + L.ov, kPT * 4);
            if constexpr ((OPS & OP_PACK) != 0) {
                bulk_s2g(static_cast<unsigned char*>(a.pack_out) + e0 * wb, ob + L.opack, kPT * wb);
                if constexpr ((OPS & OP_PUSH) != 0) {
#pragma unroll
                    for (int k = 0; k < kMaxPush; ++k)                  // group members' slots (kernel push)
                        if (k < a.npush)
                            bulk_s2g(static_cast<unsigned char*>(a.push[k]) + e0 * wb, ob + L.opack, kPT * wb);
                }
            }
            bulk_commit();
        }
    }
    if (leader) bulk_wait_all();
    if (blockIdx.x == gridDim.x - 1)
        for (int64_t e = ntiles * kPT + threadIdx.x; e < a.n; e += blockDim.x) peer_body<OPS, WIRE, G, 1>(pa, e, bad);
    if (a.flag != nullptr) {
        const unsigned any = __ballot_sync(0xffffffffu, bad);
        if (any != 0u && (threadIdx.x & 31) == 0) atomicOr(a.flag, 1u);
    }
    // 3. end barrier (all bulk stores of this CTA are complete: wait_group 0 above)
    if constexpr ((OPS & OP_NOX) == 0) {
        if (leader) fence_proxy_async_global();
        end_barrier(pa, G);
    }
}

int peer_tma_ctas() {   // DASO_PEER_TMA_CTAS, 0 = default (SMs - 16)
    static int ctas = -1;
    if (ctas < 0) {
        const char* e = getenv("DASO_PEER_TMA_CTAS");
        ctas = e ? std::max(1, atoi(e)) : 0;
    }
    return ctas;
}

template <int OPS, int WIRE, int G>
int launch_peer_tma_t(const PeerArgs& pa, cudaStream_t s, int sms) {
    constexpr int wb = WIRE == DASO_WIRE_BF16 ? 2 : 4;
    const PeerTmaLayout L = peer_tma_layout(OPS, G, pa.a.P, wb);
    const int budget = 210 * 1024 - kPeerOut * int(L.out_bytes);
    const int NS = int(std::min<int64_t>(8, (budget - 64) / L.in_bytes));
    if (NS < 2) return launch_peer_t<OPS, WIRE, G>(pa, s, sms);
    const size_t smem = size_t(NS) * L.in_bytes + size_t(kPeerOut) * L.out_bytes + 8 * size_t(NS);
    static size_t attr = 0;   // opt-in limit set so far (static + dynamic must fit the 227 KB per CTA)
    if (smem > attr) {
        const cudaError_t e = cudaFuncSetAttribute(peer_tma_kernel<OPS, WIRE, G>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (e != cudaSuccess) return int(e);
        attr = smem;
    }
    // DASO_PEER_TMA_CTAS: persistent CTAs.  Default: one per SM minus 16, so the side-stream
    // exchange's NCCL kernels always find free SMs (2x2: exchange hidden 0.98 vs 0.73 with every
    // SM taken, same kernel time; profiles/r01/b20_*).
    const int grid = peer_tma_ctas() > 0 ? std::min(peer_tma_ctas(), sms) : std::max(1, sms - 16);
    peer_tma_kernel<OPS, WIRE, G><<<dim3(unsigned(grid)), dim3(kPeerThreads), smem, s>>>(pa, NS);
    return int(cudaGetLastError());
}

// ---- warp-specialised TMA variant (DASO_PEER=ws): the same batch and arithmetic as
// peer_tma_kernel, with the data movement decoupled from the compute by mbarriers instead of
// CTA-wide barriers.  9 warps: warps 0-7 compute (8 parameters per thread of a 2048-parameter
// tile), warp 8 lane 0 is the TMA engine driver:
//   full[s]   (tx bytes)  stage s holds tile k's own x, v, the G gradient tiles (+ slot rows);
//   ofull[o]  (8 arrivals) the compute warps have consumed stage k % NS and written tile k's
//                          new x, v (+ packed row) into output buffer o = k % NO;
//   oempty[o] (1 arrival)  the bulk stores issued from output buffer o have read it.
// The driver refills a stage as soon as its tile is computed and issues the stores of every
// output buffer as soon as it is written, so NVLink reads, NVLink stores and compute of
// different tiles overlap continuously; no thread ever waits for the whole CTA.
constexpr int kWsCompute = 256, kWsThreads = kWsCompute + 32, kWsMaxOut = 4;

// cp.async.bulk.wait_group.read takes an immediate: dispatch the runtime count (1..kWsMaxOut-1)
__device__ __forceinline__ void bulk_wait_read_upto(int n) {
    if (n <= 1) bulk_wait_read<1>();
    else if (n == 2) bulk_wait_read<2>();
    else bulk_wait_read<3>();
}

// Output buffers of the warp-specialised kernel (DASO_PEER_OUT = 2..4, default 2): how many tiles'
// bulk stores may still be reading their shared-memory buffers while the compute warps fill the next.
int peer_ws_out() {   // read per launch, so a test can compare the settings in one process
    const char* e = getenv("DASO_PEER_OUT");
    return e ? std::max(2, std::min(kWsMaxOut, atoi(e))) : 2;
}

template <int OPS, int WIRE, int G>
__global__ void __launch_bounds__(kWsThreads, 1) peer_ws_kernel(const PeerArgs pa, int NS, int NO) {
    extern __shared__ __align__(128) unsigned char smem[];
    constexpr int wb = WIRE == DASO_WIRE_BF16 ? 2 : 4;
    const KernelArgs& a = pa.a;
    const PeerTmaLayout L = peer_tma_layout(OPS, G, a.P, wb);
    unsigned char* outs = smem + size_t(NS) * L.in_bytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(outs + size_t(NO) * L.out_bytes);
    uint64_t* ofull = full + NS;
    uint64_t* oempty = ofull + NO;
    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int s = 0; s < NS; ++s) mbar_init(&full[s], 1);
        for (int o = 0; o < NO; ++o) {
            mbar_init(&ofull[o], kWsCompute / 32);
            mbar_init(&oempty[o], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        fence_proxy_async_global();
    }
    if (blockIdx.x == 0 && tid < G) {   // 1a. start barrier, signal half: "my g is ready" to every peer
        __threadfence_system();
        st_release_sys(pa.sig_peer[tid] + pa.me, pa.epoch);
    }
    __syncthreads();
    const int64_t ntiles = a.n / kPT;
    const int64_t my = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    auto tile0 = [&](int64_t k) { return (int64_t(blockIdx.x) + k * gridDim.x) * kPT; };
    bool bad = false;
    if (tid == kWsCompute) {   // ---- the TMA driver
        // Only the peers' gradient tiles need the start barrier: the local part of a stage (own x, v,
        // own g, slot rows) is issued first, so the first stages load while the signals travel.
        auto issue_local = [&](int64_t k) {
            const int s = int(k % NS);
            unsigned char* st = smem + size_t(s) * L.in_bytes;
            const int64_t e0 = tile0(k);
            uint32_t tx = (2u + G) * kPT * 4u;
            if constexpr ((OPS & OP_MERGE) != 0) tx += uint32_t(a.P) * kPT * wb;
            mbar_expect_tx(&full[s], tx);
            bulk_g2s(st + L.g + uint32_t(pa.me) * kPT * 4, pa.gp[pa.me] + e0, kPT * 4, &full[s]);
            bulk_g2s(st + L.x, a.x + e0, kPT * 4, &full[s]);
            bulk_g2s(st + L.v, a.v + e0, kPT * 4, &full[s]);
            if constexpr ((OPS & OP_MERGE) != 0) {
                for (int p = 0; p < a.P; ++p)
                    bulk_g2s(st + L.slot + uint32_t(p) * kPT * wb,
                             static_cast<const unsigned char*>(a.slot) + (p * a.slot_stride + e0) * wb, kPT * wb,
                             &full[s]);
            }
        };
        auto issue_remote = [&](int64_t k) {
            const int s = int(k % NS);
            unsigned char* st = smem + size_t(s) * L.in_bytes;
            const int64_t e0 = tile0(k);
#pragma unroll
            for (int q = 1; q < G; ++q) {                       // start with the next peer: spread links
                const int qq = (pa.me + q) % G;
                bulk_g2s(st + L.g + uint32_t(qq) * kPT * 4, pa.gp[qq] + e0, kPT * 4, &full[s]);
            }
        };
        auto issue_load = [&](int64_t k) {
            issue_local(k);
            issue_remote(k);
        };
        for (int64_t k = 0; k < my && k < NS; ++k) issue_local(k);
        bool ok = true;   // 1b. start barrier, wait half: every peer's g is ready
        for (int q = 0; q < G && ok; ++q) ok = wait_geq(pa.sig_me + q, pa.epoch, pa.err, pa.timeout_ns);
        // (timed out: error bit raised; the remote tiles are never requested, the compute warps' stage
        // waits time out as well, and nothing touches peer memory)
        if (ok)
            for (int64_t k = 0; k < my && k < NS; ++k) issue_remote(k);
        for (int64_t k = 0; k < my && ok; ++k) {
            const int o = int(k % NO);
            if (!mbar_wait(&ofull[o], uint32_t((k / NO) & 1), pa.err)) break;
            if (k + NS < my) issue_load(k + NS);                // stage k % NS consumed: refill it
            unsigned char* ob = outs + size_t(o) * L.out_bytes;
            const int64_t e0 = tile0(k);
            if constexpr ((OPS & OP_NOX) == 0) {
#pragma unroll
                for (int q = 0; q < G; ++q) {
                    const int qq = (pa.me + 1 + q) % G;
                    bulk_s2g(pa.xp[qq] + e0, ob + L.ox, kPT * 4);
                }
            }
            bulk_s2g(a.v + e0, ob + L.ov, kPT * 4);
            if constexpr ((OPS & OP_PACK) != 0) {
                bulk_s2g(static_cast<unsigned char*>(a.pack_out) + e0 * wb, ob + L.opack, kPT * wb);
                if constexpr ((OPS & OP_PUSH) != 0) {
#pragma unroll
                    for (int k = 0; k < kMaxPush; ++k)                  // group members' slots (kernel push)
                        if (k < a.npush)
                            bulk_s2g(static_cast<unsigned char*>(a.push[k]) + e0 * wb, ob + L.opack, kPT * wb);
                }
            }
            bulk_commit();
            if (k >= NO - 1) {                                  // up to NO-1 tiles' stores may still read
                bulk_wait_read_upto(NO - 1);                    // their buffers; tile k-(NO-1)'s has been read
                mbar_arrive(&oempty[(k - (NO - 1)) % NO]);
            }
        }
        bulk_wait_all();
    } else if (tid < kWsCompute) {   // ---- compute warps
        for (int64_t k = 0; k < my; ++k) {
            const int s = int(k % NS), o = int(k % NO);
            unsigned char* st = smem + size_t(s) * L.in_bytes;
            unsigned char* ob = outs + size_t(o) * L.out_bytes;
            if (!mbar_wait(&full[s], uint32_t((k / NS) & 1), pa.err)) break;
            const int i = tid * 8;
            float x[8], v[8], g[8];
            Wire<DASO_WIRE_FP32>::template load_smem<8>(st + L.x, i, x);
            Wire<DASO_WIRE_FP32>::template load_smem<8>(st + L.v, i, v);
            Wire<DASO_WIRE_FP32>::template load_smem<8>(st + L.g, i, g);
#pragma unroll
            for (int q = 1; q < G; ++q) {
                float t[8];
                Wire<DASO_WIRE_FP32>::template load_smem<8>(st + L.g + uint32_t(q) * kPT * 4, i, t);
#pragma unroll
                for (int j = 0; j < 8; ++j) g[j] += t[j];                        // ascending local id (R18)
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const float d = fmaf(a.wd, x[j], g[j] * a.gscale);
                v[j] = fmaf(a.mu, v[j], d);
                x[j] = fmaf(-a.lr, v[j], x[j]);
            }
            if constexpr ((OPS & OP_MERGE) != 0) {
                float acc[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[j] = 0.f;
                for (int p = 0; p < a.P; ++p) {
                    float sv[8];
                    Wire<WIRE>::template load_smem<8>(st + L.slot + uint32_t(p) * kPT * wb, i, sv);
#pragma unroll
                    for (int j = 0; j < 8; ++j) acc[j] += sv[j] - x[j];
                }
#pragma unroll
                for (int j = 0; j < 8; ++j) x[j] = x[j] + acc[j] / a.den;
            }
            if (k >= NO && !mbar_wait(&oempty[o], uint32_t(((k / NO) - 1) & 1), pa.err)) break;
            if constexpr ((OPS & OP_NOX) == 0) Wire<DASO_WIRE_FP32>::template store_smem<8>(ob + L.ox, i, x);
            Wire<DASO_WIRE_FP32>::template store_smem<8>(ob + L.ov, i, v);
            if constexpr ((OPS & OP_PACK) != 0) Wire<WIRE>::template store_smem<8>(ob + L.opack, i, x);
#pragma unroll
            for (int j = 0; j < 8; ++j) bad |= !isfinite(x[j]);
            fence_async_smem();                                  // generic-proxy writes -> bulk stores
            __syncwarp();
            if ((tid & 31) == 0) mbar_arrive(&ofull[o]);
        }
        if (blockIdx.x == gridDim.x - 1) {                       // ragged tail through the register path
            __shared__ int s_tail_ok;                            // it reads peer g: wait for the start barrier
            if (tid == 0) {
                bool ok = true;
                for (int q = 0; q < G && ok; ++q) ok = wait_geq(pa.sig_me + q, pa.epoch, pa.err, pa.timeout_ns);
                s_tail_ok = ok;
            }
            asm volatile("bar.sync 1, %0;" ::"n"(kWsCompute) : "memory");   // the compute warps only
            if (s_tail_ok)
                for (int64_t e = ntiles * kPT + tid; e < a.n; e += kWsCompute) peer_body<OPS, WIRE, G, 1>(pa, e, bad);
        }
        if (a.flag != nullptr) {
            const unsigned any = __ballot_sync(0xffffffffu, bad);
            if (any != 0u && (tid & 31) == 0) atomicOr(a.flag, 1u);
        }
    }
    // 3. end barrier (the driver has waited for all its bulk stores: wait_group 0)
    if constexpr ((OPS & OP_NOX) == 0) {
        if (tid == kWsCompute) fence_proxy_async_global();
        end_barrier(pa, G);
    }
}

template <int OPS, int WIRE, int G>
int launch_peer_ws_t(const PeerArgs& pa, cudaStream_t s, int sms) {
    constexpr int wb = WIRE == DASO_WIRE_BF16 ? 2 : 4;
    const PeerTmaLayout L = peer_tma_layout(OPS, G, pa.a.P, wb);
    const int NO = peer_ws_out();
    const int budget = 210 * 1024 - NO * int(L.out_bytes);
    const int NS = int(std::min<int64_t>(8, (budget - 128) / L.in_bytes));
    if (NS < 2) return launch_peer_t<OPS, WIRE, G>(pa, s, sms);
    const size_t smem = size_t(NS) * L.in_bytes + size_t(NO) * L.out_bytes + 8 * size_t(NS + 2 * NO);
    static size_t attr = 0;
    if (smem > attr) {
        const cudaError_t e = cudaFuncSetAttribute(peer_ws_kernel<OPS, WIRE, G>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (e != cudaSuccess) return int(e);
        attr = smem;
    }
    const int grid = peer_tma_ctas() > 0 ? std::min(peer_tma_ctas(), sms) : std::max(1, sms - 16);
    peer_ws_kernel<OPS, WIRE, G><<<dim3(unsigned(grid)), dim3(kWsThreads), smem, s>>>(pa, NS, NO);
    return int(cudaGetLastError());
}

// ---- fused-mode blocking tail: Fig. 3 average + Fig. 4 re-publish in one kernel.
// After the blocking group all-gather each rank holds the P packed rows of its shard;
// x_shard = sum_i wire_f32(slot[i]) / P (ascending node order, R18; K4's arithmetic) is stored
// straight into every node peer's x over NVLink (the node all-gather), then the end barrier
// (end row of the signal arrays) makes every shard visible before any rank's next read of x.
// No start barrier: a peer's x[me-shard] is written only by this rank, and every peer finished
// its last read of x before it signalled the start barrier of this batch's OP_NOX node-tier
// kernel, which this rank's node-tier kernel waited for.
template <int WIRE, int G, int N>
__device__ __forceinline__ void avg_publish_body(const PeerArgs& pa, int64_t i, bool& bad) {
    const KernelArgs& a = pa.a;
    float x[N];
#pragma unroll
    for (int j = 0; j < N; ++j) x[j] = 0.f;
#pragma unroll 4
    for (int p = 0; p < a.P; ++p) {
        float s[N];
        Wire<WIRE>::template load<N>(a.slot, p * a.slot_stride + i, s);
#pragma unroll
        for (int j = 0; j < N; ++j) x[j] += s[j];
    }
#pragma unroll
    for (int j = 0; j < N; ++j) x[j] = x[j] / a.den;
#pragma unroll
    for (int q = 0; q < G; ++q) st_f32<N>(pa.xp[(pa.me + 1 + q) % G] + i, x);   // next peer first: spread links
#pragma unroll
    for (int j = 0; j < N; ++j) bad |= !isfinite(x[j]);
}

template <int WIRE, int G>
__global__ void __launch_bounds__(kPeerThreads) avg_publish_kernel(const PeerArgs pa) {
    bool bad = false;
    const int64_t n = pa.a.n;
    const int64_t nch = n / kPV;
    const int64_t stride = int64_t(gridDim.x) * kPeerThreads;
    for (int64_t c = int64_t(blockIdx.x) * kPeerThreads + threadIdx.x; c < nch; c += stride)
        avg_publish_body<WIRE, G, kPV>(pa, c * kPV, bad);
    if (blockIdx.x == gridDim.x - 1) {
        const int64_t i = nch * kPV + threadIdx.x;
        if (i < n) avg_publish_body<WIRE, G, 1>(pa, i, bad);
    }
    if (pa.a.flag != nullptr) {
        const unsigned any = __ballot_sync(0xffffffffu, bad);
        if (any != 0u && (threadIdx.x & 31) == 0) atomicOr(pa.a.flag, 1u);
    }
    end_barrier(pa, G);
}

// The same tail with the NVLink stores done by the bulk-copy engine: each 2048-parameter tile is
// averaged in registers (8 per thread), written to one of kAvgOut shared-memory output buffers, and
// one thread issues a bulk store of the buffer to every node peer (cp.async.bulk shared -> peer
// global).  Bulk stores reached 0.84 of the link in the probe against 0.79 for register stores.
// P (<= 4) is a template parameter so the next tile's P row loads are issued into registers before
// the current tile is stored (a first version without the prefetch was load-latency bound: 64 us
// for a 2x2 shard in the one-GPU virtual cluster at 18 % DRAM throughput, profiles/r02/one_s).
constexpr int kAvgOut = 4;

template <int WIRE, int G, int PT>
__global__ void __launch_bounds__(kPeerThreads) avg_publish_tma_kernel(const PeerArgs pa) {
    __shared__ __align__(128) float ob[kAvgOut][kPT];
    const KernelArgs& a = pa.a;
    const int tid = threadIdx.x;
    const int64_t ntiles = a.n / kPT;
    bool bad = false;
    float cur[PT][kPV];
    auto load_tile = [&](int64_t t, float (&dst)[PT][kPV]) {
#pragma unroll
        for (int p = 0; p < PT; ++p)
            Wire<WIRE>::template load<kPV>(a.slot, p * a.slot_stride + t * kPT + tid * kPV, dst[p]);
    };
    int64_t t = blockIdx.x;
    if (t < ntiles) load_tile(t, cur);
    for (int k = 0; t < ntiles; t += gridDim.x, ++k) {
        const int o = k % kAvgOut;
        const int64_t e0 = t * kPT;
        float nxt[PT][kPV];
        if (t + gridDim.x < ntiles) load_tile(t + gridDim.x, nxt);           // next tile's rows in flight
        float x[kPV];
#pragma unroll
        for (int j = 0; j < kPV; ++j) x[j] = 0.f;
#pragma unroll
        for (int p = 0; p < PT; ++p) {
#pragma unroll
            for (int j = 0; j < kPV; ++j) x[j] += cur[p][j];                 // ascending node order (R18)
        }
#pragma unroll
        for (int j = 0; j < kPV; ++j) {
            x[j] = x[j] / a.den;
            bad |= !isfinite(x[j]);
        }
        if (tid == 0 && k >= kAvgOut) bulk_wait_read<kAvgOut - 1>();        // buffer o has been read
        __syncthreads();
        Wire<DASO_WIRE_FP32>::template store_smem<kPV>(ob[o], tid * kPV, x);
        fence_async_smem();                                                  // generic writes -> bulk stores
        __syncthreads();
        if (tid == 0) {
#pragma unroll
            for (int q = 0; q < G; ++q) bulk_s2g(pa.xp[(pa.me + 1 + q) % G] + e0, ob[o], kPT * 4);
            bulk_commit();
        }
#pragma unroll
        for (int p = 0; p < PT; ++p) {
#pragma unroll
            for (int j = 0; j < kPV; ++j) cur[p][j] = nxt[p][j];
        }
    }
    if (tid == 0) bulk_wait_all();
    if (blockIdx.x == gridDim.x - 1)                                         // ragged tail (< one tile)
        for (int64_t e = ntiles * kPT + tid; e < a.n; e += kPeerThreads) avg_publish_body<WIRE, G, 1>(pa, e, bad);
    if (a.flag != nullptr) {
        const unsigned any = __ballot_sync(0xffffffffu, bad);
        if (any != 0u && (tid & 31) == 0) atomicOr(a.flag, 1u);
    }
    if (tid == 0) fence_proxy_async_global();
    end_barrier(pa, G);
}

// DASO_AVG_PUBLISH=ldg|tma (default tma); the TMA form needs 16-byte aligned peer shards
int avg_publish_path() {
    const char* e = getenv("DASO_AVG_PUBLISH");
    return (e && strcmp(e, "ldg") == 0) ? 0 : 1;
}

template <int WIRE, int G>
int launch_avg_publish_t(const PeerArgs& pa, cudaStream_t s, int sms) {
    uintptr_t al = reinterpret_cast<uintptr_t>(pa.a.slot);
    for (int q = 0; q < G; ++q) al |= reinterpret_cast<uintptr_t>(pa.xp[q]);
    if (avg_publish_path() == 1 && (al & 15u) == 0 && pa.a.n >= kPT && pa.a.P >= 1 && pa.a.P <= 4) {
        // two CTAs per SM on SMs - 16 (the side-stream exchange keeps free SMs, as for the node tier)
        const dim3 grid(unsigned(2 * std::max(1, sms - 16)));
        switch (pa.a.P) {
            case 1: avg_publish_tma_kernel<WIRE, G, 1><<<grid, kPeerThreads, 0, s>>>(pa); break;
            case 2: avg_publish_tma_kernel<WIRE, G, 2><<<grid, kPeerThreads, 0, s>>>(pa); break;
            case 3: avg_publish_tma_kernel<WIRE, G, 3><<<grid, kPeerThreads, 0, s>>>(pa); break;
            default: avg_publish_tma_kernel<WIRE, G, 4><<<grid, kPeerThreads, 0, s>>>(pa); break;
        }
        return int(cudaGetLastError());
    }
    const int64_t nch = pa.a.n / kPV;
    int64_t blocks = (nch + kPeerThreads - 1) / kPeerThreads;
    blocks = std::max<int64_t>(1, std::min<int64_t>(blocks, int64_t(sms) * peer_blocks_per_sm()));
    avg_publish_kernel<WIRE, G><<<dim3(unsigned(blocks)), dim3(kPeerThreads), 0, s>>>(pa);
    return int(cudaGetLastError());
}

template <int WIRE>
int dispatch_avg_publish(const PeerArgs& pa, cudaStream_t s, int sms) {
    switch (pa.G) {
        case 1: return launch_avg_publish_t<WIRE, 1>(pa, s, sms);
        case 2: return launch_avg_publish_t<WIRE, 2>(pa, s, sms);
        case 3: return launch_avg_publish_t<WIRE, 3>(pa, s, sms);
        case 4: return launch_avg_publish_t<WIRE, 4>(pa, s, sms);
        case 5: return launch_avg_publish_t<WIRE, 5>(pa, s, sms);
        case 6: return launch_avg_publish_t<WIRE, 6>(pa, s, sms);
        case 7: return launch_avg_publish_t<WIRE, 7>(pa, s, sms);
        case 8: return launch_avg_publish_t<WIRE, 8>(pa, s, sms);
        default: return int(cudaErrorInvalidValue);
    }
}

// Peer data path under daso_kernel_impl(2) "auto" (DASO_PEER=ws|tma|ldg).
int peer_path() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("DASO_PEER");
        v = (e && strcmp(e, "ldg") == 0) ? 0 : (e && strcmp(e, "tma") == 0) ? 1 : 2;
    }
    return v;
}

uintptr_t push_bits(const KernelArgs& a) {
    uintptr_t b = 0;
    for (int k = 0; k < a.npush; ++k) b |= reinterpret_cast<uintptr_t>(a.push[k]);
    return b;
}

template <int OPS, int WIRE, int G>
int launch_peer_any(const PeerArgs& pa, cudaStream_t s, int sms) {
    const bool al = ((reinterpret_cast<uintptr_t>(pa.a.x) | reinterpret_cast<uintptr_t>(pa.a.v) |
                      reinterpret_cast<uintptr_t>(pa.a.pack_out) | reinterpret_cast<uintptr_t>(pa.a.slot) |
                      push_bits(pa.a)) & 15u) == 0;
    // TMA unless the register path is forced (daso_kernel_impl(0))
    const int impl = current_kernel_impl();   // 0 register, 1 TMA, 2 auto (DASO_PEER, default ws)
    const int path = impl == 2 ? peer_path() : impl == 1 ? 1 : 0;
    if (path == 2 && al && pa.a.n >= kPT) return launch_peer_ws_t<OPS, WIRE, G>(pa, s, sms);
    if (path == 1 && al && pa.a.n >= kPT) return launch_peer_tma_t<OPS, WIRE, G>(pa, s, sms);
    return launch_peer_t<OPS, WIRE, G>(pa, s, sms);
}

template <int OPS, int WIRE>
int dispatch_g(const PeerArgs& pa, cudaStream_t s, int sms) {
    switch (pa.G) {
        case 1: return launch_peer_any<OPS, WIRE, 1>(pa, s, sms);
        case 2: return launch_peer_any<OPS, WIRE, 2>(pa, s, sms);
        case 3: return launch_peer_any<OPS, WIRE, 3>(pa, s, sms);
        case 4: return launch_peer_any<OPS, WIRE, 4>(pa, s, sms);
        case 5: return launch_peer_any<OPS, WIRE, 5>(pa, s, sms);
        case 6: return launch_peer_any<OPS, WIRE, 6>(pa, s, sms);
        case 7: return launch_peer_any<OPS, WIRE, 7>(pa, s, sms);
        case 8: return launch_peer_any<OPS, WIRE, 8>(pa, s, sms);
        default: return int(cudaErrorInvalidValue);
    }
}

template <int WIRE>
int dispatch_peer(int ops, const PeerArgs& pa, cudaStream_t s, int sms) {
    switch (ops) {
        case OP_UPDATE: return dispatch_g<OP_UPDATE, WIRE>(pa, s, sms);
        case OP_UPDATE | OP_PACK: return dispatch_g<OP_UPDATE | OP_PACK, WIRE>(pa, s, sms);
        case OP_UPDATE | OP_MERGE: return dispatch_g<OP_UPDATE | OP_MERGE, WIRE>(pa, s, sms);
        case OP_UPDATE | OP_MERGE | OP_PACK: return dispatch_g<OP_UPDATE | OP_MERGE | OP_PACK, WIRE>(pa, s, sms);
        case OP_UPDATE | OP_PACK | OP_NOX: return dispatch_g<OP_UPDATE | OP_PACK | OP_NOX, WIRE>(pa, s, sms);
        case OP_UPDATE | OP_PACK | OP_NOX | OP_PUSH:
            return dispatch_g<OP_UPDATE | OP_PACK | OP_NOX | OP_PUSH, WIRE>(pa, s, sms);
        case OP_UPDATE | OP_MERGE | OP_PACK | OP_NOX:
            return dispatch_g<OP_UPDATE | OP_MERGE | OP_PACK | OP_NOX, WIRE>(pa, s, sms);
        default: return int(cudaErrorInvalidValue);
    }
}


}  // namespace

int launch_peer(int ops, int wire, const PeerArgs& pa, void* stream) {
    if (pa.G < 1 || pa.G > kMaxPeers) return int(cudaErrorInvalidValue);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (wire == DASO_WIRE_BF16) return dispatch_peer<DASO_WIRE_BF16>(ops, pa, s, sms);
    if (wire == DASO_WIRE_FP32) return dispatch_peer<DASO_WIRE_FP32>(ops, pa, s, sms);
    return int(cudaErrorInvalidValue);
}

int launch_avg_publish(int wire, const PeerArgs& pa, void* stream) {
    if (pa.G < 1 || pa.G > kMaxPeers) return int(cudaErrorInvalidValue);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (wire == DASO_WIRE_BF16) return dispatch_avg_publish<DASO_WIRE_BF16>(pa, s, sms);
    if (wire == DASO_WIRE_FP32) return dispatch_avg_publish<DASO_WIRE_FP32>(pa, s, sms);
    return int(cudaErrorInvalidValue);
}

}  // namespace daso
