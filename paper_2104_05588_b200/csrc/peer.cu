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
// Each rank is its own GPU (one process per GPU), so the spin-waits never wait on a
// kernel of the same GPU; the grid leaves room on every SM for the side-stream NCCL
// exchange kernels to run concurrently.
#include <cuda_runtime.h>

#include "daso_internal.h"
#include "device_common.cuh"

namespace daso {
namespace {
using namespace dev;

constexpr int kPeerThreads = 256;
constexpr int kPV = 4;   // parameters per thread per iteration (one 128-bit access per stream)

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Spin until *p >= v.  A peer that never arrives (crashed process, protocol bug) must not
// hang the GPU: after kBarrierTimeoutNs the wait gives up and raises bit 1 of the flag,
// which daso_check_finite / the next step report as an error.
constexpr unsigned long long kBarrierTimeoutNs = 20ull * 1000 * 1000 * 1000;

__device__ __forceinline__ void wait_geq(const unsigned long long* p, unsigned long long v, uint32_t* flag) {
    if (ld_acquire_sys(p) >= v) return;
    const unsigned long long t0 = globaltimer_ns();
    while (ld_acquire_sys(p) < v) {
        if (globaltimer_ns() - t0 > kBarrierTimeoutNs) {
            if (flag) atomicOr(flag, 2u);
            return;
        }
        __nanosleep(64);
    }
}

template <int OPS, int WIRE, int N>
__device__ __forceinline__ void peer_body(const PeerArgs& pa, int64_t i, bool& bad) {
    const KernelArgs& a = pa.a;
    const int G = pa.G;
    float x[N], v[N], g[N];
    ld_f32<N>(a.x + i, x);
    ld_f32<N>(a.v + i, v);
    float gq[kMaxPeers][N];
#pragma unroll
    for (int q = 0; q < kMaxPeers; ++q)
        if (q < G) ld_f32<N>(pa.gp[q] + i, gq[q]);
#pragma unroll
    for (int j = 0; j < N; ++j) g[j] = gq[0][j];
#pragma unroll
    for (int q = 1; q < kMaxPeers; ++q)
        if (q < G) {
#pragma unroll
            for (int j = 0; j < N; ++j) g[j] += gq[q][j];
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
#pragma unroll
    for (int q = 0; q < kMaxPeers; ++q)
        if (q < G) st_f32<N>(pa.xp[q] + i, x);
#pragma unroll
    for (int j = 0; j < N; ++j) bad |= !isfinite(x[j]);
    if constexpr ((OPS & OP_PACK) != 0) Wire<WIRE>::template store<N>(a.pack_out, i, x);
}

template <int OPS, int WIRE>
__global__ void __launch_bounds__(kPeerThreads) peer_kernel(const PeerArgs pa) {
    const int G = pa.G;
    // 1. start barrier
    if (blockIdx.x == 0 && threadIdx.x < G) {
        __threadfence_system();
        st_release_sys(pa.sig_peer[threadIdx.x] + pa.me, pa.epoch);
    }
    if (threadIdx.x == 0)
        for (int q = 0; q < G; ++q) wait_geq(pa.sig_me + q, pa.epoch, pa.err);
    __syncthreads();
    // 2. shard update over NVLink
    bool bad = false;
    const int64_t n = pa.a.n;
    const int64_t nch = n / kPV;
    const int64_t stride = int64_t(gridDim.x) * kPeerThreads;
    for (int64_t c = int64_t(blockIdx.x) * kPeerThreads + threadIdx.x; c < nch; c += stride)
        peer_body<OPS, WIRE, kPV>(pa, c * kPV, bad);
    if (blockIdx.x == gridDim.x - 1) {
        const int64_t i = nch * kPV + threadIdx.x;
        if (i < n) peer_body<OPS, WIRE, 1>(pa, i, bad);
    }
    if (pa.a.flag != nullptr) {
        const unsigned any = __ballot_sync(0xffffffffu, bad);
        if (any != 0u && (threadIdx.x & 31) == 0) atomicOr(pa.a.flag, 1u);
    }
    // 3. end barrier
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        const unsigned prev = atomicAdd(pa.done, 1u);
        if (prev == gridDim.x - 1) {
            *reinterpret_cast<volatile unsigned*>(pa.done) = 0u;
            __threadfence_system();
            for (int q = 0; q < G; ++q) st_release_sys(pa.sig_peer[q] + G + pa.me, pa.epoch);
            for (int q = 0; q < G; ++q) wait_geq(pa.sig_me + G + q, pa.epoch, pa.err);
        }
    }
}

template <int OPS, int WIRE>
int launch_peer_t(const PeerArgs& pa, cudaStream_t s, int sms) {
    const int64_t nch = pa.a.n / kPV;
    int64_t blocks = (nch + kPeerThreads - 1) / kPeerThreads;
    blocks = std::max<int64_t>(1, std::min<int64_t>(blocks, int64_t(sms) * 2));
    peer_kernel<OPS, WIRE><<<dim3(unsigned(blocks)), dim3(kPeerThreads), 0, s>>>(pa);
    return int(cudaGetLastError());
}

template <int WIRE>
int dispatch_peer(int ops, const PeerArgs& pa, cudaStream_t s, int sms) {
    switch (ops) {
        case OP_UPDATE: return launch_peer_t<OP_UPDATE, WIRE>(pa, s, sms);
        case OP_UPDATE | OP_PACK: return launch_peer_t<OP_UPDATE | OP_PACK, WIRE>(pa, s, sms);
        case OP_UPDATE | OP_MERGE: return launch_peer_t<OP_UPDATE | OP_MERGE, WIRE>(pa, s, sms);
        case OP_UPDATE | OP_MERGE | OP_PACK: return launch_peer_t<OP_UPDATE | OP_MERGE | OP_PACK, WIRE>(pa, s, sms);
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

}  // namespace daso
