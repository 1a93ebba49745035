// Fused, HBM-bound elementwise kernels of the DASO hot path for sm_100a.
//
//   K1  update          d = g*gscale + wd*x ; v = mu*v + d ; x = x - lr*v         (App. Eq. 1)
//   K2  update + pack   ... ; pack_out = wire(x)                                  ("buffer packaging", P:162 bf16)
//   K3  update + merge  ... ; x = x + sum_i (wire_f32(slot[i]) - x) / (2S + P)    (Eq. (1), delta form)
//   K4  average         x = sum_i wire_f32(slot[i]) / P                           (Fig. 3; blocking)
//   pack-only, merge-only (+pack): the split-API pieces of the same arithmetic.
//
// Design: one templated body, instantiated per op set and wire
// type; each thread moves 8 parameters per iteration (2 x 128-bit loads per fp32
// stream, 1 x 128-bit load per bf16 row), evict-first (.cs) loads/stores since every
// byte is touched once per step and the working set (>= 12 B/param) exceeds L2;
// one chunk per thread over a grid of n/2048 CTAs (tail in the last CTA); the optional
// non-finite flag is a warp ballot + one atomicOr per warp.  No shared memory or
// tensor cores: there is no reuse and no contraction.
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include <cstdlib>
#include <cstring>

#include "daso_internal.h"
#include "device_common.cuh"

namespace daso {
namespace {

using namespace dev;

// ----------------------------------------------------------------- fused body
// PN > 0: the number of slot rows P is a compile-time constant and the P row loads of a merge are
// issued with the x, v, g loads at the top (the runtime-P loop below cannot hoist them above the v
// store, since the pointers may alias, so they would start a second round trip to HBM).
template <int OPS, int WIRE, int N, int PN = 0>
__device__ __forceinline__ void body(const KernelArgs& a, int64_t i, bool& bad) {
    float x[N];
    float sp[PN > 0 ? PN : 1][N];
    if constexpr (PN > 0 && (OPS & OP_MERGE) != 0) {
#pragma unroll
        for (int p = 0; p < PN; ++p) Wire<WIRE>::template load<N>(a.slot, p * a.slot_stride + i, sp[p]);
    }
    if constexpr ((OPS & (OP_UPDATE | OP_MERGE | OP_PACK)) != 0) ld_f32<N>(a.x + i, x);
    if constexpr ((OPS & OP_UPDATE) != 0) {
        float v[N], g[N];
        ld_f32<N>(a.v + i, v);
        ld_f32<N>(a.g + i, g);
#pragma unroll
        for (int j = 0; j < N; ++j) {
            const float d = fmaf(a.wd, x[j], g[j] * a.gscale);   // g/G + wd*x   (R4: fp32 node sum x 1/G)
            v[j] = fmaf(a.mu, v[j], d);                          // v = mu v + d
            x[j] = fmaf(-a.lr, v[j], x[j]);                      // x = x - lr v
        }
        st_f32<N>(a.v + i, v);
    }
    if constexpr ((OPS & OP_MERGE) != 0) {
        float acc[N];
#pragma unroll
        for (int j = 0; j < N; ++j) acc[j] = 0.f;
        if constexpr (PN > 0) {
#pragma unroll
            for (int p = 0; p < PN; ++p) {                       // ascending node order (R18)
#pragma unroll
                for (int j = 0; j < N; ++j) acc[j] += sp[p][j] - x[j];
            }
        } else {
#pragma unroll 4
            for (int p = 0; p < a.P; ++p) {                      // ascending node order (R18)
                float s[N];
                Wire<WIRE>::template load<N>(a.slot, p * a.slot_stride + i, s);
#pragma unroll
                for (int j = 0; j < N; ++j) acc[j] += s[j] - x[j];
            }
        }
#pragma unroll
        for (int j = 0; j < N; ++j) x[j] = x[j] + acc[j] / a.den;   // (2S x + sum s)/(2S+P), delta form
    }
    if constexpr ((OPS & OP_AVERAGE) != 0) {
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
    }
    if constexpr ((OPS & (OP_UPDATE | OP_MERGE | OP_AVERAGE)) != 0) {
        st_f32<N>(a.x + i, x);
#pragma unroll
        for (int j = 0; j < N; ++j) bad |= !isfinite(x[j]);
    }
    if constexpr ((OPS & OP_PACK) != 0) {
        Wire<WIRE>::template store<N>(a.pack_out, i, x);
        if constexpr ((OPS & OP_PUSH) != 0) {   // group members' slots (a separate instantiation: the
#pragma unroll                                        // push code costs the plain pack kernels registers)
            for (int k = 0; k < kMaxPush; ++k)
                if (k < a.npush) Wire<WIRE>::template store<N>(a.push[k], i, x);
        }
    }
}

// Eight parameters per thread for every op set.  Measured alternatives (profiles/r01): 32 per
// thread for the light kernels (average, pack) was slower (K4 41 -> 57 us, pack 23 -> 37 us); a
// K4 with P templated and two chunks per thread, all 2P row loads in flight before the sums, ran
// 42.0 vs 42.4 us at P = 2 and 57.6 vs 53.2 us at P = 4, and a TMA-staged K4 (bulk row loads, bulk x
// store, persistent CTAs) 97.4 us (profiles/r02/k4_variants.txt); and
// issuing the two 128-bit loads of a stream from an array loop instead of two named loads cost K1
// 9 % (75 -> 82 us, same box, A/B in one run): ptxas schedules the explicit form better.
template <int OPS, int WIRE, int PN = 0>
__global__ void __launch_bounds__(kThreads) fused_kernel(const KernelArgs a) {
    const int64_t nchunks = a.n / kVec;
    const int64_t stride = int64_t(gridDim.x) * kThreads;
    bool bad = false;
    for (int64_t c = int64_t(blockIdx.x) * kThreads + threadIdx.x; c < nchunks; c += stride)
        body<OPS, WIRE, kVec, PN>(a, c * kVec, bad);
    if (blockIdx.x == gridDim.x - 1) {                           // ragged tail (< 8 elements)
        const int64_t i = nchunks * kVec + threadIdx.x;
        if (i < a.n) body<OPS, WIRE, 1>(a, i, bad);
    }
    if (a.flag != nullptr) {
        const unsigned any = __ballot_sync(0xffffffffu, bad);
        if (any != 0u && (threadIdx.x & 31) == 0) atomicOr(a.flag, 1u);
    }
}


// K4 (blocking average) specialised on P <= 4: two 8-parameter chunks per thread, a CTA-width
// apart (each chunk's warp accesses stay coalesced), with all 2P row loads in flight before the
// sums.  tools/k4_variants.cu at P = 2 (profiles/r02/one_n/k4_variants*.jsonl): 32.8 us vs 36.8 us for one
// chunk per thread; two contiguous chunks per thread ran 39 us, 512-thread CTAs 36.9, persistent
// grids 35-42.  Same arithmetic and order as body<OP_AVERAGE> (x = ((0 + s_0) + s_1 ...) / den).
constexpr int kAvgU = 2;
template <int WIRE, int P>
__global__ void __launch_bounds__(kThreads) average_kernel(const KernelArgs a) {
    const int64_t nchunks = a.n / kVec;
    const int64_t base = int64_t(blockIdx.x) * kThreads * kAvgU;
    bool bad = false;
    if (base + int64_t(kThreads) * kAvgU <= nchunks) {
        float s[kAvgU][P][kVec];
#pragma unroll
        for (int u = 0; u < kAvgU; ++u) {
#pragma unroll
            for (int p = 0; p < P; ++p)
                Wire<WIRE>::template load<kVec>(a.slot, p * a.slot_stride + (base + u * kThreads + threadIdx.x) * kVec,
                                                s[u][p]);
        }
#pragma unroll
        for (int u = 0; u < kAvgU; ++u) {
            float x[kVec];
#pragma unroll
            for (int j = 0; j < kVec; ++j) x[j] = 0.f;
#pragma unroll
            for (int p = 0; p < P; ++p) {
#pragma unroll
                for (int j = 0; j < kVec; ++j) x[j] += s[u][p][j];          // ascending node order (R18)
            }
#pragma unroll
            for (int j = 0; j < kVec; ++j) x[j] = x[j] / a.den;
            st_f32<kVec>(a.x + (base + u * kThreads + threadIdx.x) * kVec, x);
#pragma unroll
            for (int j = 0; j < kVec; ++j) bad |= !isfinite(x[j]);
        }
    } else {
        for (int64_t c = base + threadIdx.x; c < nchunks; c += kThreads) body<OP_AVERAGE, WIRE, kVec>(a, c * kVec, bad);
    }
    if (blockIdx.x == gridDim.x - 1) {                           // ragged tail (< 8 elements)
        const int64_t i = nchunks * kVec + threadIdx.x;
        if (i < a.n) body<OP_AVERAGE, WIRE, 1>(a, i, bad);
    }
    if (a.flag != nullptr) {
        const unsigned any = __ballot_sync(0xffffffffu, bad);
        if (any != 0u && (threadIdx.x & 31) == 0) atomicOr(a.flag, 1u);
    }
}

// ----------------------------------------------------------------- TMA-staged variant
// The same K1/K2/K3 arithmetic with the streams staged through shared memory by the
// bulk-copy engine (cp.async.bulk, 1-D TMA): one persistent CTA per SM walks its tiles
// (tile = blockIdx.x + k * gridDim.x) through an NS-deep ring of stages; one elected
// thread issues the global->shared copies (completion counted in bytes on an mbarrier)
// and the shared->global stores of x, v and the packed row (bulk_group), all threads
// compute from shared memory.  NS-1 tiles of loads are in flight per SM while one is
// computed.  Ragged tail (< kTile elements) falls back to the register path.
constexpr int kTile = 2048;          // parameters per tile: 8 per thread
constexpr int kTmaThreads = 256;

struct TmaLayout {   // byte offsets inside one stage
    uint32_t x, v, g, slot, pack, bytes;
};
__host__ __device__ inline TmaLayout tma_layout(int ops, int P, int wb) {
    TmaLayout L{};
    uint32_t o = 0;
    L.x = o; o += kTile * 4;
    L.v = o; o += kTile * 4;
    L.g = o; o += kTile * 4;
    L.slot = o; if (ops & OP_MERGE) o += uint32_t(P) * kTile * wb;
    L.pack = o; if (ops & OP_PACK) o += kTile * wb;
    L.bytes = (o + 127) / 128 * 128;
    return L;
}

template <int OPS, int WIRE>
__global__ void __launch_bounds__(kTmaThreads, 1) tma_kernel(const KernelArgs a, int NS) {
    extern __shared__ __align__(128) unsigned char smem[];
    constexpr int wb = WIRE == DASO_WIRE_BF16 ? 2 : 4;
    const TmaLayout L = tma_layout(OPS, a.P, wb);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + size_t(NS) * L.bytes);
    const int64_t ntiles = a.n / kTile;
    const int64_t my = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const bool leader = threadIdx.x == 0;
    if (leader) {
        for (int s = 0; s < NS; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    auto issue_load = [&](int64_t k) {
        const int s = int(k % NS);
        unsigned char* st = smem + size_t(s) * L.bytes;
        const int64_t e0 = (int64_t(blockIdx.x) + k * gridDim.x) * kTile;
        uint32_t tx = 3u * kTile * 4u;
        if constexpr ((OPS & OP_MERGE) != 0) tx += uint32_t(a.P) * kTile * wb;
        mbar_expect_tx(&full[s], tx);
        bulk_g2s(st + L.x, a.x + e0, kTile * 4, &full[s]);
        bulk_g2s(st + L.v, a.v + e0, kTile * 4, &full[s]);
        bulk_g2s(st + L.g, a.g + e0, kTile * 4, &full[s]);
        if constexpr ((OPS & OP_MERGE) != 0) {
            for (int p = 0; p < a.P; ++p)
                bulk_g2s(st + L.slot + uint32_t(p) * kTile * wb,
                         static_cast<const unsigned char*>(a.slot) + (p * a.slot_stride + e0) * wb, kTile * wb,
                         &full[s]);
        }
    };

    if (leader)
        for (int64_t k = 0; k < my && k < NS; ++k) issue_load(k);

    bool bad = false;
    for (int64_t k = 0; k < my; ++k) {
        const int s = int(k % NS);
        unsigned char* st = smem + size_t(s) * L.bytes;
        if (!mbar_wait(&full[s], uint32_t((k / NS) & 1), a.err)) break;   // timed out: bit 2 raised, stop
        const int i = threadIdx.x * kVec;
        float* xs = reinterpret_cast<float*>(st + L.x) + i;
        float* vs = reinterpret_cast<float*>(st + L.v) + i;
        const float* gs = reinterpret_cast<const float*>(st + L.g) + i;
        float x[kVec], v[kVec], g[kVec];
#pragma unroll
        for (int j = 0; j < kVec; j += 4) {
            float4 a4 = *reinterpret_cast<float4*>(xs + j), b4 = *reinterpret_cast<float4*>(vs + j),
                   c4 = *reinterpret_cast<const float4*>(gs + j);
            x[j] = a4.x; x[j + 1] = a4.y; x[j + 2] = a4.z; x[j + 3] = a4.w;
            v[j] = b4.x; v[j + 1] = b4.y; v[j + 2] = b4.z; v[j + 3] = b4.w;
            g[j] = c4.x; g[j + 1] = c4.y; g[j + 2] = c4.z; g[j + 3] = c4.w;
        }
#pragma unroll
        for (int j = 0; j < kVec; ++j) {
            const float d = fmaf(a.wd, x[j], g[j] * a.gscale);
            v[j] = fmaf(a.mu, v[j], d);
            x[j] = fmaf(-a.lr, v[j], x[j]);
        }
        if constexpr ((OPS & OP_MERGE) != 0) {
            float acc[kVec];
#pragma unroll
            for (int j = 0; j < kVec; ++j) acc[j] = 0.f;
            for (int p = 0; p < a.P; ++p) {
                float sv[kVec];
                Wire<WIRE>::template load_smem<kVec>(st + L.slot + uint32_t(p) * kTile * wb, i, sv);
#pragma unroll
                for (int j = 0; j < kVec; ++j) acc[j] += sv[j] - x[j];
            }
#pragma unroll
            for (int j = 0; j < kVec; ++j) x[j] = x[j] + acc[j] / a.den;
        }
#pragma unroll
        for (int j = 0; j < kVec; j += 4) {
            *reinterpret_cast<float4*>(xs + j) = make_float4(x[j], x[j + 1], x[j + 2], x[j + 3]);
            *reinterpret_cast<float4*>(vs + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        }
#pragma unroll
        for (int j = 0; j < kVec; ++j) bad |= !isfinite(x[j]);
        if constexpr ((OPS & OP_PACK) != 0) Wire<WIRE>::template store_smem<kVec>(st + L.pack, i, x);
        fence_async_smem();
        __syncthreads();
        if (leader) {
            const int64_t e0 = (int64_t(blockIdx.x) + k * gridDim.x) * kTile;
            bulk_s2g(a.x + e0, st + L.x, kTile * 4);
            bulk_s2g(a.v + e0, st + L.v, kTile * 4);
            if constexpr ((OPS & OP_PACK) != 0)
                bulk_s2g(static_cast<unsigned char*>(a.pack_out) + e0 * wb, st + L.pack, kTile * wb);
            bulk_commit();
            if (k >= 1 && k - 1 + NS < my) {   // stage of tile k-1 is free once its stores have read it
                bulk_wait_read<1>();
                issue_load(k - 1 + NS);
            }
        }
    }
    if (leader) bulk_wait_all();
    if (blockIdx.x == gridDim.x - 1) {   // ragged tail through the register path
        for (int64_t e = ntiles * kTile + threadIdx.x; e < a.n; e += blockDim.x) body<OPS, WIRE, 1>(a, e, bad);
    }
    if (a.flag != nullptr) {
        const unsigned any = __ballot_sync(0xffffffffu, bad);
        if (any != 0u && (threadIdx.x & 31) == 0) atomicOr(a.flag, 1u);
    }
}

// ----------------------------------------------------------------- launch config
struct DevInfo {
    int sms = 0;
};

int sm_count() {
    static int cached_dev = -1, cached_sms = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev != cached_dev) {
        cudaDeviceGetAttribute(&cached_sms, cudaDevAttrMultiProcessorCount, dev);
        cached_dev = dev;
    }
    return cached_sms > 0 ? cached_sms : 148;
}

template <int OPS, int WIRE, int PN = 0>
int launch_t(const KernelArgs& a, cudaStream_t s) {
    // One 8-parameter chunk per thread ("one-shot" grid): measured 95% of the copy
    // peak for K1 on B200 vs 82% for a persistent grid-stride grid of SMs x occupancy
    // (tools/k1_variants.cu); the grid-stride loop only engages past 2^31 blocks.
    const int64_t nchunks = a.n / kVec;
    int64_t blocks = (nchunks + kThreads - 1) / kThreads;
    if (blocks > 0x7fffffffLL) blocks = 0x7fffffffLL;
    if (blocks < 1) blocks = 1;
    fused_kernel<OPS, WIRE, PN><<<dim3(unsigned(blocks)), dim3(kThreads), 0, s>>>(a);
    return int(cudaGetLastError());
}

// K3 with the P slot-row loads issued up front for P <= 4 (the 2x4 / 4x2 / 2x2 topologies)
template <int OPS, int WIRE>
int launch_merge(const KernelArgs& a, cudaStream_t s) {
    switch (a.P) {
        case 1: return launch_t<OPS, WIRE, 1>(a, s);
        case 2: return launch_t<OPS, WIRE, 2>(a, s);
        case 3: return launch_t<OPS, WIRE, 3>(a, s);
        case 4: return launch_t<OPS, WIRE, 4>(a, s);
        default: return launch_t<OPS, WIRE>(a, s);
    }
}

template <int WIRE, int P>
int launch_average(const KernelArgs& a, cudaStream_t s) {
    const int64_t per = int64_t(kThreads) * kAvgU;
    int64_t blocks = (a.n / kVec + per - 1) / per;
    if (blocks > 0x7fffffffLL) return launch_t<OP_AVERAGE, WIRE>(a, s);
    if (blocks < 1) blocks = 1;
    average_kernel<WIRE, P><<<dim3(unsigned(blocks)), dim3(kThreads), 0, s>>>(a);
    return int(cudaGetLastError());
}

// 0 = register (LDG) path everywhere, 1 = TMA-staged path everywhere, 2 = auto (default):
// the measured-faster path per kernel — register path for the local fused kernels (one-shot
// grid: ~100% of the copy peak), TMA for the NVLink peer kernel (0.77 vs 0.64 of the link
// peak on B200, profiles/r01).  Default from DASO_KERNEL=ldg|tma|auto.
int g_impl = -1;

int kernel_impl() {
    if (g_impl < 0) {
        const char* e = getenv("DASO_KERNEL");
        g_impl = (e && strcmp(e, "tma") == 0) ? 1 : (e && strcmp(e, "ldg") == 0) ? 0 : 2;
    }
    return g_impl;
}

template <int OPS, int WIRE>
int launch_tma(const KernelArgs& a, cudaStream_t s) {
    constexpr int wb = WIRE == DASO_WIRE_BF16 ? 2 : 4;
    const TmaLayout L = tma_layout(OPS, a.P, wb);
    const int budget = 200 * 1024;
    int NS = int(std::min<int64_t>(8, (budget - 64) / L.bytes));
    if (NS < 2) return launch_t<OPS, WIRE>(a, s);
    const size_t smem = size_t(NS) * L.bytes + 8 * size_t(NS);
    static size_t attr = 0;   // opt-in limit set so far
    if (smem > attr) {
        const cudaError_t e = cudaFuncSetAttribute(tma_kernel<OPS, WIRE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   int(smem));
        if (e != cudaSuccess) return int(e);
        attr = smem;
    }
    tma_kernel<OPS, WIRE><<<dim3(unsigned(sm_count())), dim3(kTmaThreads), smem, s>>>(a, NS);
    return int(cudaGetLastError());
}

bool tma_ok(const KernelArgs& a, int wb) {
    auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
    return a.n >= kTile && al(a.x) && al(a.v) && al(a.g) && (a.pack_out == nullptr || al(a.pack_out)) &&
           (a.slot == nullptr || (al(a.slot) && (a.slot_stride * wb) % 16 == 0)) && a.P <= 16;
}

template <int WIRE>
int dispatch(int ops, const KernelArgs& a, cudaStream_t s) {
    constexpr int wb = WIRE == DASO_WIRE_BF16 ? 2 : 4;
    if (kernel_impl() == 1 && tma_ok(a, wb) && a.npush == 0) {
        switch (ops) {
            case OP_UPDATE: return launch_tma<OP_UPDATE, WIRE>(a, s);
            case OP_UPDATE | OP_PACK: return launch_tma<OP_UPDATE | OP_PACK, WIRE>(a, s);
            case OP_UPDATE | OP_MERGE: return launch_tma<OP_UPDATE | OP_MERGE, WIRE>(a, s);
            case OP_UPDATE | OP_MERGE | OP_PACK: return launch_tma<OP_UPDATE | OP_MERGE | OP_PACK, WIRE>(a, s);
            default: break;
        }
    }
    switch (ops) {
        case OP_UPDATE: return launch_t<OP_UPDATE, WIRE>(a, s);
        case OP_UPDATE | OP_PACK: return launch_t<OP_UPDATE | OP_PACK, WIRE>(a, s);
        case OP_UPDATE | OP_PACK | OP_PUSH: return launch_t<OP_UPDATE | OP_PACK | OP_PUSH, WIRE>(a, s);
        case OP_UPDATE | OP_MERGE: return launch_merge<OP_UPDATE | OP_MERGE, WIRE>(a, s);
        case OP_UPDATE | OP_MERGE | OP_PACK: return launch_merge<OP_UPDATE | OP_MERGE | OP_PACK, WIRE>(a, s);
        case OP_MERGE: return launch_t<OP_MERGE, WIRE>(a, s);
        case OP_MERGE | OP_PACK: return launch_t<OP_MERGE | OP_PACK, WIRE>(a, s);
        case OP_AVERAGE:
            switch (a.P) {
                case 1: return launch_average<WIRE, 1>(a, s);
                case 2: return launch_average<WIRE, 2>(a, s);
                case 3: return launch_average<WIRE, 3>(a, s);
                case 4: return launch_average<WIRE, 4>(a, s);
                default: return launch_t<OP_AVERAGE, WIRE>(a, s);
            }
        case OP_PACK: return launch_t<OP_PACK, WIRE>(a, s);
        default: return int(cudaErrorInvalidValue);
    }
}

// ----------------------------------------------------------------- K0 gather / scatter
constexpr int kMaxTensorsPerLaunch = 96;
struct CopyTable {
    const float* src[kMaxTensorsPerLaunch];
    float* dst[kMaxTensorsPerLaunch];
    int64_t n[kMaxTensorsPerLaunch];
};

__global__ void __launch_bounds__(kThreads) copy_tensors_kernel(const CopyTable t) {
    const int k = blockIdx.y;
    const float* __restrict__ src = t.src[k];
    float* __restrict__ dst = t.dst[k];
    const int64_t n = t.n[k];
    const int64_t tid = int64_t(blockIdx.x) * kThreads + threadIdx.x;
    const int64_t stride = int64_t(gridDim.x) * kThreads;
    const bool vec = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15u) == 0;
    int64_t done = 0;
    if (vec) {
        const int64_t n4 = n / 4;
        for (int64_t i = tid; i < n4; i += stride)
            reinterpret_cast<float4*>(dst)[i] = __ldcs(reinterpret_cast<const float4*>(src) + i);
        done = n4 * 4;
    }
    for (int64_t i = done + tid; i < n; i += stride) dst[i] = src[i];
}

int copy_tensors(const float* const* src, float* const* dst, const int64_t* n, int count, cudaStream_t s) {
    for (int base = 0; base < count; base += kMaxTensorsPerLaunch) {
        CopyTable t{};
        const int m = std::min(kMaxTensorsPerLaunch, count - base);
        int64_t maxn = 1;
        for (int k = 0; k < m; ++k) {
            t.src[k] = src[base + k];
            t.dst[k] = dst[base + k];
            t.n[k] = n[base + k];
            maxn = std::max<int64_t>(maxn, n[base + k]);
        }
        int64_t bx = (maxn / 4 + kThreads - 1) / kThreads;
        bx = std::max<int64_t>(1, std::min<int64_t>(bx, sm_count() * 4));
        copy_tensors_kernel<<<dim3(unsigned(bx), unsigned(m)), kThreads, 0, s>>>(t);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return int(e);
    }
    return 0;
}

// ----------------------------------------------------------------- checksum
__global__ void __launch_bounds__(kThreads) checksum_kernel(const uint32_t* __restrict__ w, int64_t n,
                                                            unsigned long long* out) {
    unsigned long long acc = 0;
    const int64_t stride = int64_t(gridDim.x) * kThreads;
    for (int64_t i = int64_t(blockIdx.x) * kThreads + threadIdx.x; i < n; i += stride) acc += w[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    __shared__ unsigned long long part[kThreads / 32];
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (int k = 0; k < kThreads / 32; ++k) t += part[k];
        atomicAdd(out, t);
    }
}

__global__ void fill_u64_kernel(unsigned long long* base, int rows, int row_stride, int cols, unsigned long long v) {
    for (int k = threadIdx.x; k < rows * cols; k += blockDim.x) base[(k / cols) * row_stride + k % cols] = v;
}

}  // namespace

int launch_fill_u64(unsigned long long* base, int rows, int row_stride, int cols, unsigned long long value,
                    void* stream) {
    fill_u64_kernel<<<1, 128, 0, static_cast<cudaStream_t>(stream)>>>(base, rows, row_stride, cols, value);
    return int(cudaGetLastError());
}

int current_kernel_impl() { return kernel_impl(); }

int set_kernel_impl(int impl) {
    const int prev = kernel_impl();
    if (impl == 0 || impl == 1 || impl == 2) g_impl = impl;
    return prev;
}

int launch_fused(int ops, int wire, const KernelArgs& a, void* stream) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (a.n <= 0) return 0;
    if (wire == DASO_WIRE_BF16) return dispatch<DASO_WIRE_BF16>(ops, a, s);
    if (wire == DASO_WIRE_FP32) return dispatch<DASO_WIRE_FP32>(ops, a, s);
    return int(cudaErrorInvalidValue);
}

int launch_gather(const float* const* src, const size_t* numel, const size_t* offsets, int count,
                  float* dst, void* stream) {
    float* d[kMaxTensorsPerLaunch];
    int64_t n[kMaxTensorsPerLaunch];
    for (int base = 0; base < count; base += kMaxTensorsPerLaunch) {
        const int m = std::min(kMaxTensorsPerLaunch, count - base);
        for (int k = 0; k < m; ++k) {
            d[k] = dst + offsets[base + k];
            n[k] = int64_t(numel[base + k]);
        }
        int e = copy_tensors(src + base, d, n, m, static_cast<cudaStream_t>(stream));
        if (e) return e;
    }
    return 0;
}

int launch_scatter(const float* src, float* const* dst, const size_t* numel, const size_t* offsets,
                   int count, void* stream) {
    const float* s[kMaxTensorsPerLaunch];
    int64_t n[kMaxTensorsPerLaunch];
    for (int base = 0; base < count; base += kMaxTensorsPerLaunch) {
        const int m = std::min(kMaxTensorsPerLaunch, count - base);
        for (int k = 0; k < m; ++k) {
            s[k] = src + offsets[base + k];
            n[k] = int64_t(numel[base + k]);
        }
        int e = copy_tensors(s, dst + base, n, m, static_cast<cudaStream_t>(stream));
        if (e) return e;
    }
    return 0;
}

int launch_checksum(const float* x, int64_t n, uint64_t* out, void* stream) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaError_t e = cudaMemsetAsync(out, 0, sizeof(uint64_t), s);
    if (e != cudaSuccess) return int(e);
    int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((n + kThreads - 1) / kThreads, sm_count() * 8));
    checksum_kernel<<<unsigned(blocks), kThreads, 0, s>>>(reinterpret_cast<const uint32_t*>(x), n,
                                                        reinterpret_cast<unsigned long long*>(out));
    return int(cudaGetLastError());
}

}  // namespace daso
