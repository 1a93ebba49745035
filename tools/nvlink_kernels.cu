// NVLink ceiling probe for the fused node-tier kernel's traffic pattern.
// One process drives all visible GPUs (G = 2..8, peer access enabled between all); every GPU
// runs the same kernel at the same time on its own shard of n parameters, so each link
// direction carries what it carries in DASO_MODE_FUSED.  No kernel waits on another.
//
//   tma_rw   : per 2048-param tile, cp.async.bulk reads of the tile of every node peer's g
//              (G-1 remote) + bulk stores of a tile to every peer's x (G-1 remote) — the fused
//              kernel's data movement without its arithmetic.  Bytes per direction per GPU:
//              2 (G-1)/G 4n
//   tma_r    : only the remote bulk reads ((G-1)/G 4n per direction)
//   tma_w    : only the remote bulk stores ((G-1)/G 4n per direction)
//   ldg_rw   : the same as tma_rw with 128-bit register loads/stores (the register peer path)
//   push_rs  : write-only node tier, phase A: every GPU stores its g tile q into owner q's
//              receive buffer (remote 128-bit stores), phase B = tma_w; reported per phase
//   ce_bidi  : copy engines, every GPU copies (G-1)/G 4n to its peers (cudaMemcpyPeerAsync)
//   tma_r+ce_w: the node tier's two halves on different engines at once — SM bulk reads of the
//              peers' g tiles (tma_r) while the copy engines push (G-1)/G 4n to the peers' x
//   ce_rw    : both halves on copy engines — pulls of the peers' g shards + pushes to their x
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/nvk tools/nvlink_kernels.cu
//   /tmp/nvk [n_params] [ctas (0 = SMs-16)] [stages (0 = auto)] [tile floats (2048)]
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t e_ = (x);                                                                  \
        if (e_ != cudaSuccess) {                                                               \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
            exit(1);                                                                           \
        }                                                                                      \
    } while (0)

constexpr int kMax = 8, kThr = 256;

struct Args {
    const float* gp[kMax];   // every GPU's g at this GPU's shard
    float* xp[kMax];         // every GPU's x at this GPU's shard
    float* rp[kMax];         // push: owner q's receive buffer, row `me`
    const float* gq[kMax];   // push: this GPU's g at shard q
    int64_t n;               // shard length
    int G, me, NS, T;        // T = tile (floats per bulk copy)
};

__device__ __forceinline__ uint32_t su32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

template <bool RD, bool WR>
__global__ void __launch_bounds__(kThr, 1) tma_kernel(Args a) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int G = a.G, NS = a.NS, kT = a.T;
    const uint32_t stage = uint32_t(G) * kT * 4;
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + size_t(NS) * stage);
    const int64_t nt = a.n / kT;
    const int64_t my = nt > blockIdx.x ? (nt - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[s])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x != 0) return;   // one thread drives the copy engine
    auto load = [&](int64_t k) {
        const int s = int(k % NS);
        const int64_t e0 = (int64_t(blockIdx.x) + k * gridDim.x) * kT;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"(stage) : "memory");
        for (int q = 0; q < G; ++q)
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    su32(sm + size_t(s) * stage + size_t(q) * kT * 4)),
                "l"(a.gp[q] + e0), "r"(kT * 4), "r"(su32(&bar[s]))
                : "memory");
    };
    if (RD)
        for (int64_t k = 0; k < my && k < NS; ++k) load(k);
    for (int64_t k = 0; k < my; ++k) {
        const int s = int(k % NS);
        if (RD) {
            uint32_t ok = 0;
            while (!ok)
                asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                             : "=r"(ok)
                             : "r"(su32(&bar[s])), "r"(uint32_t((k / NS) & 1))
                             : "memory");
        }
        const int64_t e0 = (int64_t(blockIdx.x) + k * gridDim.x) * kT;
        if (WR) {
            for (int q = 0; q < G; ++q) {
                const int qq = (a.me + 1 + q) % G;
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(a.xp[qq] + e0),
                             "r"(su32(sm + size_t(s) * stage)), "r"(kT * 4)
                             : "memory");
            }
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        if (RD && !WR && k + NS < my) load(k + NS);
        if (RD && WR && k >= 1 && k - 1 + NS < my) {   // stage of tile k-1 is free once its stores read it
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            load(k - 1 + NS);
        }
    }
    if (WR) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void __launch_bounds__(kThr) ldg_rw_kernel(Args a) {
    const int64_t n4 = a.n / 4;
    for (int64_t i = int64_t(blockIdx.x) * kThr + threadIdx.x; i < n4; i += int64_t(gridDim.x) * kThr) {
        float4 acc = make_float4(0, 0, 0, 0);
        float4 t[kMax];
#pragma unroll
        for (int q = 0; q < kMax; ++q)
            if (q < a.G) t[q] = __ldcs(reinterpret_cast<const float4*>(a.gp[q]) + i);
#pragma unroll
        for (int q = 0; q < kMax; ++q)
            if (q < a.G) { acc.x += t[q].x; acc.y += t[q].y; acc.z += t[q].z; acc.w += t[q].w; }
#pragma unroll
        for (int q = 0; q < kMax; ++q)
            if (q < a.G) __stcs(reinterpret_cast<float4*>(a.xp[q]) + i, acc);
    }
}

__global__ void __launch_bounds__(kThr) push_kernel(Args a) {   // phase A of push_rs
    const int64_t n4 = a.n / 4;
    for (int64_t i = int64_t(blockIdx.x) * kThr + threadIdx.x; i < n4; i += int64_t(gridDim.x) * kThr) {
#pragma unroll
        for (int q = 0; q < kMax; ++q)
            if (q < a.G) {
                const int qq = (a.me + 1 + q) % a.G;
                __stcs(reinterpret_cast<float4*>(a.rp[qq]) + i, __ldcs(reinterpret_cast<const float4*>(a.gq[qq]) + i));
            }
    }
}

int main(int argc, char** argv) {
    int G = 0;
    CK(cudaGetDeviceCount(&G));
    G = std::min(G, kMax);
    const int64_t N = argc > 1 ? atoll(argv[1]) : 25557056;
    int ctas = argc > 2 ? atoi(argv[2]) : 0;
    const int NSreq = argc > 3 ? atoi(argv[3]) : 0;
    const int kT = argc > 4 ? atoi(argv[4]) : 2048;
    const int64_t n = (N / G) / kT * kT;   // shard, whole tiles
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    if (ctas <= 0) ctas = sms - 16;
    std::vector<float*> g(G), x(G), r(G);
    std::vector<cudaStream_t> st(G);
    for (int d = 0; d < G; ++d) {
        CK(cudaSetDevice(d));
        for (int e = 0; e < G; ++e)
            if (e != d) CK(cudaDeviceEnablePeerAccess(e, 0));
        CK(cudaMalloc(&g[d], size_t(n) * G * 4));
        CK(cudaMalloc(&x[d], size_t(n) * G * 4));
        CK(cudaMalloc(&r[d], size_t(n) * G * 4));
        CK(cudaMemset(g[d], 0, size_t(n) * G * 4));
        CK(cudaStreamCreateWithFlags(&st[d], cudaStreamNonBlocking));
    }
    const uint32_t stage = uint32_t(G) * kT * 4;
    const int NS = NSreq > 0 ? NSreq : int(std::min<int64_t>(8, (200 * 1024) / stage));
    if (NS < 2) {
        printf("{\"skip\": \"tile %d x G %d leaves < 2 stages\"}\n", kT, G);
        return 0;
    }
    const size_t smem = size_t(NS) * stage + 8 * NS;
    auto args = [&](int d) {
        Args a{};
        for (int q = 0; q < G; ++q) {
            a.gp[q] = g[q] + size_t(d) * n;
            a.xp[q] = x[q] + size_t(d) * n;
            a.rp[q] = r[q] + size_t(d) * n;
            a.gq[q] = g[d] + size_t(q) * n;
        }
        a.n = n;
        a.G = G;
        a.me = d;
        a.NS = NS;
        a.T = kT;
        return a;
    };
    auto run = [&](const char* name, double bytes_dir, auto launch) {
        const int iters = 20;
        std::vector<cudaEvent_t> e0(G), e1(G);
        for (int d = 0; d < G; ++d) {
            CK(cudaSetDevice(d));
            launch(d);   // warm-up
        }
        for (int d = 0; d < G; ++d) {
            CK(cudaSetDevice(d));
            CK(cudaStreamSynchronize(st[d]));
            CK(cudaEventCreate(&e0[d]));
            CK(cudaEventCreate(&e1[d]));
        }
        for (int d = 0; d < G; ++d) {
            CK(cudaSetDevice(d));
            CK(cudaEventRecord(e0[d], st[d]));
        }
        for (int i = 0; i < iters; ++i)
            for (int d = 0; d < G; ++d) {
                CK(cudaSetDevice(d));
                launch(d);
            }
        for (int d = 0; d < G; ++d) {
            CK(cudaSetDevice(d));
            CK(cudaEventRecord(e1[d], st[d]));
        }
        float worst = 0;
        for (int d = 0; d < G; ++d) {
            CK(cudaSetDevice(d));
            CK(cudaEventSynchronize(e1[d]));
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, e0[d], e1[d]));
            worst = std::max(worst, ms / iters);
        }
        printf("{\"probe\": \"%s\", \"G\": %d, \"shard\": %lld, \"ctas\": %d, \"stages\": %d, \"tile\": %d, "
               "\"us\": %.1f, \"GBs_per_dir\": %.1f, \"frac_770\": %.3f}\n",
               name, G, (long long)n, ctas, NS, kT, worst * 1e3, bytes_dir / (worst * 1e-3) / 1e9,
               bytes_dir / (worst * 1e-3) / 1e9 / 770.0);
        fflush(stdout);
    };
    const double one = double(G - 1) * n * 4;   // remote bytes one way per GPU
    for (int d = 0; d < G; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaFuncSetAttribute(tma_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        CK(cudaFuncSetAttribute(tma_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        CK(cudaFuncSetAttribute(tma_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    }
    run("tma_rw", 2 * one, [&](int d) { tma_kernel<true, true><<<ctas, kThr, smem, st[d]>>>(args(d)); });
    run("tma_r", one, [&](int d) { tma_kernel<true, false><<<ctas, kThr, smem, st[d]>>>(args(d)); });
    run("tma_w", one, [&](int d) { tma_kernel<false, true><<<ctas, kThr, smem, st[d]>>>(args(d)); });
    for (int bpsm : {2, 4, 8})
        run((std::string("ldg_rw_bpsm") + std::to_string(bpsm)).c_str(), 2 * one,
            [&](int d) { ldg_rw_kernel<<<sms * bpsm, kThr, 0, st[d]>>>(args(d)); });
    for (int bpsm : {2, 4, 8})
        run((std::string("push_rs_phaseA_bpsm") + std::to_string(bpsm)).c_str(), one,
            [&](int d) { push_kernel<<<sms * bpsm, kThr, 0, st[d]>>>(args(d)); });
    std::vector<cudaStream_t> st2(G);
    std::vector<cudaEvent_t> fork(G), join(G);
    for (int d = 0; d < G; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaStreamCreateWithFlags(&st2[d], cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&fork[d], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&join[d], cudaEventDisableTiming));
    }
    auto ce_push = [&](int d, cudaStream_t s) {
        for (int k = 1; k < G; ++k) {
            const int q = (d + k) % G;
            CK(cudaMemcpyPeerAsync(x[q] + size_t(d) * n, q, r[d] + size_t(d) * n, d, size_t(n) * 4, s));
        }
    };
    run("tma_r+ce_w", 2 * one, [&](int d) {
        CK(cudaEventRecord(fork[d], st[d]));
        CK(cudaStreamWaitEvent(st2[d], fork[d], 0));
        tma_kernel<true, false><<<ctas, kThr, smem, st[d]>>>(args(d));
        ce_push(d, st2[d]);
        CK(cudaEventRecord(join[d], st2[d]));
        CK(cudaStreamWaitEvent(st[d], join[d], 0));
    });
    run("ce_rw", 2 * one, [&](int d) {
        CK(cudaEventRecord(fork[d], st[d]));
        CK(cudaStreamWaitEvent(st2[d], fork[d], 0));
        for (int k = 1; k < G; ++k) {   // pulls: peer q's g at this GPU's shard -> local receive buffer
            const int q = (d + k) % G;
            CK(cudaMemcpyPeerAsync(r[d] + size_t(q) * n, d, g[q] + size_t(d) * n, q, size_t(n) * 4, st[d]));
        }
        ce_push(d, st2[d]);
        CK(cudaEventRecord(join[d], st2[d]));
        CK(cudaStreamWaitEvent(st[d], join[d], 0));
    });
    run("ce_bidi", one, [&](int d) {
        for (int q = 0; q < G; ++q)
            if (q != d) CK(cudaMemcpyPeerAsync(x[q] + size_t(d) * n, q, g[d] + size_t(q) * n, d, size_t(n) * 4, st[d]));
    });
    return 0;
}
