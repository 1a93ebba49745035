// Device helpers shared by the fused kernels (kernels.cu) and the peer-memory
// local-tier kernel (peer.cu): 128-bit streaming loads/stores and the wire formats.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include <cstdint>

#include "daso_internal.h"

namespace daso {
namespace dev {

constexpr int kThreads = 256;
constexpr int kVec = 8;

// ----------------------------------------------------------------- fp32 streams
template <int N>
__device__ __forceinline__ void ld_f32(const float* p, float (&r)[N]) {
    if constexpr (N == 8) {
        float4 a = __ldcs(reinterpret_cast<const float4*>(p));
        float4 b = __ldcs(reinterpret_cast<const float4*>(p) + 1);
        r[0] = a.x; r[1] = a.y; r[2] = a.z; r[3] = a.w;
        r[4] = b.x; r[5] = b.y; r[6] = b.z; r[7] = b.w;
    } else {
#pragma unroll
        for (int j = 0; j < N; ++j) r[j] = __ldcs(p + j);
    }
}

template <int N>
__device__ __forceinline__ void st_f32(float* p, const float (&r)[N]) {
    if constexpr (N == 8) {
        __stcs(reinterpret_cast<float4*>(p), make_float4(r[0], r[1], r[2], r[3]));
        __stcs(reinterpret_cast<float4*>(p) + 1, make_float4(r[4], r[5], r[6], r[7]));
    } else {
#pragma unroll
        for (int j = 0; j < N; ++j) __stcs(p + j, r[j]);
    }
}

// ----------------------------------------------------------------- wire formats
__device__ __forceinline__ float bf16lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
    __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);   // RNE (R18)
    return *reinterpret_cast<uint32_t*>(&h);
}

template <int WIRE>
struct Wire;

template <>
struct Wire<DASO_WIRE_BF16> {
    template <int N>
    static __device__ __forceinline__ void load(const void* base, int64_t i, float (&r)[N]) {
        const uint16_t* p = static_cast<const uint16_t*>(base) + i;
        if constexpr (N == 8) {
            uint4 u = __ldcs(reinterpret_cast<const uint4*>(p));
            r[0] = bf16lo(u.x); r[1] = bf16hi(u.x); r[2] = bf16lo(u.y); r[3] = bf16hi(u.y);
            r[4] = bf16lo(u.z); r[5] = bf16hi(u.z); r[6] = bf16lo(u.w); r[7] = bf16hi(u.w);
        } else {
#pragma unroll
            for (int j = 0; j < N; ++j) r[j] = __uint_as_float(uint32_t(p[j]) << 16);
        }
    }
    template <int N>
    static __device__ __forceinline__ void store(void* base, int64_t i, const float (&r)[N]) {
        uint16_t* p = static_cast<uint16_t*>(base) + i;
        if constexpr (N == 8) {
            uint4 u = make_uint4(pack_bf16x2(r[0], r[1]), pack_bf16x2(r[2], r[3]),
                                 pack_bf16x2(r[4], r[5]), pack_bf16x2(r[6], r[7]));
            __stcs(reinterpret_cast<uint4*>(p), u);
        } else {
#pragma unroll
            for (int j = 0; j < N; ++j) p[j] = __bfloat16_as_ushort(__float2bfloat16_rn(r[j]));
        }
    }
    template <int N>
    static __device__ __forceinline__ void load_smem(const void* base, int i, float (&r)[N]) {
        static_assert(N == 8, "");
        uint4 u = *reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(base) + i);
        r[0] = bf16lo(u.x); r[1] = bf16hi(u.x); r[2] = bf16lo(u.y); r[3] = bf16hi(u.y);
        r[4] = bf16lo(u.z); r[5] = bf16hi(u.z); r[6] = bf16lo(u.w); r[7] = bf16hi(u.w);
    }
    template <int N>
    static __device__ __forceinline__ void store_smem(void* base, int i, const float (&r)[N]) {
        static_assert(N == 8, "");
        *reinterpret_cast<uint4*>(static_cast<uint16_t*>(base) + i) =
            make_uint4(pack_bf16x2(r[0], r[1]), pack_bf16x2(r[2], r[3]), pack_bf16x2(r[4], r[5]),
                       pack_bf16x2(r[6], r[7]));
    }
};

template <>
struct Wire<DASO_WIRE_FP32> {
    template <int N>
    static __device__ __forceinline__ void load(const void* base, int64_t i, float (&r)[N]) {
        ld_f32<N>(static_cast<const float*>(base) + i, r);
    }
    template <int N>
    static __device__ __forceinline__ void store(void* base, int64_t i, const float (&r)[N]) {
        st_f32<N>(static_cast<float*>(base) + i, r);
    }
    template <int N>
    static __device__ __forceinline__ void load_smem(const void* base, int i, float (&r)[N]) {
#pragma unroll
        for (int j = 0; j < N; j += 4) {
            float4 q = *reinterpret_cast<const float4*>(static_cast<const float*>(base) + i + j);
            r[j] = q.x; r[j + 1] = q.y; r[j + 2] = q.z; r[j + 3] = q.w;
        }
    }
    template <int N>
    static __device__ __forceinline__ void store_smem(void* base, int i, const float (&r)[N]) {
#pragma unroll
        for (int j = 0; j < N; j += 4)
            *reinterpret_cast<float4*>(static_cast<float*>(base) + i + j) = make_float4(r[j], r[j + 1], r[j + 2], r[j + 3]);
    }
};

// ---- TMA (bulk-copy engine) and mbarrier PTX -------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// Wait for an mbarrier phase.  A transfer that never completes (a bug, a dead peer
// mapping) must not hang the GPU: after 20 s give up, raise bit 2 of *err and return
// false (the caller stops using the stage: its data never arrived).
__device__ __forceinline__ bool mbar_wait(uint64_t* bar, uint32_t parity, uint32_t* err = nullptr) {
    if (mbar_try_wait(bar, parity)) return true;
    const unsigned long long t0 = globaltimer_ns();
    while (!mbar_try_wait(bar, parity)) {
        if (globaltimer_ns() - t0 > 20ull * 1000 * 1000 * 1000) {
            if (err) atomicOr(err, 4u);
            return false;
        }
    }
    return true;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

}  // namespace dev
}  // namespace daso
