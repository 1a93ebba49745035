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
// a grid-stride loop over a grid sized to full occupancy on all SMs; the optional
// non-finite flag is a warp ballot + one atomicOr per warp.  No shared memory or
// tensor cores: there is no reuse and no contraction.
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include "daso_internal.h"

namespace daso {
namespace {

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
};

// ----------------------------------------------------------------- fused body
template <int OPS, int WIRE, int N>
__device__ __forceinline__ void body(const KernelArgs& a, int64_t i, bool& bad) {
    float x[N];
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
#pragma unroll 4
        for (int p = 0; p < a.P; ++p) {                          // ascending node order (R18)
            float s[N];
            Wire<WIRE>::template load<N>(a.slot, p * a.slot_stride + i, s);
#pragma unroll
            for (int j = 0; j < N; ++j) acc[j] += s[j] - x[j];
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
    if constexpr ((OPS & OP_PACK) != 0) Wire<WIRE>::template store<N>(a.pack_out, i, x);
}

template <int OPS, int WIRE>
__global__ void __launch_bounds__(kThreads) fused_kernel(const KernelArgs a) {
    const int64_t nchunks = a.n / kVec;
    const int64_t stride = int64_t(gridDim.x) * kThreads;
    bool bad = false;
    for (int64_t c = int64_t(blockIdx.x) * kThreads + threadIdx.x; c < nchunks; c += stride)
        body<OPS, WIRE, kVec>(a, c * kVec, bad);
    if (blockIdx.x == gridDim.x - 1) {                           // ragged tail (< 8 elements)
        const int64_t i = nchunks * kVec + threadIdx.x;
        if (i < a.n) body<OPS, WIRE, 1>(a, i, bad);
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

template <int OPS, int WIRE>
int launch_t(const KernelArgs& a, cudaStream_t s) {
    static int occ = 0;
    if (occ == 0) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fused_kernel<OPS, WIRE>, kThreads, 0);
        if (occ <= 0) occ = 1;
    }
    const int64_t nchunks = a.n / kVec;
    int64_t blocks = (nchunks + kThreads - 1) / kThreads;
    const int64_t cap = int64_t(sm_count()) * occ;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    fused_kernel<OPS, WIRE><<<dim3(unsigned(blocks)), dim3(kThreads), 0, s>>>(a);
    return int(cudaGetLastError());
}

template <int WIRE>
int dispatch(int ops, const KernelArgs& a, cudaStream_t s) {
    switch (ops) {
        case OP_UPDATE: return launch_t<OP_UPDATE, WIRE>(a, s);
        case OP_UPDATE | OP_PACK: return launch_t<OP_UPDATE | OP_PACK, WIRE>(a, s);
        case OP_UPDATE | OP_MERGE: return launch_t<OP_UPDATE | OP_MERGE, WIRE>(a, s);
        case OP_UPDATE | OP_MERGE | OP_PACK: return launch_t<OP_UPDATE | OP_MERGE | OP_PACK, WIRE>(a, s);
        case OP_MERGE: return launch_t<OP_MERGE, WIRE>(a, s);
        case OP_MERGE | OP_PACK: return launch_t<OP_MERGE | OP_PACK, WIRE>(a, s);
        case OP_AVERAGE: return launch_t<OP_AVERAGE, WIRE>(a, s);
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

}  // namespace

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
