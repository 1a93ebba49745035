// Standalone exploration of data-movement variants for the K1 update stream
// (x, v read+write, g read; 20 B/param) at ResNet-50 size on one B200.
// Not part of libdaso.so: results feed the choice made in csrc/kernels.cu.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o k1v tools/k1_variants.cu && ./k1v
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

struct A { float* x; float* v; const float* g; long long n; float lr, mu, wd, gs; };

template <int UNROLL, bool CS>
__device__ __forceinline__ void step8(const A& a, long long i) {
    float4 x[2 * UNROLL], v[2 * UNROLL], g[2 * UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
        const float4* xp = reinterpret_cast<const float4*>(a.x + i) + 2 * u;
        const float4* vp = reinterpret_cast<const float4*>(a.v + i) + 2 * u;
        const float4* gp = reinterpret_cast<const float4*>(a.g + i) + 2 * u;
        if (CS) { x[2*u] = __ldcs(xp); x[2*u+1] = __ldcs(xp + 1); v[2*u] = __ldcs(vp); v[2*u+1] = __ldcs(vp + 1); g[2*u] = __ldcs(gp); g[2*u+1] = __ldcs(gp + 1); }
        else { x[2*u] = xp[0]; x[2*u+1] = xp[1]; v[2*u] = vp[0]; v[2*u+1] = vp[1]; g[2*u] = __ldg(gp); g[2*u+1] = __ldg(gp + 1); }
    }
#pragma unroll
    for (int k = 0; k < 2 * UNROLL; ++k) {
        float* xe = &x[k].x; float* ve = &v[k].x; const float* ge = &g[k].x;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            float d = fmaf(a.wd, xe[j], ge[j] * a.gs);
            ve[j] = fmaf(a.mu, ve[j], d);
            xe[j] = fmaf(-a.lr, ve[j], xe[j]);
        }
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
        float4* xp = reinterpret_cast<float4*>(a.x + i) + 2 * u;
        float4* vp = reinterpret_cast<float4*>(a.v + i) + 2 * u;
        if (CS) { __stcs(xp, x[2*u]); __stcs(xp + 1, x[2*u+1]); __stcs(vp, v[2*u]); __stcs(vp + 1, v[2*u+1]); }
        else { xp[0] = x[2*u]; xp[1] = x[2*u+1]; vp[0] = v[2*u]; vp[1] = v[2*u+1]; }
    }
}

template <int UNROLL, bool CS, int MINB>
__global__ void __launch_bounds__(256, MINB) k1(const A a) {
    const long long per = 8LL * UNROLL;
    const long long nch = a.n / per;
    for (long long c = (long long)blockIdx.x * 256 + threadIdx.x; c < nch; c += (long long)gridDim.x * 256)
        step8<UNROLL, CS>(a, c * per);
}

__global__ void flush(float* p, long long n) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) p[i] = p[i] * 0.5f + 1.f;
}

template <int UNROLL, bool CS, int MINB>
int run(const char* name, A a, int grid_mult, float* fl, long long fn, int sms) {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k1<UNROLL, CS, MINB>, 256, 0);
    long long nch = a.n / (8LL * UNROLL);
    long long blocks = grid_mult > 0 ? (long long)sms * occ * grid_mult : (nch + 255) / 256;
    if (blocks > (nch + 255) / 256) blocks = (nch + 255) / 256;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float tot = 0; int it = 20;
    for (int r = 0; r < it + 3; ++r) {
        flush<<<sms * 4, 512>>>(fl, fn);
        cudaEventRecord(e0);
        k1<UNROLL, CS, MINB><<<(unsigned)blocks, 256>>>(a);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (r >= 3) tot += ms;
    }
    double us = tot / it * 1e3;
    printf("%-34s occ=%d blocks=%lld  %8.2f us  %7.1f GB/s\n", name, occ, blocks, us, 20.0 * a.n / (us * 1e-6) / 1e9);
    return 0;
}

int main() {
    const long long n = 25557032LL / 16 * 16;
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *x, *v, *g, *fl;
    const long long fn = 64LL << 20;   // 256 MB flush buffer
    CK(cudaMalloc(&x, n * 4)); CK(cudaMalloc(&v, n * 4)); CK(cudaMalloc(&g, n * 4)); CK(cudaMalloc(&fl, fn * 4));
    cudaMemset(x, 0, n * 4); cudaMemset(v, 0, n * 4); cudaMemset(g, 0, n * 4); cudaMemset(fl, 0, fn * 4);
    A a{x, v, g, n, 1e-3f, 0.9f, 1e-4f, 0.5f};
    run<1, true, 1>("u1 cs persistent(occ)", a, 1, fl, fn, sms);
    run<1, true, 8>("u1 cs minb8 persistent", a, 1, fl, fn, sms);
    run<1, true, 1>("u1 cs one-shot grid", a, 0, fl, fn, sms);
    run<1, false, 1>("u1 default-cache persistent", a, 1, fl, fn, sms);
    run<2, true, 1>("u2 cs persistent", a, 1, fl, fn, sms);
    run<2, true, 4>("u2 cs minb4 persistent", a, 1, fl, fn, sms);
    run<2, false, 1>("u2 default-cache persistent", a, 1, fl, fn, sms);
    run<4, true, 1>("u4 cs persistent", a, 1, fl, fn, sms);
    run<1, true, 8>("u1 cs minb8 one-shot", a, 0, fl, fn, sms);
    run<2, true, 1>("u2 cs one-shot", a, 0, fl, fn, sms);
    // copy reference: 8 B/param (read x write v) through cudaMemcpy
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float tot = 0;
    for (int r = 0; r < 23; ++r) {
        flush<<<sms * 4, 512>>>(fl, fn);
        cudaEventRecord(e0); cudaMemcpyAsync(v, x, n * 4, cudaMemcpyDeviceToDevice); cudaEventRecord(e1);
        cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (r >= 3) tot += ms;
    }
    printf("%-34s %8.2f us  %7.1f GB/s (r+w)\n", "cudaMemcpy D2D 102MB", tot / 20 * 1e3, 8.0 * n / (tot / 20 * 1e-3) / 1e9);
    return 0;
}
