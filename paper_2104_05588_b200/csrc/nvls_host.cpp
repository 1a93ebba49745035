// Host-only setup of the NVLS buckets (DASO_MODE_NVLS): register x and g as NCCL symmetric
// windows on the node communicator and create a device communicator with multimem enabled
// on the load-store-accessible team, then resolve the multicast and peer addresses of the two
// windows.  Compiled as plain C++ (no device code) because NCCL's device API headers declare
// device functions that only the NCCL device implementation defines.
#include <cuda_runtime.h>
#include <nccl.h>
#include <nccl_device/core.h>
#include <nccl_device/impl/comm__types.h>
#include <nccl_device/impl/core__types.h>

#include <new>

#include "daso_internal.h"

namespace daso {

int nvls_setup(void* node_comm, void* x, void* g, size_t bytes, int G, NvlsBuckets* out, const char** why) {
    ncclComm_t comm = static_cast<ncclComm_t>(node_comm);
    ncclWindow_t wx = nullptr, wg = nullptr;
    if (ncclCommWindowRegister(comm, x, bytes, &wx, NCCL_WIN_COLL_SYMMETRIC) != ncclSuccess ||
        ncclCommWindowRegister(comm, g, bytes, &wg, NCCL_WIN_COLL_SYMMETRIC) != ncclSuccess) {
        *why = "ncclCommWindowRegister failed";
        return 1;
    }
    out->win_x = wx;
    out->win_g = wg;
    auto* dc = new (std::nothrow) ncclDevComm{};
    if (!dc) {
        *why = "out of host memory";
        return 3;
    }
    ncclDevCommRequirements req{};
    req.lsaMultimem = true;
    if (ncclDevCommCreate(comm, &req, dc) != ncclSuccess) {
        delete dc;
        *why = "ncclDevCommCreate(lsaMultimem) failed";
        return 1;
    }
    out->devcomm = dc;
    if (dc->lsaMultimem.mcBasePtr == nullptr || dc->lsaSize != G) {
        *why = "no NVLS multicast on the node's load-store-accessible team";
        return 2;
    }
    ncclWindow_vidmem vx{}, vg{};
    if (cudaMemcpy(&vx, wx, sizeof vx, cudaMemcpyDefault) != cudaSuccess ||
        cudaMemcpy(&vg, wg, sizeof vg, cudaMemcpyDefault) != cudaSuccess) {
        *why = "cannot read the window descriptors";
        return 3;
    }
    char* mc = static_cast<char*>(dc->lsaMultimem.mcBasePtr);
    out->x_mc = reinterpret_cast<float*>(mc + size_t(vx.mcOffset4K) * 4096);
    out->g_mc = reinterpret_cast<float*>(mc + size_t(vg.mcOffset4K) * 4096);
    for (int q = 0; q < G && q < kMaxPeers; ++q) {
        out->peer_x[q] = reinterpret_cast<float*>(vx.lsaFlatBase + (size_t(q) * vx.stride4G << 32));
        out->peer_g[q] = reinterpret_cast<float*>(vg.lsaFlatBase + (size_t(q) * vg.stride4G << 32));
    }
    return 0;
}

void nvls_teardown(void* node_comm, NvlsBuckets* b) {
    ncclComm_t comm = static_cast<ncclComm_t>(node_comm);
    if (b->devcomm) {
        auto* dc = static_cast<ncclDevComm*>(b->devcomm);
        ncclDevCommDestroy(comm, dc);
        delete dc;
        b->devcomm = nullptr;
    }
    if (b->win_x) ncclCommWindowDeregister(comm, static_cast<ncclWindow_t>(b->win_x));
    if (b->win_g) ncclCommWindowDeregister(comm, static_cast<ncclWindow_t>(b->win_g));
    b->win_x = b->win_g = nullptr;
}

}  // namespace daso
