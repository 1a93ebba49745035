// Internal declarations shared by the translation units of libdaso.so.
#pragma once

#include <algorithm>
#include <cstdint>
#include <string>

#include "daso.h"

namespace daso {

int resolved_S(const daso_sched_config& c);
const char* validate_sched(const daso_sched_config& c);   // nullptr = valid
int phase_of(int64_t epoch, const daso_sched_config& c);

struct Schedule {
    daso_sched_config cfg;
    int B = 1, S = 0;
    int64_t step = 0;
    int batch_in_cycle = 0;
    int64_t n_syncs = 0;
    bool has_pending = false;
    int64_t pend_due = -1, pend_sent = -1;
    int pend_S = 0, pend_group = -1;

    explicit Schedule(const daso_sched_config& c);
    daso_record next(int plateau);
};

// ---- kernel launchers (kernels.cu); return a cudaError_t as int ----------
enum Op : int {
    OP_UPDATE = 1,   // K1
    OP_MERGE = 2,    // Eq. (1)
    OP_PACK = 4,     // wire cast into pack_out
    OP_AVERAGE = 8,  // K4 blocking average
    OP_NOX = 16,     // peer kernels only: no x stores, no end barrier (blocking batch: the average
                     // that follows replaces x; launch_avg_publish's end barrier covers the g reads)
    OP_PUSH = 32,    // with OP_PACK: also store the packed row into KernelArgs::push[0..npush) (kernel push)
};

struct KernelArgs {
    float* x = nullptr;
    float* v = nullptr;
    const float* g = nullptr;
    int64_t n = 0;
    float lr = 0.f, mu = 0.f, wd = 0.f, gscale = 1.f;
    const void* slot = nullptr;   // [P][slot_stride] wire elements
    int64_t slot_stride = 0;
    int P = 0;
    float den = 1.f;              // 2S + P (merge) or P (average)
    void* pack_out = nullptr;
    // blocking sync with the copy-engine transport: the packed row is also stored into these
    // npush remote slot rows (group members' slots over NVLink) by the same kernel
    void* push[7] = {};
    int npush = 0;
    uint32_t* flag = nullptr;     // bit 0: non-finite parameter (nullable: check off)
    uint32_t* err = nullptr;      // bit 2: TMA (mbarrier) wait timed out (nullable)
};

constexpr int kMaxPush = 7;   // KernelArgs::push capacity (groups of up to 8 members)
int launch_fused(int ops, int wire, const KernelArgs& a, void* stream);

// fused node-local tier over NVLink peer memory (peer.cu)
constexpr int kMaxPeers = 8;
struct PeerArgs {
    KernelArgs a;                              // x, v, pack_out, slot: this rank's shard
    float* xp[kMaxPeers] = {};                 // every node peer's x at this shard (xp[me] = own)
    const float* gp[kMaxPeers] = {};           // every node peer's g at this shard
    unsigned long long* sig_peer[kMaxPeers] = {};   // every peer's signal array [2][G]
    unsigned long long* sig_me = nullptr;      // this rank's signal array
    unsigned* done = nullptr;                  // this rank's CTA completion counter
    uint32_t* err = nullptr;                   // bit 1 set on a barrier timeout
    unsigned long long epoch = 0;              // monotonically increasing barrier value
    unsigned long long timeout_ns = 20ull * 1000 * 1000 * 1000;   // barrier wait limit (then bit 1 of err)
    int G = 1, me = 0;
};
int launch_peer(int ops, int wire, const PeerArgs& pa, void* stream);
// Fused-mode blocking tail (Fig. 3 average + Fig. 4 re-publish): x_shard = sum_i wire_f32(slot[i]) / den
// stored into every node peer's x (pa.xp), then the end barrier (end row of the signal arrays).
int launch_avg_publish(int wire, const PeerArgs& pa, void* stream);

int set_kernel_impl(int impl);   // returns the previous selection
int current_kernel_impl();       // 0 register path, 1 TMA-staged path
int launch_gather(const float* const* src, const size_t* numel, const size_t* offsets, int count,
                  float* dst, void* stream);
int launch_scatter(const float* src, float* const* dst, const size_t* numel, const size_t* offsets,
                   int count, void* stream);
int launch_checksum(const float* x, int64_t n, uint64_t* out, void* stream);
// Set base[r * row_stride + c] = value for r < rows, c < cols (virtual-cluster barrier pre-set).
int launch_fill_u64(unsigned long long* base, int rows, int row_stride, int cols, unsigned long long value,
                    void* stream);

}  // namespace daso
