/*
 * daso.h — C ABI of libdaso.so, the B200-native hot path of DASO
 * ("Distributed Asynchronous and Selective Optimization", arXiv 2104.05588).
 *
 * Citations: P:n = line n of the paper text (reference PAPER.md); readings
 * R1..R21 = DESIGN.md §3.  No torch / CUDA / NCCL types appear in any
 * signature: device memory is passed as plain pointers, CUDA streams as
 * `void*` (a cudaStream_t, NULL = legacy default stream), the NCCL unique id
 * as 128 opaque bytes.
 *
 * Conventions for every entry point
 *   - returns a daso_status, never throws, never aborts;
 *   - a failing ctx call stores a message readable with daso_last_error();
 *   - stream-ordered: no host synchronisation on the step path; asynchronous
 *     CUDA / NCCL errors surface as DASO_ERR_CUDA / DASO_ERR_NCCL at the next
 *     call (polled with cudaPeekAtLastError / ncclCommGetAsyncError);
 *   - one ctx per process and rank, bound to the CUDA device current at
 *     daso_init; not thread-safe;
 *   - every rank of the world must make the same sequence of collective calls
 *     (daso_init, daso_local_sync, daso_global_send, daso_global_merge,
 *     daso_step, daso_finalize).
 */
#ifndef DASO_H
#define DASO_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------ status */
typedef enum {
    DASO_OK = 0,
    DASO_ERR_CONFIG = 1,    /* invalid cluster / schedule configuration (R10)   */
    DASO_ERR_RANGE = 2,     /* rank or group index out of range                        */
    DASO_ERR_PROTOCOL = 3,  /* call out of protocol order: merge with nothing due, second send
                               while one is in flight, bind twice, step before bind */
    DASO_ERR_ARGUMENT = 4,  /* null / misaligned pointer, n = 0 where n > 0 is required, bad enum   */
    DASO_ERR_CUDA = 5,      /* a CUDA runtime error (message in daso_last_error)                   */
    DASO_ERR_NCCL = 6,      /* an NCCL error (message in daso_last_error)                          */
    DASO_ERR_NONFINITE = 7  /* the fused non-finite check saw NaN/Inf in the parameters */
} daso_status;

enum { DASO_WARMUP = 0, DASO_CYCLING = 1, DASO_COOLDOWN = 2 };   /* P:97 phases            */
enum { DASO_WIRE_BF16 = 0, DASO_WIRE_FP32 = 1 };                 /* P:86 / P:88, reading R3 */
enum { DASO_MODE_FAITHFUL = 0,  /* v1: rotating group exchange + node broadcast (Fig. 4)   */
       DASO_MODE_SHARDED = 1,   /* v2: node reduce-scatter, shard update, all groups exchange
                                   their shard, node all-gather; numerically the same */
       DASO_MODE_FUSED = 2,     /* v3: the sharded batch with the node tier (gradient reduce over
                                   peers + update/merge/pack + parameter all-gather) in ONE kernel
                                   over NVLink peer memory (CUDA IPC); G <= 8; caller buffers must
                                   be cudaMalloc-backed (torch's default allocator is) or come from
                                   daso_alloc_bind.  (Value 3, an NVSwitch-multicast variant of
                                   round 1, was measured slower and removed: DESIGN.md §7.) */ };

const char* daso_status_string(daso_status s);
const char* daso_version(void);

/* ---------------------------------------------------------------- schedule
 * The warm-up / cycling / cool-down B,S schedule of P:97-99 (§3).  Pure host
 * code, no GPU needed.  Record fields are the per-batch decisions the oracle
 * (oracle/schedule.py) makes; the two must agree bit-exactly.
 */
typedef struct {
    int32_t B_init;           /* batches between global syncs in cycling ("B is specified manually"), >= 1 */
    int32_t S_init;           /* batches to wait for the exchange (the paper's W, Eq. (1)'s S); < 0 selects
                                 max(1, B_init/4) ("an initial value of B/4"); 0 = blocking every B batches */
    int32_t warmup_epochs;    /* blocking epochs at the start, >= 0                                    */
    int32_t cooldown_epochs;  /* blocking epochs at the end, >= 0, warmup + cooldown <= total          */
    int32_t total_epochs;     /* >= 1; epochs past the end stay in cool-down                                 */
    int32_t steps_per_epoch;  /* >= 1; every B of the halving chain B_init, B_init/2, ..., 1 must divide it (R10) */
    int32_t gpus_per_node;    /* G >= 1, sets the rotation period of the active group (R9)              */
} daso_sched_config;

/* One batch's schedule decision.  All fields int64 (plain, padding-free layout). */
typedef struct {
    int64_t step;            /* global batch index k (0-based)                                       */
    int64_t epoch;           /* k / steps_per_epoch                                                  */
    int64_t phase;           /* DASO_WARMUP / DASO_CYCLING / DASO_COOLDOWN                    */
    int64_t B, S;            /* cycling B and S in force at this batch (after any plateau action)    */
    int64_t batch_in_cycle;  /* position in the B-cycle (cycling), 0 in blocking phases              */
    int64_t plateau_action;  /* 0 none, 1 halved, 2 reset to (B_init, S_init) at this batch  */
    int64_t send;            /* 1 = a global sync is issued after this batch's update               */
    int64_t blocking;        /* 1 = that sync is blocking (warm-up/cool-down, or S = 0)       */
    int64_t send_group;      /* active group (local id) of the send, -1 if none (P:79 rotation)      */
    int64_t n_syncs;         /* global syncs issued up to and including this batch                   */
    int64_t merge;           /* 1 = a non-blocking exchange is merged by Eq. (1) in this batch      */
    int64_t merge_S;         /* its S_p (S at send time), 0 if none                                  */
    int64_t merge_group;     /* its group, -1 if none                                                */
    int64_t merge_sent;      /* batch it was sent after, -1 if none                                  */
    int64_t pending;         /* 1 = an exchange is in flight after this batch                        */
    int64_t due;             /* its due batch, -1 if none                                            */
} daso_record;

typedef struct daso_sched daso_sched;

/* Create / advance / destroy a host-only schedule.  `plateau` is consulted only at
 * the first batch of an epoch e >= 1: 1 = the training loss plateaued at the end of
 * epoch e-1; it acts only if epoch e-1 was a cycling epoch.
 * Errors: DASO_ERR_CONFIG (config), DASO_ERR_ARGUMENT (null pointer). */
daso_status daso_sched_create(const daso_sched_config* cfg, daso_sched** out);
daso_status daso_sched_next(daso_sched* s, int plateau, daso_record* out);
daso_status daso_sched_destroy(daso_sched* s);

/* ------------------------------------------------- plateau detector and LR
 * Host-only.  P:162 "When the training loss plateaus, i.e. the training loss is not
 * decreasing by more than a set percentage threshold, the scheduler decreases the
 * learning rate by a set factor"; "decays by a factor of 0.5 when the training
 * cross entropy loss is stable for 5 epochs"; P:99 the same events halve B and S.
 * Reading R20: feed one mean training loss per epoch; an epoch improves iff
 * loss < best - threshold * |best|; `patience` consecutive non-improving epochs set
 * *fired = 1 (then the count restarts).  Pass the result as `plateau` at the next
 * epoch's first daso_step.  Errors: DASO_ERR_CONFIG (patience < 1, threshold < 0),
 * DASO_ERR_NONFINITE (NaN/Inf loss: training diverged). */
typedef struct daso_plateau daso_plateau;
daso_status daso_plateau_create(int patience, double threshold, daso_plateau** out);
daso_status daso_plateau_update(daso_plateau* p, double loss, int* fired);
daso_status daso_plateau_destroy(daso_plateau* p);
/* Learning rate at global batch `step`: linear warm-up from 0 to peak = base_lr * world
 * over warmup_epochs, then peak * factor^n_plateaus. */
daso_status daso_lr_at(int64_t step, int steps_per_epoch, double base_lr, int world, int warmup_epochs,
                       double factor, int n_plateaus, double* out);

/* ------------------------------------------------------------ full context */
typedef struct daso_ctx daso_ctx;

typedef struct {
    int32_t rank;             /* this process's global rank, rank = node * G + local (R9 / SPEC S:38)   */
    int32_t warmup_epochs, cooldown_epochs, total_epochs, steps_per_epoch;  /* as daso_sched_config */
    float   momentum;         /* mu, P:172 uses 0.9 */
    float   weight_decay;     /* wd, P:172 uses 1e-4 */
    int32_t wire;             /* DASO_WIRE_BF16 (default) or DASO_WIRE_FP32 (R3) */
    int32_t mode;             /* DASO_MODE_FAITHFUL / _SHARDED / _FUSED (see the enum above) */
    int32_t check_finite;     /* 1 = fused non-finite flag in every update kernel */
    int32_t nccl_max_ctas;    /* >0: cap NCCL CTAs on the group (side-stream) comm to leave SMs to compute; 0 = NCCL default */
    int32_t exchange;         /* global-tier transport: DASO_EXCH_NCCL = in-place ncclAllGather on the
                                 group comm (side stream); DASO_EXCH_CE = copy-engine pushes into the group members'
                                 CUDA-IPC-mapped slots + stream memory-op flags, no SMs used */
} daso_config;

enum { DASO_EXCH_NCCL = 0, DASO_EXCH_CE = 1 };

/* Fill `out` (128 bytes) with a fresh NCCL unique id.  Call on rank 0 only and
 * broadcast the bytes to every rank (torch.distributed does this in the binding). */
daso_status daso_get_unique_id(void* out128);

/* daso_init(world, gpus_per_node, B, S): collective over all `world` ranks.
 * P = world / gpus_per_node virtual nodes.  Creates the world NCCL communicator
 * from `nccl_uid`, splits it into the node communicator (color = node, key =
 * local; "node-local networks") and the group communicator (color = local,
 * key = node; "groups between GPUs with the same local identifier"),
 * a non-blocking high-priority side stream and its events.
 * Errors: DASO_ERR_CONFIG (world % G != 0, G < 1, B < 1, S > B, schedule config),
 * DASO_ERR_RANGE (rank outside [0, world)), DASO_ERR_ARGUMENT (null), DASO_ERR_NCCL / CUDA. */
daso_status daso_init(daso_ctx** out, int world, int gpus_per_node, int B, int S,
                      const daso_config* cfg, const void* nccl_uid128);

/* n rounded up to a multiple of 64 * gpus_per_node: the bucket capacity the sharded,
 * and fused modes require (shards of n_pad / G elements, 256-byte aligned). */
size_t daso_padded_numel(size_t n, int gpus_per_node);

/* Attach the caller's flat fp32 buckets ("buffer packaging"): params x[n],
 * grads g[n], momentum v[n], device pointers on the ctx's device, 16-byte aligned.
 * DASO_MODE_SHARDED / DASO_MODE_FUSED: each buffer must hold daso_padded_numel(n, G)
 * elements with a zero pad (x, g, v); the faithful mode touches only the first n.
 * DASO_MODE_FUSED: collective over the node — exchanges CUDA IPC handles of x and g
 * with the node peers, which then read g and write x of this rank directly.
 * Caller-owned; they must stay alive and unmoved until daso_finalize.  x must be
 * identical on every rank (R17) and v zero-initialised by the caller.  The library
 * allocates its exchange slot here: [P][seg] wire elements (seg = n_pad in the faithful
 * mode, n_pad / G otherwise; n_pad = n rounded up to 64 * G).  Errors:
 * DASO_ERR_PROTOCOL (bound twice), DASO_ERR_ARGUMENT (null, n = 0, misaligned; in the
 * fused mode: not a device allocation, or memory CUDA IPC cannot export — cuMem /
 * expandable_segments — use daso_alloc_bind), DASO_ERR_CUDA / DASO_ERR_NCCL. */
daso_status daso_bind(daso_ctx* c, float* x, float* g, float* v, size_t n);

/* Allocate the flat buckets x, g, v (daso_padded_numel(n, G) fp32 each, zeroed) with
 * cudaMalloc and bind them; returns the device pointers (owned by the library, valid until
 * daso_finalize).  The fused mode's CUDA IPC export needs cudaMalloc memory: use this when
 * the caller's allocator hands out cuMem memory (e.g. PYTORCH_CUDA_ALLOC_CONF=
 * expandable_segments:True).  Collective over the node in the fused mode.  Errors: as
 * daso_bind. */
daso_status daso_alloc_bind(daso_ctx* c, size_t n, float** x, float** g, float** v);

/* ----- split API (each a collective over the world; what daso_step composes) -----
 * daso_local_sync: g <- sum of g over the node (in place, NCCL all-reduce over
 *   the node communicator; the 1/G of Fig. 2's average is applied by the update).
 * daso_local_update: x, v <- momentum-SGD step with g/G, no communication.
 * daso_global_send(group, S): members of `group` pack their x into their slot
 *   segment (wire cast) and start the group all-gather on the side stream.
 *   S >= 1: non-blocking, merged S batches later by daso_global_merge.
 *   S == 0: blocking sync: wait, average (Fig. 3), node broadcast (Fig. 4).
 *   Errors: DASO_ERR_PROTOCOL if an exchange is in flight; DASO_ERR_RANGE bad group.
 * daso_global_merge: members of the in-flight exchange's group wait for it and apply
 *   Eq. (1) with its S, then broadcast to their node (Fig. 4).
 *   Errors: DASO_ERR_PROTOCOL if nothing is in flight.
 */
daso_status daso_local_sync(daso_ctx* c, void* stream);
daso_status daso_local_update(daso_ctx* c, float lr, void* stream);
daso_status daso_global_send(daso_ctx* c, int group, int S, void* stream);
daso_status daso_global_merge(daso_ctx* c, void* stream);

/* daso_step: one batch of DASO after backward has produced g (Fig. 5):
 * advance the schedule (record in *out if non-null), node all-reduce of g, the fused
 * update (+ Eq. (1) merge if due) (+ wire pack if this rank sends) kernel, node
 * broadcast after a merge, side-stream group all-gather for a send, and — blocking
 * — the average kernel and broadcast.  Sharded / fused modes run the same batch
 * element-sharded over the node; fused puts the whole node tier
 * in one kernel.  Blocking batches of the fused mode (Fig. 3 / Fig. 4): the node-tier
 * kernel only packs (no parameter stores), the group exchange runs, then one kernel averages
 * the P rows of the shard and stores the result into every node peer's x, ending with the
 * node barrier.  With the copy-engine transport the local pack kernel of a blocking batch
 * (G = 1, sharded mode; and the fused node-tier kernel for groups of P >= 3) stores the
 * packed row straight into every group member's slot (environment DASO_BLOCKING_PUSH: 0 never,
 * 1 default, 2 always; DASO_AVG_PUBLISH=ldg|tma selects the tail's store path; all
 * choices give bit-identical results).
 * `lr` is this batch's learning rate; `plateau` as in daso_sched_next.
 * Errors: DASO_ERR_PROTOCOL (not bound; schedule/flight-state mismatch), asynchronous
 * DASO_ERR_CUDA / DASO_ERR_NCCL from earlier work. */
daso_status daso_step(daso_ctx* c, float lr, int plateau, void* stream, daso_record* out);

/* ----- backward-overlapped local sync ("The local networks utilize
 * PyTorch's DistributedDataParallel") -----
 * daso_local_sync_bucket: node all-reduce (sum) of g[offset, offset + count) on a dedicated
 *   node communicator, enqueued on `stream` (typically a comm stream fed by gradient-ready
 *   hooks during backward).  Every rank must issue the same buckets in the same order.
 *   Faithful mode only (DASO_ERR_PROTOCOL otherwise); DASO_ERR_RANGE outside [0, n).
 * daso_step_ex: daso_step with flags; DASO_STEP_GRADS_REDUCED = g already holds the node
 *   sum (the buckets covered [0, n) and `stream` waits on them): skip the node all-reduce. */
enum { DASO_STEP_GRADS_REDUCED = 1 };
daso_status daso_local_sync_bucket(daso_ctx* c, size_t offset, size_t count, void* stream);
daso_status daso_step_ex(daso_ctx* c, float lr, int plateau, int flags, void* stream, daso_record* out);

/* daso_step_host: daso_step fed from HOST memory: copies host_grads[n] (pinned
 * for async) into the bound g on `stream`, runs daso_step, then copies the 4-byte
 * non-finite flag back into *host_flag (if non-null) and synchronises `stream`. */
daso_status daso_step_host(daso_ctx* c, const float* host_grads, float lr, int plateau,
                           void* stream, daso_record* out, uint32_t* host_flag);

/* ----- tracing: CUDA events around every phase of daso_step -----
 * With tracing on, daso_step records an event pair around each phase on the stream
 * that runs it; daso_trace_read synchronises the ctx's streams and returns the summed
 * device durations and the algorithmic byte counts since the last reset.
 * The byte counts are the method's minimum per launch (e.g. K1 = 20 B/param), not
 * measured DRAM traffic. */
typedef struct {
    int64_t steps;
    int64_t kernel_launches;  double kernel_ms;  double kernel_bytes;  /* fused update/merge/pack/average (HBM) */
    int64_t local_ops;        double local_ms;   double local_bytes;   /* node all-reduce / reduce-scatter of g (bus bytes) */
    int64_t node_ops;         double node_ms;    double node_bytes;    /* node broadcast / all-gather of x (bus bytes) */
    int64_t wait_ops;         double wait_ms;                          /* compute-stream time blocked on the exchange */
    int64_t exch_ops;         double exch_ms;    double exch_bytes;    /* side-stream group all-gathers (bytes received) */
    double kernel_nvl_bytes;  /* NVLink bytes per direction of the fused-mode node-tier launches (counted in
                                 kernel_*): (G-1) * 4 B per shard element for each of the peer gradient reads
                                 and the peer parameter stores a launch performs */
} daso_trace;
daso_status daso_trace_enable(daso_ctx* c, int on);
daso_status daso_trace_read(daso_ctx* c, daso_trace* out, int reset);

/* ----- measurement knobs (bench.py, SURVEY §8(d) hidden fraction) -----
 * daso_set_exchange(c, 0) suppresses the side-stream group all-gather (the events that
 *   order it are still recorded): the T_step,without leg of hidden = 1 - (T_with -
 *   T_without) / T_AG,alone.  Nodes are then NOT synchronised — never use it in training.
 *   1 re-enables; any other value only queries.  Returns the previous setting (-1: null c).
 * daso_exchange_alone(c, iters, &ms): collective over the group (every rank must call it);
 *   runs the group all-gather of the bound slot `iters` times back to back on the side
 *   stream with nothing else running (T_AG,alone), returns the mean ms per all-gather
 *   (CUDA events on the side stream; one untimed warm-up).  Synchronises the device.  The
 *   slot's rows are overwritten with every member's current packed row, as in a real send.
 *   0 ms if P = 1.  Errors: DASO_ERR_PROTOCOL (exchange in flight, virtual cluster),
 *   DASO_ERR_ARGUMENT, DASO_ERR_NCCL / CUDA. */
int daso_set_exchange(daso_ctx* c, int enabled);
daso_status daso_exchange_alone(daso_ctx* c, int iters, double* ms_out);

/* Last schedule record and whether an exchange is in flight (host-only, no sync). */
daso_status daso_query(const daso_ctx* c, daso_record* last);
/* Synchronise `stream` and read (then clear) the fused non-finite flag:
 * DASO_ERR_NONFINITE if it was set. */
daso_status daso_check_finite(daso_ctx* c, void* stream);
/* Drain any in-flight exchange, destroy comms / streams / events / slots, free c. */
daso_status daso_finalize(daso_ctx* c);
const char* daso_last_error(const daso_ctx* c);
/* Topology of the ctx: P, G, node, local. */
daso_status daso_topology(const daso_ctx* c, int* P, int* G, int* node, int* local);

/* -------------------------------------------- virtual cluster on ONE GPU (parity harness)
 * W = world virtual ranks (P = world / gpus_per_node nodes x G), all on the CUDA device
 * current at create, each a full ctx running the product batch (daso_step_ex and the same
 * kernels); only the transport is emulated:
 *   - node tier (DASO_MODE_FUSED, G > 1): the fused kernel of every rank reads its node
 *     peers' g and writes their x directly in the sibling ranks' buffers on the same GPU
 *     (Fig. 2 / Fig. 4).  The G kernels of a node run one after another on one
 *     stream; the node's barrier signals are pre-set so no launch ever waits on another;
 *   - global tier: the group all-gather is a device-to-device copy of every
 *     packed row into every group member's slot, issued on `stream` after all ranks' batch;
 *     blocking syncs finish with the average (Fig. 3) after that copy.
 * Stream order provides what the barriers and events provide across GPUs, and the shards
 * are disjoint, so every rank computes what it computes on its own GPU.
 * Modes: DASO_MODE_FUSED with any G <= 8; DASO_MODE_FAITHFUL / _SHARDED only with G = 1
 * (their node tier is NCCL, which cannot loop back on one GPU); else DASO_ERR_CONFIG.
 * Buckets x, g, v (daso_padded_numel(n, G) fp32 each, zeroed; x must be set identical on
 * every rank, R17) are owned by the cluster.  cfg->rank is ignored.
 * daso_vcluster_create: errors as daso_init (CONFIG / RANGE / ARGUMENT), DASO_ERR_CUDA.
 * daso_vcluster_buffers: a rank's device pointers (nullable outputs); DASO_ERR_RANGE.
 * daso_vcluster_rank: the rank's ctx (for daso_trace_* / daso_query / daso_check_finite;
 *   never daso_finalize it), NULL if out of range.
 * daso_vcluster_step: one batch of every rank in rank order (gradients already in each g);
 *   out (nullable) receives world records.  Errors as daso_step; DASO_ERR_PROTOCOL if the
 *   ranks' schedules disagree.
 * daso_vcluster_destroy: synchronise, finalize every rank, free the buckets. */
typedef struct daso_vcluster daso_vcluster;
daso_status daso_vcluster_create(daso_vcluster** out, int world, int gpus_per_node, int B, int S,
                                 const daso_config* cfg, size_t n);
daso_status daso_vcluster_buffers(daso_vcluster* v, int rank, float** x, float** g, float** vb);
daso_ctx* daso_vcluster_rank(daso_vcluster* v, int rank);
daso_status daso_vcluster_step(daso_vcluster* v, float lr, int plateau, void* stream, daso_record* out);
daso_status daso_vcluster_destroy(daso_vcluster* v);
const char* daso_vcluster_last_error(const daso_vcluster* v);

/* ------------------------------------------------------ kernel entry points
 * Stream-ordered launches of the fused sm_100a kernels on caller memory, without
 * communication (what daso_step launches; exported for the 1-GPU parity tests and
 * for callers that bring their own collectives).  All pointers are device pointers,
 * 16-byte aligned; n = number of fp32 parameters.
 *   update:       d = g*gscale + wd*x; v = mu*v + d; x = x - lr*v        (K1)
 *   + merge:      x = x + sum_{i<P} (wire_f32(slot[i]) - x) / (2S + P)   (K3, Eq. (1), delta form)
 *   + pack:       pack_out = wire(x)                                     (K2)
 *   average:      x = sum_{i<P} wire_f32(slot[i]) / P                    (K4, Fig. 3)
 * n = 0 is a successful no-op (pointers are not inspected).
 * slot is P rows of `slot_stride` wire elements (row i = node i).  `wire` is
 * DASO_WIRE_BF16 (uint16 bf16 rows) or DASO_WIRE_FP32 (float rows).  flag (nullable)
 * gets bit 0 set if any written parameter is non-finite. */
daso_status daso_k_update(float* x, float* v, const float* g, size_t n, float lr, float mu, float wd,
                          float gscale, void* pack_out, int wire, uint32_t* flag, void* stream);
daso_status daso_k_update_merge(float* x, float* v, const float* g, size_t n, float lr, float mu, float wd,
                                float gscale, const void* slot, size_t slot_stride, int P, int S,
                                void* pack_out, int wire, uint32_t* flag, void* stream);
daso_status daso_k_merge(float* x, size_t n, const void* slot, size_t slot_stride, int P, int S,
                         void* pack_out, int wire, uint32_t* flag, void* stream);
daso_status daso_k_average(float* x, size_t n, const void* slot, size_t slot_stride, int P, int wire,
                           uint32_t* flag, void* stream);
daso_status daso_k_pack(const float* x, size_t n, void* pack_out, int wire, void* stream);

/* K0 (bind time, "buffer packaging"): gather `count` tensors src[i] (numel[i]
 * fp32 each, device pointers listed in HOST arrays) into dst at offsets[i]
 * (daso_flat_layout), or scatter back (daso_k_scatter).  Order-preserving copies. */
daso_status daso_flat_layout(const size_t* numel, int count, size_t align_elems, size_t* offsets, size_t* total);
daso_status daso_k_gather(const float* const* src, const size_t* numel, const size_t* offsets, int count,
                          float* dst, void* stream);
daso_status daso_k_scatter(const float* src, float* const* dst, const size_t* numel, const size_t* offsets,
                           int count, void* stream);

/* Select how the fused kernels move data; returns the previous selection.
 * 0 = register path everywhere (128-bit LDG/STG), 1 = TMA-staged path everywhere
 * (cp.async.bulk global<->shared through an mbarrier ring, one persistent CTA per SM;
 * for the fused peer kernel the bulk copies read and write NVLink peer memory),
 * 2 = auto (default): register path for the local kernels, TMA for the peer kernel.
 * Identical arithmetic in the same order: results are bit-identical.  Any other value
 * only queries.  Process-wide; default from the environment (DASO_KERNEL=ldg|tma|auto). */
int daso_kernel_impl(int impl);

/* Order-independent 64-bit checksum of the bit patterns of x[n] (sum of the uint32
 * words, mod 2^64), written to *out_dev (device).  Used to check the node-replica
 * invariant (Fig. 4: node GPUs hold bitwise-identical parameters). */
daso_status daso_k_checksum(const float* x, size_t n, uint64_t* out_dev, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DASO_H */
