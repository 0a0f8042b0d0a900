/*
 * hsim.h — C ABI of the B200-native batched evaluator of the heterogeneity-
 * aware LLM-training simulator of arXiv 2508.05370.
 *
 * The library evaluates millions of candidate mappings of one model onto one
 * heterogeneous cluster.  A candidate = device groups + TP/PP/DP degrees +
 * non-uniform layer / micro-batch split + placement (§3
 * "Device grouping", "Non-uniform workload partitioning"
 * §4 "Input Description [A1, A2]").  For each it predicts one training-
 * iteration time in int64 nanoseconds ("predicting training
 * time") through the five steps of DESIGN.md §1:
 *   (1) partition, (2) per-layer roofline cost, (3) TP / PP-p2p / gradient-
 *   sync alpha-beta collective costs incl. resharding,
 *   (4) 1F1B max-plus schedule, (5) max over DP groups + sync, top-k.
 * The space, the placement rule and every formula are defined in DESIGN.md
 * §2 (readings C.0-C.8, A1-A24); results are bit-exact to the CPU oracle.
 *
 * Conventions
 *   - All structs are POD, little-endian, caller-owned; hsim_create deep-copies
 *     them.  No pointer passed to hsim_create is retained.
 *   - Device buffers (out_ns, out_t_ns, out_idx, cands.idx) are caller-owned
 *     CUDA device memory; `stream` is a cudaStream_t passed as void* (0 = the
 *     legacy default stream).  hsim_eval_batch / hsim_topk enqueue their
 *     kernels and return; they do not wait for the GPU, with one bounded
 *     exception: a block-cyclic list (cands.block > 0) stages its chunk plan
 *     (16 B per block) through a ring of 4 pinned host buffers, so the host
 *     waits if the copy issued 4 such calls earlier has not run yet.  Launch
 *     errors return HSIM_ECUDA; asynchronous faults surface at the caller's
 *     next synchronisation.
 *   - Streams: the handle owns scratch and side streams.  Consecutive calls on
 *     one handle are ordered on the device even when the caller passes
 *     different streams (each call waits for the previous call's completion
 *     event); the caller's outputs are complete when its `stream` reaches the
 *     point after the call.
 *   - A handle may be used by one host thread at a time.  Different handles
 *     are independent (any thread, any device current at hsim_create).
 *   - Errors: a non-zero hsim_status; hsim_last_error() (thread-local) holds a
 *     one-line message naming the SPEC.md error kind where one applies
 *     (MissingField / InvalidValue / DivisibilityViolation, SPEC.md:63;
 *     UnknownGpuType / RailMismatch; NonPositiveBandwidth,
 *     SPEC.md:335).
 *   - Per-candidate status is in-band in the int64 result: >= 0 iteration time
 *     in ns; -1 a stage received < 1 layer; -2 a replica received < 1
 *     micro-batch; -3 some device exceeds its memory capacity (only when
 *     hsim_model_desc.mem_check = 1; DESIGN.md M.1).
 */
#ifndef HSIM_H
#define HSIM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HSIM_OK = 0,
  HSIM_EINVAL = 1, /* invalid descriptor / argument                          */
  HSIM_ENOMEM = 2, /* host or device allocation failed                        */
  HSIM_ECUDA = 3,  /* CUDA launch / copy failed                               */
  HSIM_ERANGE = 4, /* numerator >= 2^53, overflow, index out of range, too big */
  HSIM_ESTATE = 5  /* NULL / destroyed handle                                 */
} hsim_status;

/* layer-op kinds: index of eff_flop / eff_mem */
enum { HSIM_KIND_ATTN = 0, HSIM_KIND_MLP = 1, HSIM_KIND_MOE = 2, HSIM_KIND_EMB = 3, HSIM_KIND_HEAD = 4, HSIM_NKIND = 5 };

#define HSIM_MAX_TYPES 4
#define HSIM_MAX_GPUS_PER_NODE 8
#define HSIM_MAX_HOPS 4
#define HSIM_MAX_LINK_KINDS 4

/* One hop of an interconnect path, as Table 4 lists it:
 * a bandwidth in Gbps, bidirectional aggregate (NVLink, PCIe columns) or
 * per direction (NIC).  Its delay is frame*8/uni-dir Gbps. */
typedef struct { double gbps; int32_t bidir; int32_t _pad; } hsim_hop;

/* A fixed path of 1..4 hops (e.g. GPU->NVSwitch->GPU = 2 NVLink hops;
 * GPU->PCIe switch->NIC = 2 PCIe trips). */
typedef struct { int32_t n_hops; int32_t _pad; hsim_hop hops[HSIM_MAX_HOPS]; } hsim_path;

/* One GPU type and the node type that hosts it (one node type per GPU type):
 * compute (peak x efficiency roofline) + the Table 4 interconnect row. */
typedef struct {
  char name[16];
  double peak_flop_per_ns;          /* dense peak, FLOP/ns (= TFLOP/s x 1000)        */
  double hbm_bytes_per_ns;          /* HBM bandwidth, B/ns (= GB/s)                   */
  double eff_flop[HSIM_NKIND];      /* achieved fraction per layer kind, (0, 1]       */
  double eff_mem[HSIM_NKIND];
  int64_t mem_bytes;                /* capacity in bytes (memory pruning, mem_check)  */
  int32_t gpus_per_node;            /* 1, 2, 4 or 8; == NICs per node (rail-only)     */
  int32_t n_link_kinds;             /* 1..4                                           */
  hsim_path link_kinds[HSIM_MAX_LINK_KINDS];
  int8_t intra_kind[HSIM_MAX_GPUS_PER_NODE][HSIM_MAX_GPUS_PER_NODE]; /* GPU i->j path kind; diagonal ignored */
  hsim_path gpu_nic;                /* GPU -> its rail NIC                            */
  double nic_gbps;                  /* NIC bandwidth per direction                    */
  int64_t nic_delay_ns;             /* NIC processing delay (Table 4 column)          */
} hsim_device_type;

/* Cluster / topology description (PAPER.md:299 (3); rail-only, Fig 2). */
typedef struct {
  int32_t n_device_types;           /* 1..HSIM_MAX_TYPES                              */
  int32_t n_nodes;                  /* 1..4096; node id order = placement order       */
  const hsim_device_type* device_types;
  const int32_t* node_type_of;      /* [n_nodes] device-type index per node           */
  int64_t rail_alpha_ns;            /* rail switch hop latency (>= 0)                 */
  double rail_gbps;                 /* rail switch port rate per direction (> 0)      */
  int64_t frame_bytes;              /* jumbo frame for the delay formula (9200)       */
} hsim_cluster_desc;

/* Model description (Table 5 row) + framework search space
 * (PAPER.md:299 (2), explored per PAPER.md:183 "all possible combinations"). */
typedef struct {
  int32_t layers, hidden, heads, kv_heads, ffn, mlp_mats /* 2 GELU, 3 SwiGLU */, seq, vocab, tied;
  int32_t moe_experts /* 1 = dense */, moe_topk;
  int32_t bpe_act /* bytes per activation / weight element, e.g. 2 */, bpe_grad /* e.g. 4 */;
  int64_t global_batch;
  /* search space (DESIGN.md C.2): */
  int32_t n_bset; int32_t bset[8];            /* micro-batch sizes                            */
  int32_t tpset_mask[HSIM_MAX_TYPES];         /* per type: bit k => TP = 2^k allowed (k <= 3) */
  int32_t n_pset; int32_t pset[16];           /* pipeline depths                              */
  int32_t homo, mixed;                        /* families: type-homogeneous / mixed pipelines */
  int32_t use_all;                            /* every used type fully used                   */
  int32_t r_layer, pmax_perturb, r_batch;     /* perturbation radii / max perturbed depth     */
  /* memory-feasibility pruning (the paper never gates on
   * memory): 1 = a candidate any of whose devices needs more than
   * its type's mem_bytes -- parameters x (bpe_act + bpe_grad + 12 B Adam state)
   * + min(P - s, m) in-flight micro-batches x layers x s b h (10 + 24/t) B of
   * activations (DESIGN.md M.1) -- gets status -3.  0 = off (default). */
  int32_t mem_check;
  /* gradient-sync schedule: 0 = after the barrier at T0,
   * segments in ascending layer order (DESIGN.md C.8, default); 1 = overlapped
   * with the backward: a segment starts once every stage group holding its
   * layers has ended its last backward, segments in descending layer order,
   * FIFO per group (DESIGN.md S.1; Table 1: DP sync is
   * exposed in the backward pass). */
  int32_t sync_overlap;
  /* SURVEY.md §8(f) f4 variants, off when 0 (a zero-initialised descriptor
   * keeps the default path):
   * interleave: 0 or 1 = the non-interleaved 1F1B (DESIGN.md C.7); v = 2..8 =
   *   every pipeline of >= 2 stages runs Megatron-LM's interleaved 1F1B with v
   *   model chunks per stage (DESIGN.md V.2): chunk k of a stage with l layers
   *   holds floor(l/v) + [k < l mod v] layers, virtual stage k P + s = chunk k
   *   of stage s; a stage with fewer than v layers -> status -1, a replica
   *   whose micro-batch count is not a multiple of its depth -> -2.
   * ep_dp: 1 = in single-class MoE templates the experts of a stage are
   *   sharded over every replica's TP group of that stage, g = D tp devices
   *   (DESIGN.md V.3): the all-to-all spans them and couples the replicas
   *   into lockstep, and expert gradients are not all-reduced.
   * mixtp: 1 = add the MIXTP template family (DESIGN.md V.1): one class
   *   whose every stage is a mixed TP group of tp devices, tp/2 of type a and
   *   tp/2 of type a2 > a at the same local base on two nodes (tp >= 2 in both
   *   TP sets, tp/2 | GPUs per node); each op lasts as long as on the slower
   *   type (the bottleneck device, PAPER.md:280 C4); its collectives and p2p
   *   run over the group's two nodes.  Enumerated after the MIXED family of
   *   each micro-batch size.
   * None of them combines with mem_check (HSIM_EINVAL at create) nor with
   * hsim_flow_resim (HSIM_EINVAL); ep_dp does not combine with mixtp. */
  int32_t interleave;
  int32_t ep_dp;
  int32_t mixtp;
  /* gradient buckets per stage group (DESIGN.md B.1;
   * Table 1's "DP frequency 2"): 0 or 1 = one (the segments of
   * C.6), 2 = a stage's l layers sync as two buckets, the lower ceil(l/2) (+ the
   * embedding) and the upper rest (+ the head); with sync_overlap the upper
   * bucket is ready once the last backward has passed it (the backward runs
   * head, layers top-down, embedding).  Not with interleave (HSIM_EINVAL). */
  int32_t sync_buckets;
} hsim_model_desc;

/* Which candidates the t-th work item (t = 0..n-1) evaluates. */
typedef struct {
  const int64_t* idx;  /* != NULL: i = idx[t] (device pointer; explicit list)                   */
  int64_t first;       /* idx == NULL, block == 0: i = first + t (contiguous range)               */
  int64_t block;       /* idx == NULL, block > 0:  i = first + (t / block) * stride + (t % block) */
  int64_t stride;      /*   (block-cyclic shard across GPUs)                                      */
} hsim_cands;

typedef struct hsim_handle hsim_handle;

/* Validates the descriptors, derives per-op durations and link classes, builds
 * the candidate-template tables on the host and copies them to the current
 * CUDA device.  On error *out = NULL and a message is set.
 * Returns HSIM_EINVAL (bad descriptor), HSIM_ERANGE (a numerator >= 2^53, too
 * many link classes / stages), HSIM_ENOMEM, HSIM_ECUDA. */
int hsim_create(const hsim_cluster_desc* cluster, const hsim_model_desc* model, hsim_handle** out);

/* Frees host and device memory.  NULL is a no-op. */
void hsim_destroy(hsim_handle* h);

/* N = number of candidates (linear indices 0..N-1), or -1 for a NULL handle. */
int64_t hsim_space_size(const hsim_handle* h);

/* Number of templates, and the first candidate index of template k
 * (k == n_templates returns N); -1 if out of range.  Host only. */
int64_t hsim_n_templates(const hsim_handle* h);
int64_t hsim_template_first(const hsim_handle* h, int64_t k);

/* Host-side explicit plan of candidate i as a JSON object (template, b,
 * per-class stages (type, tp), layer split, micro-batches per replica,
 * placement, status).  Writes at most cap bytes incl. NUL.
 * HSIM_ERANGE if i is out of range or cap is too small. */
int hsim_decode(const hsim_handle* h, int64_t i, char* json, size_t cap);

/* Enqueues the evaluation of n candidates (see hsim_cands) on `stream`;
 * writes out_ns[t] (device, n int64) = iteration time or a negative status.
 * out_ns may be NULL (then nothing is written; useful for timing only).
 * Indices >= N yield HSIM_ERANGE at enqueue time for range mode; for explicit
 * lists they are written as INT64_MIN. n == 0 is a no-op. */
int hsim_eval_batch(hsim_handle* h, const hsim_cands* cands, int64_t n, int64_t* out_ns, void* stream);

/* Enqueues the evaluation of n candidates and the selection of the k
 * smallest valid results ordered by (time asc, index asc) (DESIGN.md C.8);
 * writes out_t_ns[0..k) and out_idx[0..k) (device); unused slots are
 * (INT64_MAX, -1).  1 <= k <= 1024.  Optionally also writes out_ns if not
 * NULL. */
int hsim_topk(hsim_handle* h, const hsim_cands* cands, int64_t n, int32_t k,
              int64_t* out_t_ns, int64_t* out_idx, int64_t* out_ns, void* stream);

/* Merges nlists top-k lists (device; list l at lists + l*2k holds k times then
 * k indices, each list sorted by (time, index), padded with (INT64_MAX, -1) —
 * the layout of an all_gather of [out_t_ns | out_idx] across ranks) into the
 * global top-k (out_t_ns, out_idx, device).  Used by the multi-GPU sweep after
 * the NCCL all_gather.  1 <= k <= 1024, nlists >= 0. */
int hsim_merge_topk(const int64_t* lists, int32_t nlists, int32_t k, int64_t* out_t_ns, int64_t* out_idx, void* stream);

/* flow-level contention re-simulation of the gradient
 * synchronisation of k candidates (DESIGN.md F.1; "bandwidth
 * contention", :400 flow completion time per flow, :409-412 the slowest flow
 * of a blocking collective gates it; SPEC.md:358-373 fluid max-min).  Every
 * reshard / ring step of the candidate's C.8 sync becomes flows on the
 * rail-only link graph (NVLink ports, GPU-NIC PCIe paths, NIC-rail wires) that
 * share links max-min fairly; a step starts when the previous step's last
 * flow completes.
 *   idx   device, k candidate indices (e.g. hsim_topk's out_idx), 0 <= k <= 1024
 *   out   device, k x 8 int64: status (0, or the candidate's -1 / -2 / -3, or
 *         INT32_MIN for an index out of range), sync_ab (the alpha-beta C.8
 *         sync time beyond T0, = T_iter - T0), sync_flow (the same schedule at
 *         flow level, >= sync_ab), n_flows, then the nearest-rank FCT
 *         percentiles p50, p99, p99.9 and the maximum FCT (ns).
 *   fct   device, k x fct_cap int64 or NULL: each candidate's flow completion
 *         times (unordered; the first min(n_flows, fct_cap)) for a CCDF.
 * Blocking: sizes its scratch from a device-side flow count, so it returns
 * after the work on `stream` has finished.  Models up to 256 layers. */
int hsim_flow_resim(hsim_handle* h, const int64_t* idx, int32_t k, int64_t* out, int64_t* fct, int64_t fct_cap,
                    void* stream);

/* Number of device kernels the last hsim_eval_batch / hsim_topk call launched. */
int32_t hsim_last_launch_count(const hsim_handle* h);

/* Executed 1F1B max-plus cells of the candidates [first, first + n): runs the
 * same device kernels as hsim_eval_batch in a counting mode on the legacy
 * default stream and blocks until they finish.  A pipeline of P stages and m
 * micro-batches has 2 P m cells; the exact steady-regime jumps of DESIGN.md §5
 * skip some of them, and only the cells actually executed are counted (this is
 * the numerator of the ALU-roofline fraction in bench.py).  A re-queued job
 * (lane compaction) is counted once, by its complete run; with the pipeline
 * dedupe on (hsim_set_dedup) a class pipeline shared by several candidates of
 * a batch is run, and counted, once.  Returns -1 on error. */
int64_t hsim_count_cells(const hsim_handle* h, int64_t first, int64_t n);

/* Gradient-sync work of the last hsim_topk call on this handle: with k <= 32
 * and out_ns == NULL the sync runs inside the final kernel, only for candidates
 * whose pipeline time T0 can still enter the top-k (T >= T0; DESIGN.md §5
 * "pruned sync"), and this returns the sum over the synced candidates of
 * their segment bound J = sum_c P_c - C + 1 (the roofline numerator's sync
 * term in bench.py).  -1 when the last call did not prune (out_ns given, k >
 * 32, interleave) or on error.  Blocks until the device is idle. */
int64_t hsim_last_sync_units(const hsim_handle* h);

/* on = 1 (default): a top-k call with k <= 32 and out_ns == NULL computes the
 * gradient sync only for candidates whose pipeline time can still enter the
 * top-k (exact: the same top-k).  on = 0: every candidate's sync is computed
 * (as with out_ns).  HSIM_ESTATE for a NULL handle. */
int hsim_set_prune(hsim_handle* h, int on);

/* on = 1 (default): every call (hsim_eval_batch, hsim_topk, hsim_count_cells)
 * runs the 1F1B recurrence (PAPER.md:186-190 step 4, DESIGN.md C.7) once per
 * DISTINCT class pipeline of a batch instead of once per (candidate, class):
 * a class's T_pipe depends only on (template, class, its layer-boundary
 * digits, its sub-classes' micro-batch counts), so candidates that agree on
 * those share one run through a device hash table (DESIGN.md §5 "pipeline
 * dedupe").  Exact: the same int64 results.  Not used with sync_overlap (S.1
 * needs per-candidate stage ends) or interleave > 1 (V.2), nor when the key
 * does not fit 63 bits (hsim_dedup_active says whether it applies).  on = 0:
 * one run per (candidate, class).  HSIM_ESTATE for a NULL handle. */
int hsim_set_dedup(hsim_handle* h, int on);

/* 1 if calls on this handle currently use the pipeline dedupe (the knob is on
 * and the handle's description allows it), 0 if not, -1 for a NULL handle. */
int hsim_dedup_active(const hsim_handle* h);

/* Message of the last failing call on this thread ("" if none). */
const char* hsim_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* HSIM_H */
