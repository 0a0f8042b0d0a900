// kernels.cu — the hot path on the B200 (sm_100a).
//
// A call (hsim_eval_batch / hsim_topk / hsim_count_cells) maps its candidate
// list onto 32-candidate chunks that never straddle a template (range and
// block-cyclic lists; explicit lists use 32 consecutive entries) and runs in
// batches of up to 2^17 chunks (one batch unless the scratch cap forces
// more).  Each phase is a small kernel with its own register budget; a
// chunk's 32 lanes occupy 32 scratch "slots":
//
//   K_split   warp per chunk, lane per candidate: decode (mixed-radix digits)
//             + step (1) partition -> compact per-class split in HBM; appends
//             one job segment per (depth P, class) of the chunk's template.
//   K_pipe<P> P = 1..16, one launch per depth present: warp per segment, lane
//             = (candidate, class of depth P) of one template and class;
//             register-resident 1F1B max-plus (step 4) over stage durations
//             (step 2) and p2p costs (step 3) with the exact steady-regime
//             jumps -> T_pipe per class.  P >= 9 on high-priority streams.
//   K_pipe_cont<P>  P = 2..8: the jobs K_pipe<P> re-queued (unsettled after
//             the first block), 32 per warp (lane compaction).
//   K_deep    depth > 16: warp per candidate; the warp sweeps the 1F1B
//             anti-diagonal wavefront, lane = stage, __shfl max-plus.
//   K_sync    thread per candidate: step (5) gradient sync incl. reshard as the
//             T0-independent "extra" (runs concurrently with the 1F1B kernels);
//             K_sync_overlap instead (S.1 mode) after them.
//   K_final   T = max over classes of T_pipe + extra, coalesced int64 store,
//             per-warp top-k lists with a global pruning bound.
//   K_merge   (top-k only, once per call) merges the per-block sorted lists.
// The depth kernels, K_deep and K_sync of a batch run concurrently on fork /
// join side streams.  HSIM_TRACE=1 prints a per-launch timeline.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#include "hsim.h"
#include "hsim_core.cuh"

namespace hsim {

int ensure_block_scratch(hsim_handle* h, size_t entries, int64_t** out);
int ensure_work_scratch(hsim_handle* h, size_t entries, int64_t** out);
int sm_count(const hsim_handle* h);
uint32_t depth_mask(const hsim_handle* h);
int prune_enabled(const hsim_handle* h);
int dedup_enabled(const hsim_handle* h);
int class_max(const hsim_handle* h);
int ensure_hash_scratch(hsim_handle* h, int q, size_t cap, u64** keys, int64_t** res);
int depth_jobs_max(const hsim_handle* h, int P);
int64_t depth_jobs_space(const hsim_handle* h, int P);
int stages_max(const hsim_handle* h);
int sync_overlap(const hsim_handle* h);
int interleave_v(const hsim_handle* h);
int ilv_jobs_max(const hsim_handle* h);
int ilv_depth_max(const hsim_handle* h);
int sync_buckets(const hsim_handle* h);
void set_sync_counter(hsim_handle* h, i64* p);
cudaStream_t side_stream(const hsim_handle* h, int q);
cudaEvent_t fork_event(const hsim_handle* h);
cudaEvent_t join_event(const hsim_handle* h, int q);
cudaEvent_t pool_event(const hsim_handle* h, int q);
constexpr int NSTREAM_FINAL = 19;
i64 host_plan(hsim_handle* h, i64 first, i64 block, i64 stride, i64 n, i64 nr, i64** buf, cudaEvent_t* ev);
i64 range_chunks(const hsim_handle* h, i64 first, i64 n, i64* c0);
void call_begin(hsim_handle* h, cudaStream_t st);
void call_end(hsim_handle* h, cudaStream_t st);
int* grid_cache(hsim_handle* h);
void set_launches(hsim_handle* h, int n);
void set_error(const char* m);

// Optional timeline (env HSIM_TRACE=1, diagnostics only): timing events around
// every launch of a call, printed to stderr as (kernel, stream, start, end) us.
struct Trace {
  static constexpr int MAXE = 256;
  bool on = false;
  int n = 0;
  cudaEvent_t e0[MAXE], e1[MAXE];
  const char* name[MAXE];
  int sid[MAXE];
  cudaEvent_t t0;
  void begin(cudaStream_t st) {
    static int env = -1;
    if (env < 0) env = getenv("HSIM_TRACE") ? 1 : 0;
    on = env == 1;
    n = 0;
    if (!on) return;
    cudaEventCreate(&t0);
    cudaEventRecord(t0, st);
  }
  int pre(const char* nm, int s, cudaStream_t st) {
    if (!on || n >= MAXE) return -1;
    cudaEventCreate(&e0[n]);
    cudaEventCreate(&e1[n]);
    name[n] = nm;
    sid[n] = s;
    cudaEventRecord(e0[n], st);
    return n++;
  }
  void post(int q, cudaStream_t st) {
    if (q >= 0) cudaEventRecord(e1[q], st);
  }
  void dump() {
    if (!on) return;
    cudaDeviceSynchronize();
    for (int q = 0; q < n; ++q) {
      float a = 0, b = 0;
      cudaEventElapsedTime(&a, t0, e0[q]);
      cudaEventElapsedTime(&b, t0, e1[q]);
      fprintf(stderr, "TRACE %-16s s%-2d %9.1f %9.1f %8.1f\n", name[q], sid[q], a * 1e3, b * 1e3, (b - a) * 1e3);
      cudaEventDestroy(e0[q]);
      cudaEventDestroy(e1[q]);
    }
    cudaEventDestroy(t0);
    n = 0;
  }
};
static thread_local Trace g_trace;  // diagnostics only (HSIM_TRACE=1)

constexpr int NT = 128;              // threads per block (phase kernels)
constexpr int MT = 256;              // threads of K_merge
constexpr int KMAX = 1024;           // max k
constexpr i64 CBMAX = 1 << 17;       // chunks per batch (2^22 slots)
constexpr i64 KEY_INF = INT64_MAX;
constexpr i64 LIST_PAD = 0x7F7F7F7F7F7F7F7FLL;  // memset(0x7F) sentinel of the per-warp lists
constexpr unsigned FULL = 0xffffffffu;
// counter slots: P (1..FASTP) = work counter of K_pipe<P>; CNT_FULL + P = #jobs of
// depth P in full (32-aligned) chunks, CNT_PART + P = #jobs from partial chunks
constexpr int CNT_DEEP = 17, CNT_NDEEP = 18, CNT_CELLS = 19, CNT_FULL = 20, CNT_PART = 40, CNT_REQ = 55, NCNT = 64;
// V.2 (interleaved 1F1B): #jobs in the K_ilv list, K_ilv's work counter
constexpr int CNT_ILV = 37, CNT_ILVW = 38;
// K_pipe_multi's work counters (depths 1..8, 9..16)
constexpr int CNT_MULTI = 39, CNT_MULTI2 = 0;  // (slot 0: no depth 0)
// re-queued jobs of depth P (lane compaction), P in [2, HSIM_REQ_MAXP]: count at CNT_REQ + P
#ifndef HSIM_REQ_MAXP
#define HSIM_REQ_MAXP 8
#endif
#ifndef HSIM_REQ_MINP
#define HSIM_REQ_MINP 2  // every register depth with enough jobs in the space (HSIM_REQ_MINJOBS)
#endif
#ifndef HSIM_REQ_MINJOBS
#define HSIM_REQ_MINJOBS (1LL << 20)  // ... and depths with few jobs in the space (extra launch, no gain)
#endif
static_assert(CNT_REQ + HSIM_REQ_MAXP < NCNT, "counter layout");
static_assert(FASTP <= 16, "counter layout");

struct Cands {
  const i64* idx;
  i64 first, block, stride, n;
  const i64* plan;   // device [c0 (nr) | pre (nr + 1)] (block-cyclic lists)
  i64 nr;
  i64 c0;            // contiguous range (block == 0): chunk of its first candidate (no staged plan)
};

__device__ __forceinline__ i64 cand_index(const Cands& c, i64 t) {
  if (c.idx) return c.idx[t];
  if (c.block == 0) return c.first + t;
  return c.first + (t / c.block) * c.stride + (t % c.block);
}

// per-batch scratch, indexed by slot = (chunk - first chunk of the batch) * 32 + lane
struct Scratch {
  i64* tpos;          // [ns] position t in the call's candidate list, -1 = empty slot
  int32_t* tau;       // [ns] template index, -1 = none / index out of range
  int32_t* status;    // [ns] 0 ok, -1 / -2 invalid split
  u32* dig;           // [MAXC][ns]
  int32_t* q;         // [MAXC][ns]
  int32_t* seats;     // [MAXC][ns]
  int32_t* add;       // [MAXC][ns]
  int32_t* rm;        // [ns] (last class)
  i64* Tc;            // [MAXC][ns] max T_pipe over the class's sub-classes
  i64* extra;         // [ns] gradient-sync time beyond T0 (C.8), by K_sync
  i64* Rs;            // [spmax][ns] overlap mode (S.1): end of each stage's last backward; else nullptr
  i64* req[HSIM_REQ_MAXP + 1];  // per depth: re-queued jobs (slot << 16 | u << 4 | class)
  i64 req_cap[HSIM_REQ_MAXP + 1];
  int32_t* deep;      // [ns] slots with a class deeper than FASTP (compacted)
  int32_t* ilv;       // V.2: jobs (slot << 2 | class) of interleaved pipelines (P >= 2), or nullptr
  int32_t* full[FASTP + 1];  // per depth: jobs (slot << 2 | class) of full chunks, 32-aligned groups
  int32_t* part[FASTP + 1];  // per depth: jobs of partial chunks, packed (dedupe: hash entries of the distinct pipelines)
  unsigned long long* counters;  // [NCNT]
  i64 ns;             // slot capacity (row stride of the [MAXC][ns] arrays)
  // pipeline dedupe, or hkeys == nullptr: open-addressing table
  // of 2^hbits entries (key + 1, 0 = empty) and the T_pipe of each entry;
  // hj[c][slot] = the slot's entry of class c (| HJ_OWN for the slot whose
  // insert created it), -1 = none
  u64* hkeys;
  i64* hres;
  int32_t* hj;        // [MAXC][ns]
  int hbits;
};
constexpr int32_t HJ_OWN = 1 << 30, HJ_MASK = HJ_OWN - 1;

// --- pipeline dedupe keys ------------------------------------------
__device__ __forceinline__ u64 dd_pack(const Tables& T, i64 tau, int c, u32 dig, i64 base, int a, int b) {
  const int sd = T.dd_wt + 2, sm = sd + T.dd_wd, sa = sm + T.dd_wm, sb = sa + T.dd_wu;
  return ((u64)tau | (u64)c << T.dd_wt | (u64)dig << sd | (u64)base << sm | (u64)a << sa | (u64)b << sb) + 1;
}
struct DKey {
  int tau, c, a, b;
  u32 dig;
  i64 base;
};
__device__ __forceinline__ u64 dd_field(u64 v, int sh, int w) { return (v >> sh) & (((u64)1 << w) - 1); }
__device__ __forceinline__ DKey dd_unpack(const Tables& T, u64 key) {
  key -= 1;
  const int sd = T.dd_wt + 2, sm = sd + T.dd_wd, sa = sm + T.dd_wm, sb = sa + T.dd_wu;
  DKey d;
  d.tau = (int)dd_field(key, 0, T.dd_wt);
  d.c = (int)dd_field(key, T.dd_wt, 2);
  d.dig = (u32)dd_field(key, sd, T.dd_wd);
  d.base = (i64)dd_field(key, sm, T.dd_wm);
  d.a = (int)dd_field(key, sa, T.dd_wu);
  d.b = (int)dd_field(key, sb, T.dd_wu);
  return d;
}
// the key of class c's pipeline: base = m of the last sub-class, a / b = the
// sub-classes with m >= base + 2 / base + 1 (a prefix: sub-classes are in
// ascending lowest-replica order and m is non-increasing in the replica)
__device__ __forceinline__ u64 dd_key(const Tables& T, i64 tau, int c, int32_t off, const ClassSplit& cs) {
  const CrecHdr* h = crec_hdr(T, off);
  const int P = h->P, U = h->U;
  const i64 base = mb_of(cs, U == 1 ? 0 : crec_sub(T, off, P, U - 1)[0]);  // sub-class 0 starts at replica 0
  int a = 0, b = 0;
  for (int u = 0; u + 1 < U; ++u) {
    const i64 m = mb_of(cs, crec_sub(T, off, P, u)[0]);
    a += m >= base + 2;
    b += m >= base + 1;
  }
  return dd_pack(T, tau, c, cs.dig, base, a, b);
}
// a ClassSplit reproducing the key's micro-batch vector: sub-class u (lowest
// replica k_u, ascending) gets base + [k_u < k_a] + [k_u < k_b]
__device__ __forceinline__ ClassSplit dd_split(const Tables& T, int32_t off, const DKey& d) {
  const CrecHdr* h = crec_hdr(T, off);
  ClassSplit cs;
  cs.dig = d.dig;
  cs.q = d.base;
  cs.add = 0;
  cs.seats = d.a < h->U ? crec_sub(T, off, h->P, d.a)[0] : h->D;
  cs.rm = d.b < h->U ? crec_sub(T, off, h->P, d.b)[0] : h->D;
  return cs;
}
// Table layout: 2^hbits entries = nb buckets of 32.  A key's home keeps the
// keys of one (template, class, base, a, b) group with consecutive boundary
// digits in consecutive entries (the lanes of a chunk: class-0 digits run
// with the lane), so probes, job reads, result gathers and clears of a warp
// touch one or two lines: offset x = dig + r (r a hash of the group), home
// bucket = hash(group, x >> 5), entry = bucket * 32 + (x & 31).  Probing
// steps by one bucket at the same offset (coalescing kept on collisions);
// after nb steps the offset advances, so the sequence visits every entry.
__device__ __forceinline__ u32 dd_mix32(u32 h) {  // murmur3 finaliser
  h ^= h >> 16;
  h *= 0x85EBCA6Bu;
  h ^= h >> 13;
  h *= 0xC2B2AE35u;
  return h ^ (h >> 16);
}
__device__ __forceinline__ u64 dd_home(const Tables& T, const Scratch& S, u64 key) {
  const u64 kr = key - 1;
  const int sd = T.dd_wt + 2;
  const u64 dmask = (((u64)1 << T.dd_wd) - 1) << sd;
  const u32 dig = (u32)((kr & dmask) >> sd);
  const u64 g = kr & ~dmask;
  const u32 h = dd_mix32((u32)g * 0x9E3779B1u ^ (u32)(g >> 32) * 0x7FEB352Du);
  const u32 x = dig + (h & 31);
  const u32 bk = dd_mix32(h ^ (x >> 5) * 0x27D4EB2Fu) >> (32 - (S.hbits - 5));
  return (u64)bk << 5 | (x & 31);
}
__device__ __forceinline__ u64 dd_step(const Scratch& S, u64 e, u64& j) {
  const u64 nb = (u64)1 << (S.hbits - 5);
  ++j;
  u64 o = e & 31;
  if ((j & (nb - 1)) == 0) o = (o + 1) & 31;
  return (((e >> 5) + 1) & (nb - 1)) << 5 | o;
}
// insert-or-find along the probe sequence from its j-th entry e; returns the
// entry, *own = the insert created it
__device__ __forceinline__ int dd_insert(const Scratch& S, u64 key, u64 e, u64 j, bool* own) {
  for (;;) {
    const u64 v = __ldcg(&S.hkeys[e]);
    if (v == key) { *own = false; return (int)e; }
    if (v == 0) {
      const u64 prev = atomicCAS((unsigned long long*)&S.hkeys[e], 0ull, (unsigned long long)key);
      if (prev == 0) { *own = true; return (int)e; }
      if (prev == key) { *own = false; return (int)e; }
    }
    e = dd_step(S, e, j);
  }
}

__device__ __forceinline__ ClassSplit load_split(const Scratch& S, int c, int C, i64 t) {
  ClassSplit cs;
  cs.dig = S.dig[c * S.ns + t];
  cs.q = S.q[c * S.ns + t];
  cs.seats = S.seats[c * S.ns + t];
  cs.add = S.add[c * S.ns + t];
  cs.rm = c == C - 1 ? S.rm[t] : 0;
  return cs;
}

// first stage of class c among the template's stages (row of S.Rs)
__device__ __forceinline__ int class_stage_off(const Tables& T, const TplRec& tp, int c) {
  int off = 0;
  for (int q = 0; q < c; ++q) off += crec_hdr(T, tp.crec[q])->P;
  return off;
}

__device__ void load_tables(Tables& sT, const Tables* __restrict__ gT) {
  const int words = sizeof(Tables) / 8;
  const i64* src = (const i64*)gT;
  i64* dst = (i64*)&sT;
  for (int w = threadIdx.x; w < words; w += blockDim.x) dst[w] = src[w];
  __syncthreads();
}

__device__ __forceinline__ i64 warp_sum(i64 v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, (long long)v, o);
  return v;
}

// steps a0 + a1 for a C-class template; stores the compact split of each class
template <int C, bool ILV>
__device__ __forceinline__ int split_store(const Tables& T, const TplRec& tp, i64 tau, i64 local, const Scratch& S, i64 slot,
                                           u64 (&kk)[MAXC], int (&Pk)[MAXC]) {
  ClassSplit cs[C];
  const int st = partition_c<C, ILV>(T, tp, local, cs);
  if (st == 0) {
#pragma unroll
    for (int k = 0; k < C; ++k) {
      S.dig[k * S.ns + slot] = cs[k].dig;
      S.q[k * S.ns + slot] = (int32_t)cs[k].q;
      S.seats[k * S.ns + slot] = (int32_t)cs[k].seats;
      S.add[k * S.ns + slot] = (int32_t)cs[k].add;
      if (!ILV && S.hkeys) {
        kk[k] = dd_key(T, tau, k, tp.crec[k], cs[k]);
        Pk[k] = crec_hdr(T, tp.crec[k])->P;
      }
    }
    S.rm[slot] = (int32_t)cs[C - 1].rm;
  }
  return st;
}

// ---- K_split -------------------------------------------------------------------
#ifndef HSIM_SPLIT_MINB
#define HSIM_SPLIT_MINB 8  // measured with the dedupe: 8 beats 6 on configs 2-4 (0.301 -> 0.296 ms on config 2)
#endif
// ILV: V.2 (interleaved schedule) compiled in -- its partition rules and the
// K_ilv job list; the default path carries none of it
template <bool ILV>
__global__ void __launch_bounds__(NT, HSIM_SPLIT_MINB) k_split(const Tables* __restrict__ gT, Cands c, i64 ca, i64 cb, Scratch S,
                                              uint32_t pm_all) {
  __shared__ Tables sT;
  load_tables(sT, gT);
  const int lane = threadIdx.x & 31;
  const i64 nwarp = (i64)gridDim.x * (NT / 32);
  for (i64 item = ca + (i64)blockIdx.x * (NT / 32) + (threadIdx.x >> 5); item < cb; item += nwarp) {
    const i64 slot = (item - ca) * 32 + lane;
    i64 t = -1, i = -1, tau = -1;
    if (c.idx) {
      t = item * 32 + lane;
      if (t < c.n) {
        i = c.idx[t];
        if (i >= 0 && i < sT.N) tau = find_template(sT, i);
      } else {
        t = -1;
      }
    } else {
      i64 r = 0, g = c.c0 + item;
      if (c.block) {
        const i64* c0 = c.plan;
        const i64* pre = c.plan + c.nr;
        r = bsearch_le(pre, c.nr, item);
        g = c0[r] + (item - pre[r]);
      }
      const i64 tg = find_template_of_chunk(sT, g);
      const i64 lo = sT.tpl_prefix[tg] + (g - sT.tpl_cprefix[tg]) * CHUNK;
      const i64 start = c.block ? c.first + r * c.stride : c.first;
      const i64 len = c.block ? imin(c.block, c.n - r * c.block) : c.n;
      const i64 end = imin(start + len, sT.tpl_prefix[tg + 1]);
      if (lo + lane >= start && lo + lane < end) {
        i = lo + lane;
        tau = tg;
        t = (c.block ? r * c.block : 0) + (i - start);
      }
    }
    S.tpos[slot] = t;
    S.tau[slot] = (int32_t)tau;
    int st = 1;
    uint32_t mypm = 0;
    u64 kk[MAXC] = {0, 0, 0, 0};  // dedupe keys of the classes (0: none) and their depths
    int Pk[MAXC] = {0, 0, 0, 0};
    if (tau >= 0) {
      const TplRec& tp = sT.tpl[tau];
      // class count specialised: the per-class split stays in registers
      switch (tp.C) {
        case 1: st = split_store<1, ILV>(sT, tp, tau, i - tp.prefix, S, slot, kk, Pk); break;
        case 2: st = split_store<2, ILV>(sT, tp, tau, i - tp.prefix, S, slot, kk, Pk); break;
        case 3: st = split_store<3, ILV>(sT, tp, tau, i - tp.prefix, S, slot, kk, Pk); break;
        default: st = split_store<4, ILV>(sT, tp, tau, i - tp.prefix, S, slot, kk, Pk); break;
      }
      S.status[slot] = st;
      if (st == 0) mypm = tp.pmask;
    }
    if (!ILV && S.hkeys) {
      // pipeline dedupe: lanes with equal keys share one insert (warp match);
      // the inserts of all classes are in flight at once (probe load, then the
      // CAS of the empty home entries, then the rare collision walks); the
      // creator of an entry appends it to its depth's job list.  Deep classes
      // (P > FASTP) get an entry too (K_deep runs the owner's).
      const int Cw = (int)__reduce_max_sync(FULL, (unsigned)((kk[0] != 0) + (kk[1] != 0) + (kk[2] != 0) + (kk[3] != 0)));
      int ldr[MAXC];
      bool lead[MAXC], own[MAXC];
      u64 e[MAXC], v[MAXC];
#pragma unroll
      for (int k = 0; k < MAXC; ++k) {
        ldr[k] = 0;
        lead[k] = own[k] = false;
        e[k] = v[k] = 0;
        if (k < Cw) {
          ldr[k] = __ffs(__match_any_sync(FULL, kk[k])) - 1;
          lead[k] = kk[k] != 0 && lane == ldr[k];
          if (lead[k]) e[k] = dd_home(sT, S, kk[k]);
        }
      }
#pragma unroll
      for (int k = 0; k < MAXC; ++k)
        if (lead[k]) v[k] = __ldcg(&S.hkeys[e[k]]);
#pragma unroll
      for (int k = 0; k < MAXC; ++k)
        if (lead[k] && v[k] == 0) {
          v[k] = atomicCAS((unsigned long long*)&S.hkeys[e[k]], 0ull, (unsigned long long)kk[k]);
          own[k] = v[k] == 0;
        }
#pragma unroll
      for (int k = 0; k < MAXC; ++k)
        if (lead[k] && !own[k] && v[k] != kk[k]) {
          bool o = false;
          u64 j = 0;
          const u64 e1 = dd_step(S, e[k], j);
          e[k] = (u64)dd_insert(S, kk[k], e1, j, &o);
          own[k] = o;
        }
      bool app[MAXC];
      unsigned bal[MAXC];
      int P0[MAXC];
      bool uni = true;
#pragma unroll
      for (int k = 0; k < MAXC; ++k) {
        app[k] = false;
        bal[k] = 0;
        P0[k] = 0;
        if (k < Cw) {
          const int ek = __shfl_sync(FULL, (int)e[k], ldr[k]);
          e[k] = (u64)ek;
          S.hj[k * S.ns + slot] = kk[k] ? (ek | (own[k] ? HJ_OWN : 0)) : -1;
          app[k] = own[k] && Pk[k] <= FASTP;
          bal[k] = __ballot_sync(FULL, app[k]);
          if (bal[k]) {
            P0[k] = __shfl_sync(FULL, Pk[k], __ffs(bal[k]) - 1);
            uni = uni && __ballot_sync(FULL, app[k] && Pk[k] == P0[k]) == bal[k];
          }
        } else {
          S.hj[k * S.ns + slot] = -1;
        }
      }
      if (uni) {
        // one depth per class (range lists: a chunk is one template): lane k
        // reserves class k's appends, all reservations in flight at once
        unsigned long long o = 0;
#pragma unroll
        for (int k = 0; k < MAXC; ++k)
          if (lane == k && bal[k]) o = atomicAdd(&S.counters[CNT_PART + P0[k]], (unsigned long long)__popc(bal[k]));
#pragma unroll
        for (int k = 0; k < MAXC; ++k) {
          const unsigned long long ok = __shfl_sync(FULL, o, k) + __popc(bal[k] & ((1u << lane) - 1));
          if (app[k]) S.part[P0[k]][ok] = (int32_t)e[k];
        }
      } else {
#pragma unroll
        for (int k = 0; k < MAXC; ++k) {
          unsigned pend = bal[k];
          while (pend) {
            const int src = __ffs(pend) - 1;
            const int PP = __shfl_sync(FULL, Pk[k], src);
            const unsigned bb = __ballot_sync(FULL, app[k] && Pk[k] == PP);
            unsigned long long o = 0;
            if (lane == src) o = atomicAdd(&S.counters[CNT_PART + PP], (unsigned long long)__popc(bb));
            o = __shfl_sync(FULL, o, src) + __popc(bb & ((1u << lane) - 1));
            if (app[k] && Pk[k] == PP) {
              S.part[PP][o] = (int32_t)e[k];
              app[k] = false;
            }
            pend &= ~bb;
          }
        }
      }
    }
    // deep candidates: compacted, warp-aggregated
    const bool deep = (mypm >> (FASTP + 1)) != 0;
    const unsigned dbal = __ballot_sync(FULL, deep);
    if (dbal) {
      unsigned long long off = 0;
      if (lane == 0) off = atomicAdd(&S.counters[CNT_NDEEP], (unsigned long long)__popc(dbal));
      off = __shfl_sync(FULL, off, 0) + __popc(dbal & ((1u << lane) - 1));
      if (deep) S.deep[off] = (int32_t)slot;
    }
    // jobs per (depth, class) present in the chunk: a full chunk (32 jobs of one
    // template and class) keeps its own aligned group of 32, so a K_pipe warp's
    // lanes have near-equal micro-batch counts; partial chunks (small-radix
    // templates) are packed densely
    u64 combos = 0;
    uint32_t ilvc = 0;  // V.2: classes of this lane's candidate that run interleaved (K_ilv)
    if (mypm && (ILV || !S.hkeys))
      for (int k = 0; k < sT.tpl[tau].C; ++k) {
        const int P = crec_hdr(sT, sT.tpl[tau].crec[k])->P;
        if (ILV && P >= 2) ilvc |= 1u << k;
        else if (P <= FASTP) combos |= (u64)1 << ((P - 1) * 4 + k);
      }
    if (ILV && __any_sync(FULL, ilvc != 0))
      for (int k = 0; k < MAXC; ++k) {
        const bool has = ilvc >> k & 1;
        const unsigned bal = __ballot_sync(FULL, has);
        if (!bal) continue;
        unsigned long long o = 0;
        if (lane == 0) o = atomicAdd(&S.counters[CNT_ILV], (unsigned long long)__popc(bal));
        o = __shfl_sync(FULL, o, 0) + __popc(bal & ((1u << lane) - 1));
        if (has) S.ilv[o] = (int32_t)(slot << 2 | k);
      }
    // one list reservation per combo, all of a warp's reservations in flight at
    // once (lane j reserves for the warp's j-th combo), then the appends: the
    // atomics' round trips overlap instead of forming a chain
    u64 all = (u64)__reduce_or_sync(FULL, (unsigned)combos) | (u64)__reduce_or_sync(FULL, (unsigned)(combos >> 32)) << 32;
    while (all) {
      u64 grp = 0, rest = all;
      unsigned long long mine = 0;
      for (int j = 0; j < 32 && rest; ++j) {
        const int bit = __ffsll((long long)rest) - 1;
        rest &= rest - 1;
        grp |= (u64)1 << bit;
        const int cnt = __popc(__ballot_sync(FULL, combos >> bit & 1));
        if (lane == j) mine = atomicAdd(&S.counters[(cnt == 32 ? CNT_FULL : CNT_PART) + bit / 4 + 1], (unsigned long long)cnt);
      }
      all = rest;
      for (int j = 0; grp; ++j) {
        const int bit = __ffsll((long long)grp) - 1;
        grp &= grp - 1;
        const int P = bit / 4 + 1, k = bit & 3;
        const bool has = combos >> bit & 1;
        const unsigned bal = __ballot_sync(FULL, has);
        const unsigned long long o = __shfl_sync(FULL, mine, j) + __popc(bal & ((1u << lane) - 1));
        if (has) (__popc(bal) == 32 ? S.full[P] : S.part[P])[o] = (int32_t)(slot << 2 | k);
      }
    }
  }
}

// ---- K_pipe<P> -------------------------------------------------------------------
#ifndef HSIM_NBATCH
#define HSIM_NBATCH 1  // target number of batches per call (more only when the scratch cap forces it; measured: 1 beats 2 and 3 on config 2 once the deep tails were fixed)
#endif
#ifndef HSIM_PIPE_MINB
#define HSIM_PIPE_MINB 6  // measured with the dedupe: 6 beats 8 (and 4) on configs 2-4
#endif
#ifndef HSIM_SYNC_MINB
#define HSIM_SYNC_MINB 6
#endif
// one work item of depth P: the 32 jobs item * 32 + lane of its list (full
// chunks' aligned groups first, then the packed partial list / the dedupe
// entries); rq: unsettled jobs may re-queue to K_pipe_cont<P>
template <int P>
__device__ __forceinline__ void pipe_item(const Tables& sT, const Scratch& S, i64 item, i64 gfull, i64 npart, bool rq,
                                          i64& cells) {
  const int lane = threadIdx.x & 31;
  const i64 q = item < gfull ? item * 32 + lane : (item - gfull) * 32 + lane;
  if (item >= gfull && q >= npart) return;
  const int job = item < gfull ? S.full[P][q] : S.part[P][q];
  constexpr bool rqP = P >= HSIM_REQ_MINP && P <= HSIM_REQ_MAXP;
  if (S.hkeys) {  // dedupe: job = a distinct pipeline's table entry
    const DKey d = dd_unpack(sT, __ldcg(&S.hkeys[job]));
    const int32_t off = sT.tpl[d.tau].crec[d.c];
    const DeferCtx dc{rqP ? S.req[rqP ? P : 0] : nullptr, &S.counters[CNT_REQ + (rqP ? P : 0)], rqP ? S.req_cap[rqP ? P : 0] : 0,
                      (i64)job << 16 | d.c};
    const PipeOut r = class_pipes_inl<P>(sT, off, dd_split(sT, off, d), nullptr, 0, rqP && rq ? &dc : nullptr);
    S.hres[job] = r.T0;
#ifdef HSIM_WARPCELLS
    cells += 32 * __reduce_max_sync(__activemask(), (unsigned)r.cells);
#else
    cells += r.cells;
#endif
    return;
  }
  const int c = job & 3;
  const i64 slot = job >> 2;
  const int tau = S.tau[slot];
  if (tau < 0 || S.status[slot] != 0) return;
  const TplRec& tp = sT.tpl[tau];
  i64* R = S.Rs ? S.Rs + (i64)class_stage_off(sT, tp, c) * S.ns + slot : nullptr;
  // depths gated off on the host have req_cap 0: the re-queue attempt fails
  // and the lane continues in place (rare: only unsettled jobs try)
  const DeferCtx dc{rqP ? S.req[rqP ? P : 0] : nullptr, &S.counters[CNT_REQ + (rqP ? P : 0)], rqP ? S.req_cap[rqP ? P : 0] : 0,
                    slot << 16 | c};
  const PipeOut r = class_pipes_inl<P>(sT, tp.crec[c], load_split(S, c, tp.C, slot), R, S.ns, rqP && rq ? &dc : nullptr);
  S.Tc[c * S.ns + slot] = r.T0;
#ifdef HSIM_WARPCELLS  // diagnostic: count mode reports warp-slot cells (32 x warp max)
  cells += 32 * __reduce_max_sync(__activemask(), (unsigned)r.cells);
#else
  cells += r.cells;
#endif
}

template <int P>
__global__ void __launch_bounds__(NT, P <= 4 ? HSIM_PIPE_MINB : 1) k_pipe(const Tables* __restrict__ gT, Scratch S, int count) {
  __shared__ Tables sT;
  load_tables(sT, gT);
  const int lane = threadIdx.x & 31;
  const i64 nfull = (i64)S.counters[CNT_FULL + P], npart = (i64)S.counters[CNT_PART + P];
  const i64 gfull = nfull / 32, items = gfull + (npart + 31) / 32;
  i64 cells = 0;
  for (;;) {
    i64 item = 0;
    if (lane == 0) item = (i64)atomicAdd(&S.counters[P], 1ull);
    item = __shfl_sync(FULL, item, 0);
    if (item >= items) break;
    pipe_item<P>(sT, S, item, gfull, npart, true, cells);
  }
  if (count) {
    cells = warp_sum(cells);
    if (lane == 0 && cells) atomicAdd(&S.counters[CNT_CELLS], (unsigned long long)cells);
  }
}

// K_pipe_multi: the register depths in `mask` (those with few jobs in the
// space) in ONE launch instead of one each: a warp takes the next item of a
// combined queue, deepest first (the longest chains start first), and runs
// it with that depth's code.  Saves the staggered dispatch of many
// latency-bound launches (~3.5 us apart on the front end); no re-queue.
// Two instances: depths 1..8 and 9..16 (measured: one kernel for both
// groups costs config 3 12.4 -> 14.9 ms; either group alone does not).
template <int PLO, int PHI>
__global__ void __launch_bounds__(NT, 1) k_pipe_multi(const Tables* __restrict__ gT, Scratch S, int count, uint32_t mask) {
  __shared__ Tables sT;
  load_tables(sT, gT);
  const int lane = threadIdx.x & 31;
  i64 cells = 0;
  for (;;) {
    i64 item = 0;
    if (lane == 0) item = (i64)atomicAdd(&S.counters[PLO == 1 ? CNT_MULTI : CNT_MULTI2], 1ull);
    item = __shfl_sync(FULL, item, 0);
    int P = 0;
    i64 gfull = 0, npart = 0;
    for (int d = PHI; d >= PLO; --d) {
      if (!(mask >> d & 1)) continue;
      const i64 nf = (i64)S.counters[CNT_FULL + d], np = (i64)S.counters[CNT_PART + d];
      const i64 it = nf / 32 + (np + 31) / 32;
      if (item < it) {
        P = d;
        gfull = nf / 32;
        npart = np;
        break;
      }
      item -= it;
    }
    if (!P) break;
    if constexpr (PLO == 1) {
      switch (P) {
#define HSIM_MC(PP) case PP: pipe_item<PP>(sT, S, item, gfull, npart, false, cells); break;
        HSIM_MC(1) HSIM_MC(2) HSIM_MC(3) HSIM_MC(4) HSIM_MC(5) HSIM_MC(6) HSIM_MC(7) HSIM_MC(8)
        default: break;
      }
    } else {
      switch (P) {
#if HSIM_FASTP >= 16
        HSIM_MC(9) HSIM_MC(10) HSIM_MC(11) HSIM_MC(12) HSIM_MC(13) HSIM_MC(14) HSIM_MC(15) HSIM_MC(16)
#endif
#undef HSIM_MC
        default: break;
      }
    }
  }
  if (count) {
    cells = warp_sum(cells);
    if (lane == 0 && cells) atomicAdd(&S.counters[CNT_CELLS], (unsigned long long)cells);
  }
}

// max of (a, slope sa) and (b, slope sb) keeping the operand that wins now
// (ties: the faster-growing one); H = min(H, pairs before the loser catches up)
// -- the symbolic cell of Pipe<P>::sym_cell for the lane-per-stage layout
__device__ __forceinline__ void sym_max(double& a, double& sa, double b, double sb, double& H) {
  const bool bw = b > a || (b == a && sb > sa);
  const double w = bw ? b : a, sw = bw ? sb : sa, l = bw ? a : b, sL = bw ? sa : sb;
  if (sL > sw) H = fmin(H, floor((w - l) / (sL - sw)) - 1.0);
  a = w;
  sa = sw;
}

// ---- K_pipe_cont<P>: the re-queued jobs of depth P, 32 per warp ------------------
template <int P>
__global__ void __launch_bounds__(NT, P <= 4 ? HSIM_PIPE_MINB : 1) k_pipe_cont(const Tables* __restrict__ gT, Scratch S, int count) {
  __shared__ Tables sT;
  load_tables(sT, gT);
  const i64 n = imin((i64)S.counters[CNT_REQ + P], S.req_cap[P]);
  i64 cells = 0;
  for (i64 q = (i64)blockIdx.x * NT + threadIdx.x; q < n; q += (i64)gridDim.x * NT) {
    const i64 v = S.req[P][q];
    const i64 slot = v >> 16;
    const int u = (int)(v >> 4) & 0xfff, c = (int)v & 15;
    if (S.hkeys) {  // dedupe: slot = the pipeline's table entry
      const DKey d = dd_unpack(sT, __ldcg(&S.hkeys[slot]));
      const int32_t off = sT.tpl[d.tau].crec[d.c];
      const PipeOut r = class_pipes_inl<P>(sT, off, dd_split(sT, off, d), nullptr, 0, nullptr, u);
      atomicMax((unsigned long long*)&S.hres[slot], (unsigned long long)r.T0);
      cells += r.cells;
      continue;
    }
    const TplRec& tp = sT.tpl[S.tau[slot]];
    i64* R = S.Rs ? S.Rs + (i64)class_stage_off(sT, tp, c) * S.ns + slot : nullptr;
    const PipeOut r = class_pipes_inl<P>(sT, tp.crec[c], load_split(S, c, tp.C, slot), R, S.ns, nullptr, u);
    atomicMax((unsigned long long*)&S.Tc[c * S.ns + slot], (unsigned long long)r.T0);
    cells += r.cells;
  }
  if (count) {
    cells = warp_sum(cells);
    if ((threadIdx.x & 31) == 0 && cells) atomicAdd(&S.counters[CNT_CELLS], (unsigned long long)cells);
  }
}

// ---- K_deep: lane-per-stage wavefront for depth > FASTP --------------------------
// Packs floor(32 / P) sub-classes (same class, same candidate) per pass.
__device__ i64 warp_pipe_class(const Tables& T, int32_t off, const ClassSplit& cs, i64* cells, i64* R, i64 rs) {
  const int lane = threadIdx.x & 31;
  const CrecHdr* h = crec_hdr(T, off);
  const StageRec* st = crec_stages(T, off);
  const int P = h->P, U = h->U;
  const int nseg = 32 / P;
  const int seg = lane / P, s = lane - seg * P;
  // stage durations of this lane's stage (same for every sub-class)
  LayerWalk lw = walk(T, h, cs.dig);
  int l = 0;
  for (int k = 0; k <= s && k < P; ++k) l = lw.next(st);
  const double f = seg < nseg ? (double)((i64)l * st[s].layer_f + st[s].fext) : 0.0;
  const double g = seg < nseg ? (double)((i64)l * st[s].layer_b + st[s].gext) : 0.0;
  double best = 0;
  for (int base = 0; base < U; base += nseg) {
    const int u = base + seg;
    const bool act = seg < nseg && u < U;
    const i64* sub = crec_sub(T, off, P, act ? u : 0);
    LanePipe lp;
    lp.P = P; lp.s = s; lp.lane = lane;
    lp.m = act ? mb_of(cs, sub[0]) : 0;
    if (act && s == 0) *cells += 2 * P * lp.m;
    lp.f = act ? f : 0.0;
    lp.g = act ? g : 0.0;
    lp.cR = act && s + 1 < P ? (double)sub[1 + s] : 0.0;
    lp.cL = act && s > 0 ? (double)sub[s] : 0.0;
    lp.X = 0;
    lp.out = 0;
    const i64 lo = 2 * P - 1;
    const i64 hi = lp.m >= P ? 2 * lp.m : lo;
    i64 totMax = act ? 2 * (lp.m + P - 1) : 0;
    i64 hiMin = act ? hi : INT64_MAX;
    for (int o = 16; o > 0; o >>= 1) {
      totMax = imax(totMax, (i64)__shfl_xor_sync(FULL, (long long)totMax, o));
      hiMin = imin(hiMin, (i64)__shfl_xor_sync(FULL, (long long)hiMin, o));
    }
    // per-lane constants of the two steady level parities (lo = 2P-1 is odd)
    const bool oddS = s & 1;
    const int srcO = oddS ? lane - 1 : lane + 1, srcE = oddS ? lane + 1 : lane - 1;
    const double durO = oddS ? lp.f : lp.g, durE = oddS ? lp.g : lp.f;
    const double cO = oddS ? lp.cR : lp.cL, cE = oddS ? lp.cL : lp.cR;
    const bool kO = !(!oddS && s == P - 1);
    const bool kE = !(oddS ? s == P - 1 : s == 0);
    i64 lv = 0;
    for (; lv < lo && lv < totMax; ++lv) lp.level(lv, false, 0, 0, 0, true);
    auto pair = [&]() {  // levels (odd, even) of the steady range: one shuffle per level
      {
        const double v0 = shfl_d(lp.out, srcO);
        const double e = dmax2(lp.X, kO ? v0 : 0.0) + durO;
        lp.X = e;
        lp.out = e + cO;
      }
      {
        const double v0 = shfl_d(lp.out, srcE);
        const double e = dmax2(lp.X, kE ? v0 : 0.0) + durE;
        lp.X = e;
        lp.out = e + cE;
      }
    };
    // periodic-regime skip (Pipe<P>::block): the nseg sub-classes of the warp
    // skip the same number of pairs, each with its own increment d (read from
    // its stage-0 lane; X and out = X + cE all move by d): a first block of 4
    // pairs tests cyclicity 1 and c | 4, later blocks of 12 pairs c = 1 and
    // c | 12 -- for every active segment at once.
    const int lead = seg < nseg ? seg * P : lane;
    auto blk = [&](int BL) {
      const double x0 = lp.X;
      for (int b = 0; b < BL - 1; ++b) pair();
      const double x1 = lp.X;
      pair();
      lv += 2 * BL;
#ifdef HSIM_NOSKIP
      return false;
#endif
      const i64 left = (hiMin - lv) >> 1;  // remaining whole pairs
      double dd = lp.X - x1, d0 = __shfl_sync(FULL, dd, lead);
      {
        // affine regime (Pipe<P>::affine_horizon, lane = stage): the next pair
        // on (value, slope dd) operands must move X by exactly dd with the
        // slopes reproduced; H = pairs before a losing operand catches up
        double x = lp.X, sx = dd, H = 1e300;
        {
          const double v = shfl_d(lp.out, srcO), sv = shfl_d(sx, srcO);
          if (kO) sym_max(x, sx, v, sv, H);
          x += durO;
        }
        {
          const double v = shfl_d(x + cO, srcE), sv = shfl_d(sx, srcE);
          if (kE) sym_max(x, sx, v, sv, H);
          x += durE;
        }
        if (!act) H = 1e300;
        for (int k = 16; k > 0; k >>= 1) H = fmin(H, __shfl_xor_sync(FULL, H, k));
        if (__all_sync(FULL, !act || (x - lp.X == dd && sx == dd)) && H >= 1.0) {
          const i64 t = (i64)fmin(H, (double)left);
          const double td = (double)t * dd;
          lp.X += td;
          lp.out += td;
          lv += 2 * t;
          if (act && s == 0) *cells -= 2 * P * t;
          return t == left;
        }
      }
      i64 q = -1, len = 1;  // q periods of len pairs, each adding d0
      if (__all_sync(FULL, !act || dd == d0)) {
        q = left;
      } else {
        dd = lp.X - x0;
        d0 = __shfl_sync(FULL, dd, lead);
        if (__all_sync(FULL, !act || dd == d0)) { q = left / BL; len = BL; }
      }
      if (q < 0) return false;
      const i64 r = q * len;
      const double rd = (double)q * d0;
      lp.X += rd;
      lp.out += rd;
      lv += 2 * r;
      if (act && s == 0) *cells -= 2 * P * r;
      return true;
    };
    // lag scan: record X after each of HL pairs (one register per lag per
    // lane), then take the smallest lag c <= HL - 1 over which every active
    // stage moved by its segment's same d (cyclicity c, e.g. c = 7 for seven
    // identical consecutive stages, which c | 4 / c | 12 miss) and jump
    constexpr int HL = 16;
    auto lagscan = [&]() {
      double hx[HL];
#pragma unroll
      for (int b = 0; b < HL; ++b) {
        pair();
        hx[b] = lp.X;
      }
      lv += 2 * HL;
#ifdef HSIM_NOSKIP
      return false;
#endif
      const i64 left = (hiMin - lv) >> 1;
#pragma unroll
      for (int cc = 1; cc < HL; ++cc) {
        const double dd = hx[HL - 1] - hx[HL - 1 - cc], d0 = __shfl_sync(FULL, dd, lead);
        if (__all_sync(FULL, !act || dd == d0)) {
          const i64 q = left / cc;
          const double rd = (double)q * d0;
          lp.X += rd;
          lp.out += rd;
          lv += 2 * q * cc;
          if (act && s == 0) *cells -= 2 * P * q * cc;
          return true;
        }
      }
      return false;
    };
    if (lv + 7 < hiMin && !blk(4)) {
      bool done = false;
      while (!done && lv + 23 < hiMin) {
        done = blk(12);
        if (!done && lv + 2 * HL - 1 < hiMin) done = lagscan();
      }
    }
    for (; lv + 1 < hiMin; lv += 2) pair();
    for (; lv < totMax; ++lv) {
      const bool odd = lv & 1;
      lp.level(lv, lv >= lo && lv < hi, odd ? srcO : srcE, odd ? durO : durE, odd ? cO : cE, odd ? kO : kE);
    }
    if (R) {  // S.1: end of each stage's last op, max over this pass's sub-classes
      double e = act ? lp.X : 0.0;
      for (int q = 1; q < nseg; ++q) e = dmax2(e, __shfl_sync(FULL, act ? lp.X : 0.0, (s + q * P) & 31));
      if (seg == 0) R[s * rs] = base == 0 ? (i64)e : imax(R[s * rs], (i64)e);
    }
    // T_pipe of each job sits on its stage-0 lane
    double v = act && s == 0 ? lp.X : 0.0;
    for (int o = 16; o > 0; o >>= 1) v = dmax2(v, __shfl_xor_sync(FULL, v, o));
    best = dmax2(best, v);
  }
  return (i64)best;
}

// 32 < P <= 64: lane holds stages 2*lane and 2*lane+1 (generic levels only;
// such pipelines are rare).  Stage 2l+1 reads its left input from the same
// lane, stage 2l from lane-1's odd stage; B inputs mirror that.
__device__ i64 warp_pipe_class2(const Tables& T, int32_t off, const ClassSplit& cs, i64* cells, i64* R, i64 rs) {
  const int lane = threadIdx.x & 31;
  const CrecHdr* h = crec_hdr(T, off);
  const StageRec* st = crec_stages(T, off);
  const int P = h->P, U = h->U;
  const int s0 = 2 * lane, s1 = 2 * lane + 1;
  LayerWalk lw = walk(T, h, cs.dig);
  int l0 = 0, l1 = 0;
  for (int k = 0; k <= s1 && k < P; ++k) {
    const int l = lw.next(st);
    if (k == s0) l0 = l;
    if (k == s1) l1 = l;
  }
  const bool a0 = s0 < P, a1 = s1 < P;
  const i64 f0 = a0 ? (i64)l0 * st[s0].layer_f + st[s0].fext : 0, g0 = a0 ? (i64)l0 * st[s0].layer_b + st[s0].gext : 0;
  const i64 f1 = a1 ? (i64)l1 * st[s1].layer_f + st[s1].fext : 0, g1 = a1 ? (i64)l1 * st[s1].layer_b + st[s1].gext : 0;
  i64 best = 0;
  for (int u = 0; u < U; ++u) {
    const i64* sub = crec_sub(T, off, P, u);
    const i64 m = mb_of(cs, sub[0]);
    if (lane == 0) *cells += 2 * P * m;
    const i64 c0R = a0 && s0 + 1 < P ? sub[1 + s0] : 0, c0L = a0 && s0 > 0 ? sub[s0] : 0;
    const i64 c1R = a1 && s1 + 1 < P ? sub[1 + s1] : 0, c1L = a1 ? sub[s1] : 0;
    i64 X0 = 0, X1 = 0, out0 = 0, out1 = 0;
    const i64 total = 2 * (m + P - 1);
    for (i64 lv = 0; lv < total; ++lv) {
      // neighbour exports as of the previous level
      const i64 fromLeft = __shfl_up_sync(FULL, (long long)out1, 1);    // stage 2l-1 (lane-1, odd)
      const i64 fromRight = __shfl_down_sync(FULL, (long long)out0, 1); // stage 2l+2 (lane+1, even)
      const i64 own0 = out0, own1 = out1;
      // odd stage first (descending order): F reads stage s0's previous export
      if (a1) {
        const i64 js = lv - s1, jb = lv - (2 * P - 1 - s1);
        const bool isF = (js >= 0 && lv <= P - 1 && js < m) || (lv >= 2 * P - s1 && !(js & 1) && (js >> 1) < m);
        const bool isB = jb >= 0 && !(jb & 1) && (jb >> 1) < m;
        if (isF || isB) {
          const i64 v = isF ? own0 : (s1 == P - 1 ? 0 : fromRight);
          const i64 e = imax(X1, v) + (isF ? f1 : g1);
          X1 = e;
          out1 = e + (isF ? c1R : c1L);
        }
      }
      if (a0) {
        const i64 js = lv - s0, jb = lv - (2 * P - 1 - s0);
        const bool isF = (js >= 0 && lv <= P - 1 && js < m) || (lv >= 2 * P - s0 && !(js & 1) && (js >> 1) < m);
        const bool isB = jb >= 0 && !(jb & 1) && (jb >> 1) < m;
        if (isF || isB) {
          const i64 v = isF ? (s0 == 0 ? 0 : fromLeft) : (s0 == P - 1 ? 0 : own1);
          const i64 e = imax(X0, v) + (isF ? f0 : g0);
          X0 = e;
          out0 = e + (isF ? c0R : c0L);
        }
      }
    }
    if (R) {  // S.1: end of each stage's last op, max over sub-classes
      if (a0) R[s0 * rs] = u == 0 ? X0 : imax(R[s0 * rs], X0);
      if (a1) R[s1 * rs] = u == 0 ? X1 : imax(R[s1 * rs], X1);
    }
    best = imax(best, __shfl_sync(FULL, (long long)X0, 0));
  }
  return best;
}

// one warp per compacted deep candidate (its deep classes, sub-classes packed)
__global__ void __launch_bounds__(NT) k_deep(const Tables* __restrict__ gT, Scratch S, int count) {
  __shared__ Tables sT;
  load_tables(sT, gT);
  const int lane = threadIdx.x & 31;
  const i64 ndeep = (i64)S.counters[CNT_NDEEP];
  i64 cells = 0;
  for (;;) {
    i64 item = 0;
    if (lane == 0) item = (i64)atomicAdd(&S.counters[CNT_DEEP], 1ull);
    item = __shfl_sync(FULL, item, 0);
    if (item >= ndeep) break;
    const i64 sj = S.deep[item];
    const TplRec& tp = sT.tpl[S.tau[sj]];
    for (int c = 0; c < tp.C; ++c) {
      const int32_t off = tp.crec[c];
      const int P = crec_hdr(sT, off)->P;
      if (P <= FASTP) continue;
      const int32_t hj = S.hkeys ? S.hj[c * S.ns + sj] : -1;
      if (S.hkeys && !(hj & HJ_OWN)) continue;  // dedupe: the entry's creator runs it
      const ClassSplit cs = load_split(S, c, tp.C, sj);
      i64 cl = 0;
      i64* R = S.Rs ? S.Rs + (i64)class_stage_off(sT, tp, c) * S.ns + sj : nullptr;
      const i64 T0 = P <= 32 ? warp_pipe_class(sT, off, cs, &cl, R, S.ns) : warp_pipe_class2(sT, off, cs, &cl, R, S.ns);
      cells += cl;
      if (lane == 0) {
        if (S.hkeys) S.hres[hj & HJ_MASK] = T0;
        else S.Tc[c * S.ns + sj] = T0;
      }
    }
  }
  if (count) {
    cells = warp_sum(cells);
    if (lane == 0 && cells) atomicAdd(&S.counters[CNT_CELLS], (unsigned long long)cells);
  }
}

// ---- K_ilv: interleaved 1F1B (DESIGN.md V.2), warp per (candidate, class) -----
// Megatron-LM's virtual pipeline: stage s runs the table forwards F_tab[0..w),
// w = min(2(P-1-s) + (v-1)P, m v), then pairs (F_tab[w+i], B_tab[i]), then the
// remaining backwards; the tables visit micro-batches in groups of P, chunks
// 0..v-1 (forward) / v-1..0 (backward) within a group (m mod P = 0 is
// checked by the partition).  Lane l owns stages l and l + 32.  The warp
// advances all stages in rounds: a stage runs its next op once the op's input
// exists (produced in an earlier round) -- an as-soon-as-possible order of
// the same max-plus recurrence, so the values do not depend on the rounds.
// A stage keeps the end times of its last Q forward and backward ops in
// shared-memory rings indexed by table position; a consumer reads position x
// of its producer's table, and the producer is then at most P/2 + 1 positions
// ahead (tests/test_ilv_host.py checks every P <= 64, v <= 8 on the host), so
// Q >= P/2 + 2 (a power of two chosen by the host) never overwrites an unread
// slot; a violation would set status -5 (never expected).
__device__ __forceinline__ double ilv_dur(double lf, double ext, int l, int v, int k, bool with_ext) {
  return (double)(l / v + (k < l % v ? 1 : 0)) * lf + (with_ext ? ext : 0.0);
}

// dynamic shared memory per warp: ILV_WORDS(PM, Q, PJ, v) doubles (PM =
// deepest interleaved pipeline, Q = ring length, PJ = deepest pipeline with
// the steady-regime jump and its period history, all from the host)
#define ILV_WORDS(PM, Q, PJ, V) (2 * (PM) * (Q) + (PM) + (PJ) * 2 * (PJ) * (V))
// Exact steady-regime jump (the uniform-shift test of DESIGN.md §5 applied to
// the interleaved schedule): in its steady range [w_s, 2mv - w_s) stage s
// alternates F / B over the table, which repeats every P v positions (m mod P
// = 0), so its ops repeat with period L2 = 2 P v.  Each stage compares every
// steady op with the same op one period earlier (a history of L2 ends); once
// the last L2 ops of EVERY stage are the previous period's shifted by one
// common d, every later period is too (the max-plus recurrence is homogeneous
// and an op's inputs lie within its producer's last period -- the ring lead
// bound), so the warp skips q whole periods at once: ends, rings and history
// += q d, positions += q L2 (q keeps the ring slots aligned; every stage stays
// inside its steady range).
__global__ void __launch_bounds__(NT) k_ilv(const Tables* __restrict__ gT, Scratch S, int count, int PM, int Q, int PJ) {
  __shared__ Tables sT;
  extern __shared__ double ilv_smem[];
  load_tables(sT, gT);
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int v = sT.interleave;
  double* rf = ilv_smem + (size_t)wib * ILV_WORDS(PM, Q, PJ, v);  // [PM][Q] forward ends
  double* rb = rf + PM * Q;                                        // [PM][Q] backward ends
  int* cf = (int*)(rb + PM * Q);                                   // [PM] forwards done per stage
  int* cb = cf + PM;                                               // [PM] backwards done per stage
  double* hist = rb + PM * Q + PM;                                 // [PJ][2 PJ v] last period's ends
  const int HL = 2 * PJ * v;                                       // history row length
  const i64 njobs = (i64)S.counters[CNT_ILV];
  i64 cells = 0;
  for (;;) {
    i64 item = 0;
    if (lane == 0) item = (i64)atomicAdd(&S.counters[CNT_ILVW], 1ull);
    item = __shfl_sync(FULL, item, 0);
    if (item >= njobs) break;
    const int job = S.ilv[item];
    const int c = job & 3;
    const i64 slot = job >> 2;
    if (S.status[slot] != 0) continue;
    const TplRec& tp = sT.tpl[S.tau[slot]];
    const int32_t off = tp.crec[c];
    const CrecHdr* h = crec_hdr(sT, off);
    const StageRec* st = crec_stages(sT, off);
    const int P = h->P, U = h->U;
    const ClassSplit cs = load_split(S, c, tp.C, slot);
    i64* R = S.Rs ? S.Rs + (i64)class_stage_off(sT, tp, c) * S.ns + slot : nullptr;
    // this lane's stages: layers and per-op constants
    int ls[2] = {0, 0};
    {
      LayerWalk lw = walk(sT, h, cs.dig);
      for (int q = 0; q < P; ++q) {
        const int l = lw.next(st);
        if (q == lane) ls[0] = l;
        if (q == lane + 32) ls[1] = l;
      }
    }
    const int pv = P * v, L2 = 2 * pv;
    const bool jump = P <= PJ;
    // ring slots stay aligned when q P v = 0 mod Q: q a multiple of qstep
    const int qstep = Q >> min(__ffs(pv) - 1, __ffs(Q) - 1);
    double best = 0;
    bool bad = false;
    for (int u = 0; u < U; ++u) {
      const i64* sub = crec_sub(sT, off, P, u);
      const i64 m = mb_of(cs, sub[0]);
      const i64 n = m * v;
      const double cw = (double)sub[P];
      // per owned stage: op position, table positions done (and their (micro-
      // batch within group, chunk) digits), clock, warm-up, period bookkeeping
      i64 p[2] = {0, 0}, nf[2] = {0, 0}, nb[2] = {0, 0}, w[2] = {0, 0};
      int fj[2] = {0, 0}, fk[2] = {0, 0}, bj[2] = {0, 0}, bk[2] = {0, 0}, hp[2] = {0, 0}, runS[2] = {0, 0};
      double X[2] = {0, 0}, dS[2] = {-1.0, -1.0};
#pragma unroll
      for (int o = 0; o < 2; ++o) {
        const int s = lane + 32 * o;
        w[o] = s < P ? imin(2 * (P - 1 - s) + (i64)(v - 1) * P, n) : 0;
      }
      for (int q = lane; q < P; q += 32) { cf[q] = 0; cb[q] = 0; }
      __syncwarp();
      for (;;) {
        bool act = false, run[2] = {false, false};
        double ne[2] = {0, 0};
        bool isF[2] = {false, false};
        i64 ix[2] = {0, 0};
#pragma unroll
        for (int o = 0; o < 2; ++o) {
          const int s = lane + 32 * o;
          if (s >= P || p[o] >= 2 * n) continue;
          act = true;
          const bool f = p[o] < w[o] || (p[o] < 2 * n - w[o] && !((p[o] - w[o]) & 1));
          const i64 idx = f ? nf[o] : nb[o];
          const int k = f ? fk[o] : v - 1 - bk[o];
          int ps = -1;
          i64 x = 0;
          double cost = 0;
          bool fring = f;
          if (f) {
            if (s > 0) { ps = s - 1; x = idx; cost = (double)sub[s]; }
            else if (k > 0) { ps = P - 1; x = idx - P; cost = cw; }
          } else {
            if (s < P - 1) { ps = s + 1; x = idx; cost = (double)sub[1 + s]; }
            else if (k < v - 1) { ps = 0; x = idx - P; cost = cw; }
            else { ps = s; fring = true; x = idx + (i64)(v - 1) * P; cost = 0; }  // its own F(v-1, j)
          }
          double tin = 0;
          if (ps >= 0) {
            const int have = fring ? cf[ps] : cb[ps];
            if (have <= x) continue;  // input not produced yet
            if (have - x > Q) bad = true;
            tin = (fring ? rf : rb)[ps * Q + (int)(x & (Q - 1))] + cost;
          }
          const bool ext = (s == 0 && k == 0) || (s == P - 1 && k == v - 1);
          const double dur = f ? ilv_dur((double)st[s].layer_f, (double)st[s].fext, ls[o], v, k, ext)
                               : ilv_dur((double)st[s].layer_b, (double)st[s].gext, ls[o], v, k, ext);
          ne[o] = fmax(X[o], tin) + dur;
          run[o] = true;
          isF[o] = f;
          ix[o] = idx;
        }
        if (!__any_sync(FULL, act)) break;
        if (!__any_sync(FULL, run[0] || run[1])) {  // no op could run: a deadlock (never expected)
          bad = true;
          break;
        }
        __syncwarp();
#pragma unroll
        for (int o = 0; o < 2; ++o) {
          if (!run[o]) continue;
          const int s = lane + 32 * o;
          (isF[o] ? rf : rb)[s * Q + (int)(ix[o] & (Q - 1))] = ne[o];
          if (isF[o]) {
            cf[s] = (int)++nf[o];
            if (++fj[o] == P) { fj[o] = 0; if (++fk[o] == v) fk[o] = 0; }
          } else {
            cb[s] = (int)++nb[o];
            if (++bj[o] == P) { bj[o] = 0; if (++bk[o] == v) bk[o] = 0; }
          }
          if (jump) {  // period history of the steady range
            const i64 pp = p[o];
            if (pp >= w[o] && pp < 2 * n - w[o]) {
              double* hrow = hist + s * HL;
              if (pp - L2 >= w[o]) {
                const double d = ne[o] - hrow[hp[o]];
                if (d == dS[o]) ++runS[o];
                else { dS[o] = d; runS[o] = 1; }
              }
              hrow[hp[o]] = ne[o];
              if (++hp[o] == L2) hp[o] = 0;
            } else {
              runS[o] = 0;
            }
          }
          X[o] = ne[o];
          ++p[o];
          ++cells;
        }
        __syncwarp();
        if (jump) {
          const double d0 = __shfl_sync(FULL, dS[0], 0);
          bool ok = true;
#pragma unroll
          for (int o = 0; o < 2; ++o)
            if (lane + 32 * o < P) ok = ok && runS[o] >= L2 && dS[o] == d0;
          if (__all_sync(FULL, ok)) {
            i64 q = INT64_MAX;
#pragma unroll
            for (int o = 0; o < 2; ++o)
              if (lane + 32 * o < P) q = imin(q, (2 * n - w[o] - p[o]) / L2);
            for (int o2 = 16; o2 > 0; o2 >>= 1) q = imin(q, (i64)__shfl_xor_sync(FULL, (long long)q, o2));
            q -= q % qstep;
            if (q > 0) {
              const double add = (double)q * d0;
#pragma unroll
              for (int o = 0; o < 2; ++o) {
                const int s = lane + 32 * o;
                if (s >= P) continue;
                X[o] += add;
                p[o] += q * L2;
                nf[o] += q * pv;
                nb[o] += q * pv;
                cf[s] = (int)nf[o];
                cb[s] = (int)nb[o];
                for (int i = 0; i < Q; ++i) { rf[s * Q + i] += add; rb[s * Q + i] += add; }
                for (int i = 0; i < L2; ++i) hist[s * HL + i] += add;
              }
              __syncwarp();
            }
          }
        }
      }
      // T_pipe = the latest stage end; S.1: every stage's last op (its last backward)
      double mx = fmax(X[0], X[1]);
      for (int o2 = 16; o2 > 0; o2 >>= 1) mx = fmax(mx, __shfl_xor_sync(FULL, mx, o2));
      best = fmax(best, mx);
      if (R)
        for (int o = 0; o < 2; ++o) {
          const int s = lane + 32 * o;
          if (s < P) R[s * S.ns] = u == 0 ? (i64)X[o] : imax(R[s * S.ns], (i64)X[o]);
        }
      __syncwarp();
    }
    if (__any_sync(FULL, bad)) {
      if (lane == 0) S.status[slot] = -5;
    } else if (lane == 0) {
      S.Tc[c * S.ns + slot] = (i64)best;
    }
  }
  if (count) {
    cells = warp_sum(cells);
    if (lane == 0 && cells) atomicAdd(&S.counters[CNT_CELLS], (unsigned long long)cells);
  }
}

// K_sync for the interleaved schedule (C.8: concurrent with K_ilv, T0 = 0;
// S.1: after it, from the stage ends)
__device__ i64 sync_ilv_any(const Tables& T, const TplRec& tp, const Scratch& S, i64 t, const i64* R, i64 T0) {
  switch (tp.C) {
    case 1: { ClassSplit cs[1] = {load_split(S, 0, 1, t)}; return grad_sync_ilv_c<1>(T, tp, cs, R, S.ns, T0); }
    case 2: {
      ClassSplit cs[2] = {load_split(S, 0, 2, t), load_split(S, 1, 2, t)};
      return grad_sync_ilv_c<2>(T, tp, cs, R, S.ns, T0);
    }
    case 3: {
      ClassSplit cs[3] = {load_split(S, 0, 3, t), load_split(S, 1, 3, t), load_split(S, 2, 3, t)};
      return grad_sync_ilv_c<3>(T, tp, cs, R, S.ns, T0);
    }
    default: {
      ClassSplit cs[4] = {load_split(S, 0, 4, t), load_split(S, 1, 4, t), load_split(S, 2, 4, t), load_split(S, 3, 4, t)};
      return grad_sync_ilv_c<4>(T, tp, cs, R, S.ns, T0);
    }
  }
}

__global__ void __launch_bounds__(NT) k_sync_ilv(const Tables* __restrict__ gT, Scratch S, i64 ns, int overlap) {
  __shared__ Tables sT;
  load_tables(sT, gT);
  for (i64 t = (i64)blockIdx.x * NT + threadIdx.x; t < ns; t += (i64)gridDim.x * NT) {
    const int tau = S.tau[t];
    if (tau < 0 || S.status[t] != 0) continue;
    const TplRec& tp = sT.tpl[tau];
    if (tp.D == 1) { S.extra[t] = 0; continue; }
    if (!overlap) {
      S.extra[t] = sync_ilv_any(sT, tp, S, t, nullptr, 0);
      continue;
    }
    i64 T0 = 0;
    for (int q = 0; q < tp.C; ++q) T0 = imax(T0, S.Tc[q * S.ns + t]);
    S.extra[t] = sync_ilv_any(sT, tp, S, t, S.Rs + t, T0) - T0;
  }
}

// ---- per-warp top-k list in global memory: [k times | k indices], sorted ----------
struct WarpTopK {
  i64* wl;
  int k, cnt;
  i64 thrT, thrI;
  unsigned long long* gthr;  // global bound: the k-th time of any full list (>= the global k-th)
};

__device__ void warp_topk_load(WarpTopK& w) {  // lists persist across batches (pad = LIST_PAD)
  const int lane = threadIdx.x & 31;
  int cnt = 0;
  for (int base = 0; base < w.k; base += 32) {
    const int a = base + lane;
    cnt += __popc(__ballot_sync(FULL, a < w.k && w.wl[a] != LIST_PAD));
  }
  w.cnt = cnt;
  w.thrT = w.thrI = KEY_INF;
  if (cnt == w.k) { w.thrT = w.wl[w.k - 1]; w.thrI = w.wl[2 * w.k - 1]; }
}

__device__ __forceinline__ bool key_less(i64 t1, i64 i1, i64 t2, i64 i2) {
  return t1 < t2 || (t1 == t2 && i1 < i2);
}

__device__ void warp_offer(WarpTopK& w, i64 t, i64 i, bool valid) {
  const int lane = threadIdx.x & 31;
  const i64 g = (i64)*(volatile unsigned long long*)w.gthr;
  const bool cand = valid && t <= g && (w.cnt < w.k || key_less(t, i, w.thrT, w.thrI));
  unsigned mask = __ballot_sync(FULL, cand);
  if (!mask) return;
  while (mask) {
    const int src = __ffs(mask) - 1;
    mask &= mask - 1;
    const i64 xt = __shfl_sync(FULL, t, src), xi = __shfl_sync(FULL, i, src);
    if (w.cnt == w.k && !key_less(xt, xi, w.thrT, w.thrI)) continue;
    int p = 0;  // insertion position = #entries < x
    for (int base = 0; base < w.cnt; base += 32) {
      const int a = base + lane;
      const bool lt = a < w.cnt && key_less(w.wl[a], w.wl[w.k + a], xt, xi);
      p += __popc(__ballot_sync(FULL, lt));
    }
    const int last = w.cnt < w.k ? w.cnt : w.k - 1;  // entries [p, last) move up by one
    for (int hiA = last; hiA > p; hiA -= 32) {
      const int a = hiA - 1 - lane;
      i64 vt = 0, vi = 0;
      const bool mv = a >= p;
      if (mv) { vt = w.wl[a]; vi = w.wl[w.k + a]; }
      __syncwarp();
      if (mv) { w.wl[a + 1] = vt; w.wl[w.k + a + 1] = vi; }
      __syncwarp();
    }
    if (lane == 0) { w.wl[p] = xt; w.wl[w.k + p] = xi; }
    __syncwarp();
    if (w.cnt < w.k) w.cnt++;
    if (w.cnt == w.k) { w.thrT = w.wl[w.k - 1]; w.thrI = w.wl[2 * w.k - 1]; }
  }
  if (w.cnt == w.k && lane == 0) atomicMin(w.gthr, (unsigned long long)w.thrT);
}

// ---- K_sync / K_final -----------------------------------------------------------------
template <bool BK>
__device__ i64 sync_any(const Tables& T, const TplRec& tp, const Scratch& S, i64 t, i64 T0) {
  switch (tp.C) {
    case 1: { ClassSplit cs[1] = {load_split(S, 0, 1, t)}; return grad_sync_c<1, BK>(T, tp, cs, T0); }
    case 2: { ClassSplit cs[2] = {load_split(S, 0, 2, t), load_split(S, 1, 2, t)}; return grad_sync_c<2, BK>(T, tp, cs, T0); }
    case 3: {
      ClassSplit cs[3] = {load_split(S, 0, 3, t), load_split(S, 1, 3, t), load_split(S, 2, 3, t)};
      return grad_sync_c<3, BK>(T, tp, cs, T0);
    }
    default: {
      ClassSplit cs[4] = {load_split(S, 0, 4, t), load_split(S, 1, 4, t), load_split(S, 2, 4, t), load_split(S, 3, 4, t)};
      return grad_sync_c<4, BK>(T, tp, cs, T0);
    }
  }
}

// T_iter = T0 + extra with extra = max over runs of consecutive segments
// sharing a group of sum(RS + AR): every segment starts at T0 or when the
// previous one ends (C.8) -- so the sync runs concurrently with the 1F1B
// kernels (grad_sync_c with T0 = 0).
// BK: two gradient buckets per stage group (DESIGN.md B.1)
template <bool BK>
__global__ void __launch_bounds__(NT, HSIM_SYNC_MINB) k_sync(const Tables* __restrict__ gT, Scratch S, i64 ns) {
  __shared__ Tables sT;
  load_tables(sT, gT);
  for (i64 t = (i64)blockIdx.x * NT + threadIdx.x; t < ns; t += (i64)gridDim.x * NT) {
    const int tau = S.tau[t];
    if (tau < 0 || S.status[t] != 0) continue;
    const TplRec& tp = sT.tpl[tau];
    S.extra[t] = tp.D == 1 ? 0 : sync_any<BK>(sT, tp, S, t, 0);
  }
}

// S.1 (overlap mode): after the 1F1B kernels; extra = T_iter - T0 with T_iter
// from the overlapped schedule over the stages' last-backward ends (S.Rs)
template <bool BK>
__device__ i64 sync_overlap_any(const Tables& T, const TplRec& tp, const Scratch& S, i64 t, i64 T0) {
  const i64* R = S.Rs + t;
  switch (tp.C) {
    case 1: { ClassSplit cs[1] = {load_split(S, 0, 1, t)}; return grad_sync_overlap_c<1, BK>(T, tp, cs, R, S.ns, T0); }
    case 2: {
      ClassSplit cs[2] = {load_split(S, 0, 2, t), load_split(S, 1, 2, t)};
      return grad_sync_overlap_c<2, BK>(T, tp, cs, R, S.ns, T0);
    }
    case 3: {
      ClassSplit cs[3] = {load_split(S, 0, 3, t), load_split(S, 1, 3, t), load_split(S, 2, 3, t)};
      return grad_sync_overlap_c<3, BK>(T, tp, cs, R, S.ns, T0);
    }
    default: {
      ClassSplit cs[4] = {load_split(S, 0, 4, t), load_split(S, 1, 4, t), load_split(S, 2, 4, t), load_split(S, 3, 4, t)};
      return grad_sync_overlap_c<4, BK>(T, tp, cs, R, S.ns, T0);
    }
  }
}

template <bool BK>
__global__ void __launch_bounds__(NT) k_sync_overlap(const Tables* __restrict__ gT, Scratch S, i64 ns) {
  __shared__ Tables sT;
  load_tables(sT, gT);
  for (i64 t = (i64)blockIdx.x * NT + threadIdx.x; t < ns; t += (i64)gridDim.x * NT) {
    const int tau = S.tau[t];
    if (tau < 0 || S.status[t] != 0) continue;
    const TplRec& tp = sT.tpl[tau];
    if (tp.D == 1) { S.extra[t] = 0; continue; }
    i64 T0 = 0;
    for (int q = 0; q < tp.C; ++q) T0 = imax(T0, S.Tc[q * S.ns + t]);
    S.extra[t] = sync_overlap_any<BK>(sT, tp, S, t, T0) - T0;
  }
}

constexpr int MW = 32;  // warps of k_merge_small
struct RegTopK {
  i64 t, i;  // this lane's entry
  __device__ __forceinline__ void init() { t = KEY_INF; i = KEY_INF; }
  __device__ __forceinline__ void insert(i64 xt, i64 xi) {
    const int lane = threadIdx.x & 31;
    const int pos = __popc(__ballot_sync(FULL, key_less(t, i, xt, xi)));
    const i64 ut = __shfl_up_sync(FULL, (long long)t, 1), ui = __shfl_up_sync(FULL, (long long)i, 1);
    if (lane == pos) { t = xt; i = xi; }
    else if (lane > pos) { t = ut; i = ui; }
  }
};

// T of one slot (K_final), in two parts so the loop can issue the next
// chunk's loads before it works on this one (software pipelining: K_final is
// bound by memory latency, not bandwidth).  Every scratch word of the slot is
// loaded up front (independent loads, one memory latency instead of a chain);
// rows / words that do not apply to the slot (empty slot, invalid split,
// classes >= C) are read but ignored.
// K_gather (dedupe): T0 of every slot = max over its classes' table entries
// (thread per slot, all loads independent across threads: the gathers of the
// whole batch in flight at once instead of on K_final's per-chunk chain);
// the creator of an entry clears its key for the next call
__global__ void __launch_bounds__(NT) k_gather(Scratch S, i64 ns) {
  for (i64 slot = (i64)blockIdx.x * NT + threadIdx.x; slot < ns; slot += (i64)gridDim.x * NT) {
    int32_t hj[MAXC];
#pragma unroll
    for (int q = 0; q < MAXC; ++q) hj[q] = __ldcs(&S.hj[q * S.ns + slot]);
    i64 T0 = 0;
#pragma unroll
    for (int q = 0; q < MAXC; ++q)
      if (hj[q] >= 0) {
        T0 = imax(T0, __ldcg(&S.hres[hj[q] & HJ_MASK]));
        if (hj[q] & HJ_OWN) S.hkeys[hj[q] & HJ_MASK] = 0;
      }
    S.Tc[slot] = hj[0] >= 0 ? T0 : KEY_INF;  // no valid split: never a warp's best chunk (K_final)
  }
}

struct SlotW {
  i64 t, ex, tc[MAXC];
  int tau, st;
};
__device__ __forceinline__ SlotW slot_load(const Scratch& S, i64 slot) {
  SlotW w;
  w.t = __ldcs(&S.tpos[slot]);
  w.tau = __ldcs(&S.tau[slot]);
  w.st = __ldcs(&S.status[slot]);
  w.ex = __ldcs(&S.extra[slot]);
  if (S.hkeys) {  // dedupe: K_gather left the slot's T0 in row 0
    w.tc[0] = __ldcs(&S.Tc[slot]);
#pragma unroll
    for (int q = 1; q < MAXC; ++q) w.tc[q] = 0;
    return w;
  }
#pragma unroll
  for (int q = 0; q < MAXC; ++q) w.tc[q] = __ldcs(&S.Tc[q * S.ns + slot]);
  return w;
}
__device__ __forceinline__ i64 slot_T(const Tables& sT, const Cands& c, const SlotW& w, i64* t_out, i64* i_out) {
  i64 T = INT64_MIN, i = -1;
  if (w.t >= 0) {
    i = cand_index(c, w.t);
    if (w.tau >= 0) {
      if (w.st) {
        T = w.st;
      } else {
        const int C = sT.tpl[w.tau].C;
        i64 T0 = 0;
#pragma unroll
        for (int q = 0; q < MAXC; ++q)
          if (q < C) T0 = imax(T0, w.tc[q]);
        T = T0 + w.ex;
      }
    }
  }
  *t_out = w.t;
  *i_out = i;
  return T;
}

// k <= 32: each warp keeps its top-k in registers (lane j = j-th entry), warps
// share a global pruning bound, and each block merges its warps into one list
// (lists[block], kept across batches) at the end.
// MODE 0: T = T0 + extra (K_sync / K_sync_overlap ran).  MODE 1 (C.8) / 2
// (S.1), top-k without out_ns: the gradient sync is computed here, and only
// for candidates that can still enter the top-k -- T >= T0, so a candidate
// whose T0 already exceeds the global bound (the k-th best T found so far, an
// upper bound of the final k-th) or its warp list's k-th key is skipped.  Exact:
// the skipped never belong to the top-k; the others get their exact T.
#ifndef HSIM_FINALP_MINB
#define HSIM_FINALP_MINB 4  // pruned K_final: 128 registers (measured: 4 beats 1, 6 and 8 on configs 2-4)
#endif
// offer each lane's (T, i) (valid = a finite key under the global bound) to
// the warp's register top-k: many candidates (early in the scan) are sorted
// across the warp (bitonic, 15 compare-exchange steps) and rank-merged with the
// list, few are inserted one by one; then the global bound is lowered
__device__ __forceinline__ void warp_offer(RegTopK& r, i64 T, i64 i, bool valid, int k, i64 (*bt)[32], i64 (*bi)[32],
                                           unsigned long long* gthr) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  i64 thT = __shfl_sync(FULL, (long long)r.t, k - 1), thI = __shfl_sync(FULL, (long long)r.i, k - 1);
  unsigned cand = __ballot_sync(FULL, valid && key_less(T, i, thT, thI));
  if (!cand) return;
  if (__popc(cand) > 6) {
    const bool mine = cand >> lane & 1;
    i64 bt_ = mine ? T : KEY_INF, bi_ = mine ? i : KEY_INF;
#pragma unroll
    for (int size = 2; size <= 32; size <<= 1)
#pragma unroll
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        const i64 ot = __shfl_xor_sync(FULL, (long long)bt_, stride), oi = __shfl_xor_sync(FULL, (long long)bi_, stride);
        const bool up = (lane & size) == 0, lower = (lane & stride) == 0;
        const bool olt = key_less(ot, oi, bt_, bi_);
        if (lower == up ? olt : !olt && !(ot == bt_ && oi == bi_)) { bt_ = ot; bi_ = oi; }
      }
    // rank merge of the sorted lists A = r (lane j = j-th) and B = (bt_, bi_)
    int lo = 0, hi = 32;  // #B < A[lane]
#pragma unroll
    for (int it = 0; it < 6; ++it) {
      const int mid = (lo + hi) >> 1;
      const int src = mid < 32 ? mid : 31;
      const i64 mt = __shfl_sync(FULL, (long long)bt_, src), mi = __shfl_sync(FULL, (long long)bi_, src);
      if (lo < hi) { if (key_less(mt, mi, r.t, r.i)) lo = mid + 1; else hi = mid; }
    }
    const int pa = lane + lo;
    int lo2 = 0, hi2 = 32;  // #A < B[lane]
#pragma unroll
    for (int it = 0; it < 6; ++it) {
      const int mid = (lo2 + hi2) >> 1;
      const int src = mid < 32 ? mid : 31;
      const i64 mt = __shfl_sync(FULL, (long long)r.t, src), mi = __shfl_sync(FULL, (long long)r.i, src);
      if (lo2 < hi2) { if (key_less(mt, mi, bt_, bi_)) lo2 = mid + 1; else hi2 = mid; }
    }
    const int pb = lane + lo2;
    __syncwarp();
    if (pa < 32) { bt[w][pa] = r.t; bi[w][pa] = r.i; }
    if (pb < 32) { bt[w][pb] = bt_; bi[w][pb] = bi_; }
    __syncwarp();
    r.t = bt[w][lane];
    r.i = bi[w][lane];
    __syncwarp();
    thT = __shfl_sync(FULL, (long long)r.t, k - 1);
  } else {
    while (cand) {
      const int src = __ffs(cand) - 1;
      cand &= cand - 1;
      const i64 xt = __shfl_sync(FULL, (long long)T, src), xi = __shfl_sync(FULL, (long long)i, src);
      if (key_less(xt, xi, thT, thI)) {
        r.insert(xt, xi);
        thT = __shfl_sync(FULL, (long long)r.t, k - 1);
        thI = __shfl_sync(FULL, (long long)r.i, k - 1);
      }
    }
  }
  if (lane == 0 && thT != KEY_INF) atomicMin(gthr, (unsigned long long)thT);
}

// pruned K_final (MODE >= 1): sync the queue's entries [qn - cnt, qn)
// (cnt <= 32), one per lane, each re-checked against the (meanwhile lower)
// bound first, and offer them to the warp's top-k
template <int MODE, bool BK>
__device__ __forceinline__ void drain_sync(const Tables& sT, const Scratch& S, RegTopK& r, int& qn, int cnt, const int32_t* qs,
                                           const i64* q0, const i64* qi, unsigned long long* gthr, int k, i64 (*bt)[32],
                                           i64 (*bi)[32], unsigned long long& nsync) {
  const int lane = threadIdx.x & 31;
  const bool has = lane < cnt;
  const int e = qn - cnt + lane;
  const i64 slot = has ? qs[e] : 0, T0 = has ? q0[e] : KEY_INF, i = has ? qi[e] : KEY_INF;
  __syncwarp();
  qn -= cnt;
  const i64 g = (i64)*(volatile unsigned long long*)gthr;
  const i64 thT = __shfl_sync(FULL, (long long)r.t, k - 1);
  i64 T = KEY_INF;
  if (has && T0 <= g && T0 <= thT) {
    const TplRec& tp = sT.tpl[S.tau[slot]];
    if constexpr (MODE == 1) T = T0 + sync_any<BK>(sT, tp, S, slot, 0);
    else T = sync_overlap_any<BK>(sT, tp, S, slot, T0);
    int sp = 0;
    for (int q = 0; q < tp.C; ++q) sp += crec_hdr(sT, tp.crec[q])->P;
    nsync += (unsigned long long)(sp - tp.C + 1);
  }
  warp_offer(r, T, i, T != KEY_INF && T <= (i64)*(volatile unsigned long long*)gthr, k, bt, bi, gthr);
}

template <int MODE, bool BK, bool BF = false>
__global__ void __launch_bounds__(NT, MODE ? HSIM_FINALP_MINB : 1) k_final_small(const Tables* __restrict__ gT, Cands c, Scratch S, i64 ns,
                                                    i64* __restrict__ out, int k, i64* __restrict__ lists) {
  __shared__ Tables sT;
  __shared__ i64 bt[NT / 32][32], bi[NT / 32][32];
  // MODE >= 1: per-warp queue of the candidates whose sync must be computed
  // (T0 under the bound), drained 32 at a time so the sync runs with every
  // lane busy instead of the few lanes of a chunk that pass the bound
  constexpr int QN = MODE ? 64 : 1;
  __shared__ int32_t qs[NT / 32][QN];
  __shared__ i64 q0[NT / 32][QN], qi[NT / 32][QN];
  load_tables(sT, gT);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const i64 wid = (i64)blockIdx.x * (NT / 32) + w;
  const i64 nw = (i64)gridDim.x * (NT / 32);
  i64* blist = lists + (i64)blockIdx.x * 2 * k;
  unsigned long long* gthr = (unsigned long long*)(lists + (i64)gridDim.x * 2 * k);
  unsigned long long nsync = 0;  // MODE >= 1: sum over the synced candidates of J = sum P - C + 1
  RegTopK r;
  r.init();
  if (w == 0 && lane < k && blist[lane] != LIST_PAD && blist[lane] != KEY_INF) { r.t = blist[lane]; r.i = blist[k + lane]; }
  // launched as a programmatic dependent of K_gather (dedupe mode): the
  // prologue above overlaps its tail; the batch's scratch is read only after
  // K_gather has completed (a no-op for an ordinary launch)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  int qn = 0;  // queued entries (warp-uniform)
  // the warp's chunks first + j * step, j < nch, visited from its best chunk
  // (smallest T0, dedupe mode: K_gather's row) and its sync drained at once:
  // the warp's first synced candidates then set a tight list bound and a tight
  // global bound, instead of whatever its first chunk in index order holds.
  // First batch of a call only (BF): later batches start with the bound the
  // earlier ones left and run the BF = false instance (measured: the scan,
  // and the registers it takes, cost config 3 2-4 % when every batch runs it)
  const i64 first = wid * 32, step = nw * 32;
  const i64 nch = first < ns ? (ns - first + step - 1) / step : 0;
  i64 jbest = 0;
  if (BF && MODE != 0 && S.hkeys && nch > 1) {
    i64 bT = KEY_INF, bj = 0;
#pragma unroll 4
    for (i64 j = 0; j < nch; ++j) {
      const i64 v = __ldcg(&S.Tc[first + j * step + lane]);
      if (v < bT) { bT = v; bj = j; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const i64 ot = __shfl_xor_sync(FULL, (long long)bT, o), oj = __shfl_xor_sync(FULL, (long long)bj, o);
      if (ot < bT || (ot == bT && oj < bj)) { bT = ot; bj = oj; }
    }
    jbest = bj;
  }
  SlotW nxt;
  i64 nbase = first + jbest * step;  // the chunk after the current one (wrapping to the warp's first)
  if (nch > 0) nxt = slot_load(S, nbase + lane);
  for (i64 j = 0; j < nch; ++j) {
    const i64 base = nbase;
    nbase += step;
    if (nbase >= ns) nbase = first;
    const SlotW cur = nxt;
    if (j + 1 < nch) nxt = slot_load(S, nbase + lane);  // next chunk's loads in flight
    i64 t, i;
    const i64 g = (i64)*(volatile unsigned long long*)gthr;
    const i64 thT = __shfl_sync(FULL, (long long)r.t, k - 1), thI = __shfl_sync(FULL, (long long)r.i, k - 1);
    i64 T;
    if constexpr (MODE == 0) {
      T = slot_T(sT, c, cur, &t, &i);
      if (out && t >= 0) out[t] = T;
      warp_offer(r, T, i, t >= 0 && T >= 0 && T <= g, k, bt, bi, gthr);
    } else {
      SlotW z = cur;
      z.ex = 0;
      T = slot_T(sT, c, z, &t, &i);  // T0 (or the status)
      const bool live = t >= 0 && T >= 0 && T <= g && T <= thT;
      const bool needs = live && sT.tpl[cur.tau].D > 1;
      // D = 1: no sync, T = T0 now; D > 1: queued
      warp_offer(r, T, i, live && !needs, k, bt, bi, gthr);
      const unsigned nb = __ballot_sync(FULL, needs);
      if (nb) {
        const int pos = qn + __popc(nb & ((1u << lane) - 1));
        if (needs) {
          qs[w][pos] = (int32_t)(base + lane);
          q0[w][pos] = T;
          qi[w][pos] = i;
        }
        __syncwarp();
        qn += __popc(nb);
        if (qn >= 32) drain_sync<MODE, BK>(sT, S, r, qn, 32, qs[w], q0[w], qi[w], gthr, k, bt, bi, nsync);
      }
      if (BF && j == 0 && qn > 0) drain_sync<MODE, BK>(sT, S, r, qn, qn, qs[w], q0[w], qi[w], gthr, k, bt, bi, nsync);
    }
  }
  if constexpr (MODE != 0) {
    if (qn > 0) drain_sync<MODE, BK>(sT, S, r, qn, qn, qs[w], q0[w], qi[w], gthr, k, bt, bi, nsync);
  }
  bt[w][lane] = r.t;
  bi[w][lane] = r.i;
  __syncthreads();
  if (w == 0) {
    for (int o = 1; o < NT / 32; ++o)
      for (int p = 0; p < k; ++p) {
        const i64 xt = bt[o][p], xi = bi[o][p];
        const i64 thT = __shfl_sync(FULL, (long long)r.t, k - 1), thI = __shfl_sync(FULL, (long long)r.i, k - 1);
        if (xt == KEY_INF || !key_less(xt, xi, thT, thI)) break;
        r.insert(xt, xi);
      }
    if (lane < k) {
      blist[lane] = r.t;
      blist[k + lane] = r.t == KEY_INF ? -1 : r.i;
    }
  }
  if constexpr (MODE != 0) {  // the call's synced segment units (hsim_last_sync_units)
    nsync = warp_sum((i64)nsync);
    if (lane == 0 && nsync) atomicAdd(gthr + 1, nsync);
  }
}

__global__ void __launch_bounds__(NT) k_final(const Tables* __restrict__ gT, Cands c, Scratch S, i64 ns,
                                              i64* __restrict__ out, int k, i64* __restrict__ lists) {
  __shared__ Tables sT;
  load_tables(sT, gT);
  const int lane = threadIdx.x & 31;
  const i64 wid = (i64)blockIdx.x * (NT / 32) + (threadIdx.x >> 5);
  const i64 nw = (i64)gridDim.x * (NT / 32);
  WarpTopK tk{k ? lists + wid * 2 * k : nullptr, k, 0, KEY_INF, KEY_INF,
              k ? (unsigned long long*)(lists + nw * 2 * k) : nullptr};
  if (k) warp_topk_load(tk);
  SlotW nxt;
  if (wid * 32 < ns) nxt = slot_load(S, wid * 32 + lane);
  for (i64 base = wid * 32; base < ns; base += nw * 32) {
    const SlotW cur = nxt;
    if (base + nw * 32 < ns) nxt = slot_load(S, base + nw * 32 + lane);  // next chunk's loads in flight
    i64 t, i;
    const i64 T = slot_T(sT, c, cur, &t, &i);
    if (out && t >= 0) out[t] = T;
    if (k) warp_offer(tk, T, i, t >= 0 && T >= 0);
  }
}

// ---- K_merge: shared-memory running top-k over sorted lists -------------------------
struct TopK {
  i64 lt[KMAX], li[KMAX];   // sorted ascending, `count` valid
  i64 nt[KMAX], ni[KMAX];   // merge target
  i64 bt[MT], bi[MT];       // incoming batch
  int count, nbuf;
};

__device__ void topk_offer(TopK& s, int k, i64 t, i64 i, bool valid) {
  const int tid = threadIdx.x;
  const bool full = s.count >= k;
  const bool cand = valid && (!full || key_less(t, i, s.lt[k - 1], s.li[k - 1]));
  if (!__syncthreads_or(cand)) return;
  if (tid == 0) s.nbuf = 0;
  __syncthreads();
  if (cand) {
    int p = atomicAdd(&s.nbuf, 1);
    s.bt[p] = t;
    s.bi[p] = i;
  }
  __syncthreads();
  const int nb = s.nbuf;
  if (tid >= nb) { s.bt[tid] = KEY_INF; s.bi[tid] = KEY_INF; }
  __syncthreads();
  for (int size = 2; size <= MT; size <<= 1)  // bitonic sort of the batch
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      const int j = tid ^ stride;
      if (j > tid) {
        const bool up = (tid & size) == 0;
        i64 a = s.bt[tid], ai = s.bi[tid], b = s.bt[j], bi = s.bi[j];
        if (key_less(b, bi, a, ai) == up) {
          s.bt[tid] = b; s.bi[tid] = bi; s.bt[j] = a; s.bi[j] = ai;
        }
      }
      __syncthreads();
    }
  // rank merge: list element a -> a + #(batch < it); batch element b -> b + #(list <= it)
  const int cnt = s.count;
  for (int a = tid; a < cnt; a += MT) {
    int lo = 0, hi = nb;
    while (lo < hi) {
      int mid = (lo + hi) >> 1;
      if (key_less(s.bt[mid], s.bi[mid], s.lt[a], s.li[a])) lo = mid + 1; else hi = mid;
    }
    const int pos = a + lo;
    if (pos < k) { s.nt[pos] = s.lt[a]; s.ni[pos] = s.li[a]; }
  }
  if (tid < nb) {
    int lo = 0, hi = cnt;
    while (lo < hi) {
      int mid = (lo + hi) >> 1;
      if (!key_less(s.bt[tid], s.bi[tid], s.lt[mid], s.li[mid])) lo = mid + 1; else hi = mid;
    }
    const int pos = tid + lo;
    if (pos < k) { s.nt[pos] = s.bt[tid]; s.ni[pos] = s.bi[tid]; }
  }
  __syncthreads();
  const int ncnt = min(k, cnt + nb);
  for (int a = tid; a < ncnt; a += MT) { s.lt[a] = s.nt[a]; s.li[a] = s.ni[a]; }
  if (tid == 0) s.count = ncnt;
  __syncthreads();
}

// lists: nblk x [k times | k indices], each sorted, padded with LIST_PAD or
// (INT64_MAX, -1) (the all_gather layout of hsim_merge_topk)
__global__ void __launch_bounds__(MT) k_merge(const i64* __restrict__ blk, int nblk, int k, i64* __restrict__ out_t,
                                              i64* __restrict__ out_i) {
  extern __shared__ __align__(16) unsigned char dyn[];
  TopK& tk = *reinterpret_cast<TopK*>(dyn);
  if (threadIdx.x == 0) tk.count = 0;
  __syncthreads();
  // MT lists at a time: each thread walks down its (sorted) list while its
  // head can still enter the running top-k
  for (int lb = 0; lb < nblk; lb += MT) {
    const int b = lb + threadIdx.x;
    const i64* bt = blk + (i64)b * 2 * k;
    bool alive = b < nblk;
    int p = 0;
    while (__syncthreads_or(alive)) {
      i64 t = 0, i = 0;
      bool cand = false;
      if (alive && p < k) {
        t = bt[p];
        i = bt[k + p];
        cand = t != KEY_INF && t != LIST_PAD && (tk.count < k || key_less(t, i, tk.lt[k - 1], tk.li[k - 1]));
      }
      alive = cand;
      topk_offer(tk, k, t, i, cand);
      if (cand) ++p;
    }
  }
  __syncthreads();
  for (int a = threadIdx.x; a < k; a += MT) {
    out_t[a] = a < tk.count ? tk.lt[a] : KEY_INF;
    out_i[a] = a < tk.count ? tk.li[a] : -1;
  }
}

// K_merge for k <= 32: every warp keeps a sorted top-k in registers (lane j
// holds the j-th entry) and walks the heads of its share of the lists; warp 0
// then merges the per-warp results.  Same output as k_merge.
__device__ void merge_small_body(const i64* __restrict__ blk, int nblk, int k, i64* __restrict__ out_t,
                                 i64* __restrict__ out_i) {
  __shared__ i64 st[MW][32], si[MW][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  RegTopK r;
  r.init();
  for (int g = w * 32; g < nblk; g += MW * 32) {
    const int b = g + lane;
    i64 ht = KEY_INF, hi = KEY_INF;
    if (b < nblk) {
      ht = blk[(i64)b * 2 * k];
      hi = blk[(i64)b * 2 * k + k];
      if (ht == LIST_PAD) ht = hi = KEY_INF;
    }
    const i64 tt = __shfl_sync(FULL, (long long)r.t, k - 1), ti = __shfl_sync(FULL, (long long)r.i, k - 1);
    unsigned cand = __ballot_sync(FULL, ht != KEY_INF && key_less(ht, hi, tt, ti));
    while (cand) {
      const int src = __ffs(cand) - 1;
      cand &= cand - 1;
      const i64* L = blk + (i64)(g + src) * 2 * k;
      const i64 lt = lane < k ? L[lane] : KEY_INF, li = lane < k ? L[k + lane] : KEY_INF;  // whole list at once
      for (int p = 0; p < k; ++p) {
        const i64 xt = __shfl_sync(FULL, (long long)lt, p), xi = __shfl_sync(FULL, (long long)li, p);
        const i64 thT = __shfl_sync(FULL, (long long)r.t, k - 1), thI = __shfl_sync(FULL, (long long)r.i, k - 1);
        if (xt == KEY_INF || xt == LIST_PAD || !key_less(xt, xi, thT, thI)) break;
        r.insert(xt, xi);
      }
    }
  }
  st[w][lane] = r.t;
  si[w][lane] = r.i;
  __syncthreads();
  if (w == 0) {
    for (int o = 1; o < MW; ++o)
      for (int p = 0; p < k; ++p) {
        const i64 xt = st[o][p], xi = si[o][p];
        const i64 thT = __shfl_sync(FULL, (long long)r.t, k - 1), thI = __shfl_sync(FULL, (long long)r.i, k - 1);
        if (xt == KEY_INF || !key_less(xt, xi, thT, thI)) break;
        r.insert(xt, xi);
      }
    if (lane < k) {
      out_t[lane] = r.t;
      out_i[lane] = r.t == KEY_INF ? -1 : r.i;
    }
  }
}

__global__ void __launch_bounds__(MW * 32) k_merge_small(const i64* __restrict__ blk, int nblk, int k,
                                                          i64* __restrict__ out_t, i64* __restrict__ out_i) {
  merge_small_body(blk, nblk, k, out_t, out_i);
}

// k <= 32 with a global bound g >= the k-th smallest time (K_final's): only
// list entries with time <= g can be in the top-k, and every list is sorted,
// so those entries are a prefix of each list.  Thread per list walks its
// prefix (usually zero or one entry: ~300 of 19 k on config 2), compacting
// into shared memory; one bitonic sort of the survivors gives the top-k.  If
// more than CAP survive (massive ties), the register merge runs instead.
constexpr int CAP = 1024;
__global__ void __launch_bounds__(1024) k_merge_thresh(const i64* __restrict__ blk, int nblk, int k,
                                                      const unsigned long long* __restrict__ gthr,
                                                      i64* __restrict__ out_t, i64* __restrict__ out_i) {
  __shared__ i64 ct[CAP], ci[CAP];
  __shared__ int cnt;
  const int tid = threadIdx.x;
  // a programmatic dependent of K_final when the sweep ran (same stream): wait
  // for its lists before reading them (a no-op for an ordinary launch)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const i64 g = (i64)*gthr;
  if (tid == 0) cnt = 0;
  __syncthreads();
  // every (list, position) pair is an independent load (no walk down a list:
  // the loads of a thread's pairs are all in flight at once)
  const int tot = nblk * k;
#pragma unroll 8
  for (int e = tid; e < tot; e += 1024) {
    const int b = e / k, p = e - b * k;
    const i64* L = blk + (i64)b * 2 * k;
    const i64 t = L[p];
    if (t != LIST_PAD && t != KEY_INF && t <= g) {
      const int pos = atomicAdd(&cnt, 1);
      if (pos < CAP) {
        ct[pos] = t;
        ci[pos] = L[k + p];
      }
    }
  }
  __syncthreads();
  const int n = cnt;
  if (n > CAP) {  // uniform branch
    merge_small_body(blk, nblk, k, out_t, out_i);
    return;
  }
  if (n <= 1024) {
    // few survivors (the usual case; keys are unique: (T, index)): each warp
    // sorts its 32 (bitonic, shuffles), the smallest warp k-th key bounds the
    // top-k, and only the survivors under it are ranked against each other
    const int lane = tid & 31, w = tid >> 5;
    __shared__ i64 wk[32];
    __shared__ int cnt2;
    i64 x = tid < n ? ct[tid] : KEY_INF, xi = tid < n ? ci[tid] : KEY_INF;
#pragma unroll
    for (int size = 2; size <= 32; size <<= 1)
#pragma unroll
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        const i64 ot = __shfl_xor_sync(FULL, (long long)x, stride), oi = __shfl_xor_sync(FULL, (long long)xi, stride);
        const bool up = (lane & size) == 0, lower = (lane & stride) == 0;
        const bool olt = key_less(ot, oi, x, xi);
        if (lower == up ? olt : !olt && !(ot == x && oi == xi)) { x = ot; xi = oi; }
      }
    if (lane == k - 1) wk[w] = x;
    if (tid == 0) cnt2 = 0;
    __syncthreads();
    i64 thr = KEY_INF;
    for (int q = 0; q < 32; ++q) thr = imin(thr, wk[q]);
    __syncthreads();  // every thread has read ct / ci (the compaction below overwrites them)
    if (x != KEY_INF && x <= thr) {
      const int pos = atomicAdd(&cnt2, 1);
      ct[pos] = x;
      ci[pos] = xi;
    }
    __syncthreads();
    const int n2 = cnt2;
    if (tid < n2) {
      const i64 y = ct[tid], yi = ci[tid];
      int rank = 0;
      for (int j = 0; j < n2; ++j) rank += key_less(ct[j], ci[j], y, yi);
      if (rank < k) { out_t[rank] = y; out_i[rank] = yi; }
    }
    for (int r = n2 + tid; r < k; r += 1024) { out_t[r] = KEY_INF; out_i[r] = -1; }
    return;
  }
  int np = 32;
  while (np < n) np <<= 1;
  for (int e = n + tid; e < np; e += 1024) { ct[e] = KEY_INF; ci[e] = KEY_INF; }
  __syncthreads();
  for (int size = 2; size <= np; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int e = tid; e < np; e += 1024) {
        const int j = e ^ stride;
        if (j > e) {
          const bool up = (e & size) == 0;
          const i64 x = ct[e], xi = ci[e], y = ct[j], yi = ci[j];
          if (key_less(y, yi, x, xi) == up) { ct[e] = y; ci[e] = yi; ct[j] = x; ci[j] = xi; }
        }
      }
      __syncthreads();
    }
  if (tid < k) {
    out_t[tid] = tid < n ? ct[tid] : KEY_INF;
    out_i[tid] = tid < n ? ci[tid] : -1;
  }
}

static void launch_merge_any(const i64* lists, int nlists, int k, i64* out_t, i64* out_i, cudaStream_t st);

template <typename K>
static int grid_of(const hsim_handle* h, K kern, int& cache) {
  if (!cache) {
    int per = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, NT, 0) != cudaSuccess || per < 1) per = 1;
    cache = per;
  }
  return sm_count(h) * cache;
}

static void merge_attr() {
  // per device (the attribute is per device); idempotent, so a race between
  // host threads only repeats the call
  static int attr_dev[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && !attr_dev[dev]) {
    cudaFuncSetAttribute(k_merge, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(TopK));
    attr_dev[dev] = 1;
  }
}

static int finish(hsim_handle* h, int launches) {
  set_launches(h, launches);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(cudaGetErrorString(e));
    return HSIM_ECUDA;
  }
  return HSIM_OK;
}

#ifndef HSIM_MULTI_MAXJOBS
#define HSIM_MULTI_MAXJOBS (1LL << 18)  // depths with fewer (candidate, class) jobs in the space go to K_pipe_multi
#endif
#ifndef HSIM_MULTI_PMIN
#define HSIM_MULTI_PMIN 1
#endif
#ifndef HSIM_MULTI_PMAX
#define HSIM_MULTI_PMAX 16
#endif
#ifndef HSIM_FINAL_MULT
#define HSIM_FINAL_MULT 4  // K_final blocks per SM for k <= 32 (one top-k list per block; one wave of the pruned kernel at 4 resident: measured 4 beats 8 with the dedupe)
#endif
static int final_grid(const hsim_handle* h, int k) { return sm_count(h) * (k && k <= 32 ? HSIM_FINAL_MULT : 2); }

// Runs the phase kernels over all chunks of the call; out / top-k lists / cell
// count optional.
static int run_phases(hsim_handle* h, const Tables* dT, Cands c, int64_t n, int64_t* out_ns, int32_t k, i64* lists,
                      int count, i64* cells_out, cudaStream_t st, int& launches) {
  // resident blocks per SM of each kernel, cached per handle
  int* gc = grid_cache(h);
  int &g_split = gc[0], &g_deep = gc[1], &g_sync = gc[2], *g_pipe = gc + 3, *g_cont = gc + 3 + FASTP + 1, &g_multi = gc[40], &g_multi2 = gc[41];
  static_assert(3 + 2 * (FASTP + 1) <= 40, "grid cache");
  // chunk plan
  i64 nchunks;
  i64* hplan = nullptr;
  cudaEvent_t plan_ev = nullptr;
  if (c.idx) {
    nchunks = (n + 31) / 32;
    c.nr = 0;
  } else if (!c.block) {
    c.nr = 1;
    nchunks = range_chunks(h, c.first, n, &c.c0);
  } else {
    c.nr = (n + c.block - 1) / c.block;
    nchunks = host_plan(h, c.first, c.block, c.stride, n, c.nr, &hplan, &plan_ev);
    if (nchunks < 0) return HSIM_ENOMEM;
  }
  // batches of chunks, double-buffered: batch b+1's K_split overlaps batch b's
  // depth kernels, batch b's K_final overlaps batch b+1's depth kernels
  i64 cbatch = (nchunks + HSIM_NBATCH - 1) / HSIM_NBATCH;
  if (cbatch < 2048) cbatch = nchunks < 2048 ? nchunks : 2048;
  if (cbatch > CBMAX) cbatch = CBMAX;
  // S.1 overlap mode: per-stage last-backward ends, stages_max rows of ns
  // int64 per buffer, kept under ~256 MiB
  const bool overlap = sync_overlap(h) && !count;
  const i64 spmax = overlap ? stages_max(h) : 0;
  if (overlap && cbatch * 32 * spmax * 8 > ((i64)1 << 28)) cbatch = imax(1, ((i64)1 << 28) / (32 * 8 * spmax));
  const i64 ns = cbatch * 32;
  const int NBUF = count ? 1 : 2;
  // scratch per buffer (int64 words): tpos, Tc [MAXC], extra | counters | int32: tau,
  // status, rm, deep, dig / q / seats / add [MAXC], job lists (x2: full / partial)
  const uint32_t pm = depth_mask(h);
  size_t jobcap[FASTP + 1], jobw = 0;
  for (int P = 1; P <= FASTP; ++P) {
    jobcap[P] = (pm >> P & 1) ? (size_t)depth_jobs_max(h, P) * ns : 0;
    jobw += 2 * jobcap[P];
  }
  // V.2: the K_ilv job list
  const bool ilv = interleave_v(h) > 1;
  const bool bkt = sync_buckets(h) == 2;  // B.1
  // top-k only (no out_ns, k <= 32): the sync is computed in K_final for the
  // candidates that can still enter the top-k (HSIM_PRUNE=0 disables)
  static int prune_env = -1;
  if (prune_env < 0) {
    const char* e = getenv("HSIM_PRUNE");
    prune_env = e && e[0] == '0' ? 0 : 1;
  }
  const bool prune = prune_env && prune_enabled(h) && !ilv && !out_ns && k >= 1 && k <= 32 && !count;
  const size_t ilvcap = ilv ? (size_t)ilv_jobs_max(h) * ns : 0;
  jobw += ilvcap;
  // pipeline dedupe: not with S.1 (per-candidate stage ends) or V.2
  const bool dd = dedup_enabled(h) && !sync_overlap(h) && !ilv;
  size_t hcap = 0;
  int hbits = 0;
  if (dd) {  // at most ns * cmax distinct pipelines per batch: load factor <= 1/2
    const size_t need = 2 * (size_t)ns * (size_t)class_max(h);
    while (((size_t)1 << hbits) < need || hbits < 10) ++hbits;
    hcap = (size_t)1 << hbits;
    if (hbits > 30) return HSIM_ENOMEM;
  }
  const size_t planw = hplan ? (size_t)(2 * c.nr + 1) : 0;
  const size_t n32 = (size_t)(4 + 4 * MAXC + (dd ? MAXC : 0)) * ns + jobw;
  const size_t bufw0 = (size_t)(MAXC + 2) * ns + NCNT + (n32 + 1) / 2 + 8;
  size_t reqw = 0, reqcap[HSIM_REQ_MAXP + 1] = {0};
  for (int P = HSIM_REQ_MINP; P <= HSIM_REQ_MAXP && P <= FASTP; ++P) {
    if (depth_jobs_space(h, P) < HSIM_REQ_MINJOBS) continue;
    reqcap[P] = jobcap[P];  // a depth's jobs (re-queued at most once each)
    reqw += reqcap[P];
  }
  const size_t bufw = bufw0 + (size_t)spmax * ns + reqw;
  i64* base = nullptr;
  if (ensure_work_scratch(h, NBUF * bufw + planw + 8, &base)) return HSIM_ENOMEM;
  Scratch SB[2];
  for (int q = 0; q < NBUF; ++q) {
    Scratch& S = SB[q];
    i64* b0 = base + q * bufw;
    S.ns = ns;
    S.tpos = b0;
    S.Tc = b0 + ns;
    S.extra = b0 + (MAXC + 1) * ns;
    S.Rs = overlap ? b0 + bufw0 : nullptr;
    {
      i64* rp = b0 + bufw0 + (size_t)spmax * ns;
      for (int P = 0; P <= HSIM_REQ_MAXP; ++P) {
        S.req[P] = reqcap[P] ? rp : nullptr;
        S.req_cap[P] = (i64)reqcap[P];
        rp += reqcap[P];
      }
    }
    S.counters = (unsigned long long*)(b0 + (MAXC + 2) * ns);
    int32_t* p32 = (int32_t*)(b0 + (MAXC + 2) * ns + NCNT);
    S.tau = p32;
    S.status = p32 + ns;
    S.rm = p32 + 2 * ns;
    S.deep = p32 + 3 * ns;
    S.dig = (u32*)(p32 + 4 * ns);
    S.q = p32 + (4 + MAXC) * ns;
    S.seats = p32 + (4 + 2 * MAXC) * ns;
    S.add = p32 + (4 + 3 * MAXC) * ns;
    int32_t* pj = p32 + (4 + 4 * MAXC) * ns;
    S.full[0] = S.part[0] = nullptr;
    for (int P = 1; P <= FASTP; ++P) {
      S.full[P] = pj;
      S.part[P] = pj + jobcap[P];
      pj += 2 * jobcap[P];
    }
    S.ilv = ilvcap ? pj : nullptr;
    pj += ilvcap;
    S.hkeys = nullptr;
    S.hres = nullptr;
    S.hj = nullptr;
    S.hbits = hbits;
    if (dd) {
      if (ensure_hash_scratch(h, q, hcap, &S.hkeys, &S.hres)) return HSIM_ENOMEM;
      S.hj = pj;
    }
  }
  if (hplan) {
    i64* pw = base + NBUF * bufw;
    cudaMemcpyAsync(pw, hplan, planw * 8, cudaMemcpyHostToDevice, st);
    cudaEventRecord(plan_ev, st);
    c.plan = pw;
  }
  const int gs = grid_of(h, k_split<false>, g_split), gd = grid_of(h, k_deep, g_deep), gy = grid_of(h, k_sync<false>, g_sync),
            gf = final_grid(h, k);
  // launch order: longest total work first; the latency-bound deep depths run
  // on high-priority streams (host.cu), which matters more than the order
  // (measured: priority 0.50 -> 0.44 ms per config-2 sweep; deep-first order
  // with priority 0.448 ms vs this order 0.435 ms)
#ifdef HSIM_DEEPFIRST
  static const int order[16] = {16, 15, 14, 13, 12, 11, 10, 9, 8, 4, 2, 6, 5, 3, 7, 1};
#else
  static const int order[16] = {4, 8, 16, 2, 6, 5, 3, 12, 10, 7, 9, 11, 13, 14, 15, 1};
#endif
  cudaStream_t fin = side_stream(h, NSTREAM_FINAL);
  // depths with few class-jobs in the space and no re-queue share one launch
  // (K_pipe_multi); a depth alone keeps its own kernel
  uint32_t mmask = 0;
  for (int P = 1; P <= FASTP; ++P)
    if ((pm >> P & 1) && depth_jobs_space(h, P) < HSIM_MULTI_MAXJOBS && (P > HSIM_REQ_MAXP || !reqcap[P]) &&
        P >= HSIM_MULTI_PMIN && P <= HSIM_MULTI_PMAX)
      mmask |= 1u << P;
  if (__builtin_popcount(mmask & 0x1FEu) < 2) mmask &= ~0x1FEu;  // a group of one depth: its own kernel
  if (__builtin_popcount(mmask & 0x1FE00u) < 2) mmask &= ~0x1FE00u;
  i64 cells = 0;
  int b = 0;
  for (i64 ca = 0; ca < nchunks; ca += cbatch, ++b) {
    const int q = b % NBUF;
    Scratch& S = SB[q];
    const i64 cb = ca + cbatch < nchunks ? ca + cbatch : nchunks;
    const i64 nsb = (cb - ca) * 32;
    if (b >= NBUF && !count) cudaStreamWaitEvent(st, pool_event(h, 2 + q), 0);  // buffer free: final(b-2) done
    cudaMemsetAsync(S.counters, 0, NCNT * sizeof(unsigned long long), st);
    int tq = g_trace.pre("k_split", 0, st);
    if (ilv) k_split<true><<<gs, NT, 0, st>>>(dT, c, ca, cb, S, pm);
    else k_split<false><<<gs, NT, 0, st>>>(dT, c, ca, cb, S, pm);
    g_trace.post(tq, st);
    ++launches;
    cudaEventRecord(pool_event(h, q), st);
    // the depth kernels, K_deep and K_sync of a batch are independent: each on
    // its own stream after K_split, all joined by K_final
    int j = 0;
    auto side = [&](int sid) {
      cudaStream_t ss = side_stream(h, sid);
      cudaStreamWaitEvent(ss, pool_event(h, q), 0);
      return ss;
    };
    auto join = [&](cudaStream_t ss) {
      cudaEvent_t e = pool_event(h, 4 + q * 20 + j);
      cudaEventRecord(e, ss);
      cudaStreamWaitEvent(count ? st : fin, e, 0);
      ++j;
    };
    auto launch_deep = [&]() {
      if (pm >> (FASTP + 1)) {
        cudaStream_t ss = side(17);
        tq = g_trace.pre("k_deep", 17, ss);
        k_deep<<<gd, NT, 0, ss>>>(dT, S, count);
        g_trace.post(tq, ss);
        ++launches;
        join(ss);
      }
    };
#ifdef HSIM_DEEPFIRST
    launch_deep();  // the deepest pipelines first (latency-bound, high-priority stream)
#endif
    // the sparse depths in two launches (1..8, 9..16), first, on high-priority streams
    if (mmask & 0x1FEu) {
      cudaStream_t ss = side(20);
      tq = g_trace.pre("k_pipe_multi<1,8>", 20, ss);
      k_pipe_multi<1, 8><<<grid_of(h, k_pipe_multi<1, 8>, g_multi), NT, 0, ss>>>(dT, S, count, mmask);
      g_trace.post(tq, ss);
      ++launches;
      join(ss);
    }
    if (mmask & 0x1FE00u) {
      cudaStream_t ss = side(21);
      tq = g_trace.pre("k_pipe_multi<9,16>", 21, ss);
      k_pipe_multi<9, 16><<<grid_of(h, k_pipe_multi<9, 16>, g_multi2), NT, 0, ss>>>(dT, S, count, mmask);
      g_trace.post(tq, ss);
      ++launches;
      join(ss);
    }
    for (int oi = 0; oi < 16; ++oi) {
      const int P = order[oi];
      if (P > FASTP || !(pm >> P & 1) || (mmask >> P & 1)) continue;
      cudaStream_t ss = side(P);
      static const char* pn[17] = {"", "k_pipe<1>", "k_pipe<2>", "k_pipe<3>", "k_pipe<4>", "k_pipe<5>", "k_pipe<6>", "k_pipe<7>", "k_pipe<8>", "k_pipe<9>", "k_pipe<10>", "k_pipe<11>", "k_pipe<12>", "k_pipe<13>", "k_pipe<14>", "k_pipe<15>", "k_pipe<16>"};
      tq = g_trace.pre(pn[P], P, ss);
      switch (P) {
#define HSIM_PIPE(PP) case PP: k_pipe<PP><<<grid_of(h, k_pipe<PP>, g_pipe[PP]), NT, 0, ss>>>(dT, S, count); break;
        HSIM_PIPE(1) HSIM_PIPE(2) HSIM_PIPE(3) HSIM_PIPE(4) HSIM_PIPE(5) HSIM_PIPE(6) HSIM_PIPE(7) HSIM_PIPE(8)
#if HSIM_FASTP >= 16
        HSIM_PIPE(9) HSIM_PIPE(10) HSIM_PIPE(11) HSIM_PIPE(12) HSIM_PIPE(13) HSIM_PIPE(14) HSIM_PIPE(15) HSIM_PIPE(16)
#endif
#undef HSIM_PIPE
        default: break;
      }
      if (P >= HSIM_REQ_MINP && P <= HSIM_REQ_MAXP && reqcap[P]) {  // the re-queued jobs of this depth, densely
        switch (P) {
#define HSIM_CONT(PP) case PP: k_pipe_cont<PP><<<grid_of(h, k_pipe_cont<PP>, g_cont[PP]), NT, 0, ss>>>(dT, S, count); break;
          HSIM_CONT(2) HSIM_CONT(3) HSIM_CONT(4) HSIM_CONT(5) HSIM_CONT(6) HSIM_CONT(7) HSIM_CONT(8)
#undef HSIM_CONT
          default: break;
        }
        ++launches;
      }
      g_trace.post(tq, ss);
      ++launches;
      join(ss);
    }
#ifndef HSIM_DEEPFIRST
    launch_deep();
#endif
    if (ilv && ilvcap) {  // V.2: every interleaved pipeline (warp per job, rings in shared memory)
      const int PM = ilv_depth_max(h), v = interleave_v(h);
      int Q = 4;
      while (Q < PM / 2 + 2) Q *= 2;
      // steady-regime jumps for pipelines of up to PJ stages (history 2 PJ^2 v doubles per warp)
      int PJ = PM < 16 ? PM : 16;
      while (PJ > 1 && (size_t)2 * PJ * PJ * v * 8 > 32 * 1024) --PJ;
      const size_t per_warp = (size_t)ILV_WORDS(PM, Q, PJ, v) * 8;
      int W = 4;
      while (W > 1 && W * per_warp > (size_t)200 * 1024) --W;
      const size_t smem = W * per_warp;
      static int attr_set[64] = {0};
      int dev = 0;
      cudaGetDevice(&dev);
      if (smem > 48 * 1024 && dev < 64 && attr_set[dev] < (int)smem) {
        cudaFuncSetAttribute(k_ilv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr_set[dev] = (int)smem;
      }
      int per = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_ilv, 32 * W, smem) != cudaSuccess || per < 1) per = 1;
      cudaStream_t ss = side(17);
      tq = g_trace.pre("k_ilv", 17, ss);
      k_ilv<<<sm_count(h) * per, 32 * W, smem, ss>>>(dT, S, count, PM, Q, PJ);
      g_trace.post(tq, ss);
      ++launches;
      join(ss);
    }
    if (count) {
      unsigned long long v = 0;
      if (dd) cudaMemsetAsync(S.hkeys, 0, hcap * 8, st);  // no K_final in count mode: clear the table here
      cudaMemcpyAsync(&v, S.counters + CNT_CELLS, 8, cudaMemcpyDeviceToHost, st);
      if (cudaStreamSynchronize(st) != cudaSuccess) break;
      cells += (i64)v;
      continue;
    }
    if (prune) {
      // the sync runs inside K_final, pruned by the top-k bound
    } else if (ilv) {  // V.2: revisited stage groups (C.8 concurrently with K_ilv; S.1 after it)
      cudaStream_t ss = overlap ? fin : side(18);
      tq = g_trace.pre("k_sync_ilv", 18, ss);
      k_sync_ilv<<<gy, NT, 0, ss>>>(dT, S, nsb, overlap ? 1 : 0);
      g_trace.post(tq, ss);
      ++launches;
      if (!overlap) join(ss);
    } else if (overlap) {  // S.1: needs the stages' last-backward ends -> after the 1F1B kernels
      tq = g_trace.pre("k_sync_overlap", NSTREAM_FINAL, fin);
      if (bkt) k_sync_overlap<true><<<gy, NT, 0, fin>>>(dT, S, nsb);
      else k_sync_overlap<false><<<gy, NT, 0, fin>>>(dT, S, nsb);
      g_trace.post(tq, fin);
      ++launches;
    } else {
      cudaStream_t ss = side(18);
      tq = g_trace.pre("k_sync", 18, ss);
      if (bkt) k_sync<true><<<gy, NT, 0, ss>>>(dT, S, nsb);
      else k_sync<false><<<gy, NT, 0, ss>>>(dT, S, nsb);
      g_trace.post(tq, ss);
      ++launches;
      join(ss);
    }
    if (dd) {  // dedupe: every slot's T0 from the table (K_final then reads it coalesced)
      tq = g_trace.pre("k_gather", NSTREAM_FINAL, fin);
      k_gather<<<sm_count(h) * 16, NT, 0, fin>>>(S, nsb);
      g_trace.post(tq, fin);
      ++launches;
    }
    tq = g_trace.pre("k_final", NSTREAM_FINAL, fin);
    if (prune) {
      if (overlap) {
        if (bkt) k_final_small<2, true><<<gf, NT, 0, fin>>>(dT, c, S, nsb, out_ns, k, lists);
        else k_final_small<2, false><<<gf, NT, 0, fin>>>(dT, c, S, nsb, out_ns, k, lists);
      } else {
        // dedupe: a programmatic dependent launch behind K_gather (same stream)
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3(gf);
        lc.blockDim = dim3(NT);
        lc.stream = fin;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = dd ? 1 : 0;
        lc.attrs = at;
        lc.numAttrs = 1;
        if (bkt && b == 0) cudaLaunchKernelEx(&lc, k_final_small<1, true, true>, dT, c, S, nsb, out_ns, k, lists);
        else if (bkt) cudaLaunchKernelEx(&lc, k_final_small<1, true, false>, dT, c, S, nsb, out_ns, k, lists);
        else if (b == 0) cudaLaunchKernelEx(&lc, k_final_small<1, false, true>, dT, c, S, nsb, out_ns, k, lists);
        else cudaLaunchKernelEx(&lc, k_final_small<1, false, false>, dT, c, S, nsb, out_ns, k, lists);
      }
    } else if (k && k <= 32) k_final_small<0, false><<<gf, NT, 0, fin>>>(dT, c, S, nsb, out_ns, k, lists);
    else k_final<<<gf, NT, 0, fin>>>(dT, c, S, nsb, out_ns, k, lists);
    g_trace.post(tq, fin);
    ++launches;
    cudaEventRecord(pool_event(h, 2 + q), fin);
  }
  if (!count && b > 0) cudaStreamWaitEvent(st, pool_event(h, 2 + (b - 1) % NBUF), 0);  // join the final stream
  if (cells_out) *cells_out = cells;
#ifdef HSIM_DIAG
  if (count) {
    unsigned long long hd[17][16];
    cudaMemcpyFromSymbol(hd, g_diag, sizeof hd);
    for (int P = 1; P <= 16; ++P) {
      unsigned long long t = 0;
      for (int b = 0; b < 8; ++b) t += hd[P][b];
      if (!t) continue;
      fprintf(stderr, "P=%2d jobs %llu exec/kn pairs %.3f | hist", P, t, (double)hd[P][8] / (double)(hd[P][9] ? hd[P][9] : 1));
      for (int b = 0; b < 8; ++b) fprintf(stderr, " %.3f", (double)hd[P][b] / t);
      fprintf(stderr, "\n");
    }
    unsigned long long z[17][16] = {};
    cudaMemcpyToSymbol(g_diag, z, sizeof z);
  }
#endif
  return HSIM_OK;
}

static void launch_merge_any(const i64* lists, int nlists, int k, i64* out_t, i64* out_i, cudaStream_t st) {
  if (k <= 32) {
    k_merge_small<<<1, MW * 32, 0, st>>>(lists, nlists, k, out_t, out_i);
  } else {
    merge_attr();
    k_merge<<<1, MT, sizeof(TopK), st>>>(lists, nlists, k, out_t, out_i);
  }
}

int launch_merge(const int64_t* lists, int32_t nlists, int32_t k, int64_t* out_t, int64_t* out_i, cudaStream_t st) {
  launch_merge_any(lists, nlists, k, out_t, out_i, st);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(cudaGetErrorString(e));
    return HSIM_ECUDA;
  }
  return HSIM_OK;
}

int launch_eval(hsim_handle* h, const Tables* dT, const hsim_cands* cc, int64_t n, int64_t* out_ns, int32_t k,
                int64_t* out_t, int64_t* out_i, cudaStream_t st) {
  Cands c{cc->idx, cc->first, cc->block, cc->stride, n, nullptr, 0, 0};
  int launches = 0;
  i64* lists = nullptr;
  call_begin(h, st);
  const int nlists = final_grid(h, k) * (k <= 32 ? 1 : NT / 32);  // per block (k <= 32) or per warp
  if (k) {
    // lists + the global bound word + the synced-segment counter
    if (ensure_block_scratch(h, (size_t)nlists * 2 * k + 2, &lists)) return HSIM_ENOMEM;
    cudaMemsetAsync(lists, 0x7F, ((size_t)nlists * 2 * k + 1) * 8, st);
    cudaMemsetAsync(lists + (size_t)nlists * 2 * k + 1, 0, 8, st);
    set_sync_counter(h, k <= 32 && !out_ns && prune_enabled(h) && interleave_v(h) <= 1
                            ? lists + (size_t)nlists * 2 * k + 1 : nullptr);
  }
  g_trace.begin(st);
  if (n > 0) {
    const int rc = run_phases(h, dT, c, n, out_ns, k, lists, 0, nullptr, st, launches);
    if (rc) return rc;
  }
  if (k) {
    // n == 0 merges no list and only writes the (INT64_MAX, -1) padding
    // after the sweep: on the final stream right behind K_final (no cross-stream
    // event on the chain), then the caller's stream waits for it
    cudaStream_t ms = n > 0 ? side_stream(h, NSTREAM_FINAL) : st;
    const int tq = g_trace.pre("k_merge", n > 0 ? NSTREAM_FINAL : 0, ms);
    if (n > 0 && k <= 32) {
      cudaLaunchConfig_t lc = {};
      lc.gridDim = dim3(1);
      lc.blockDim = dim3(1024);
      lc.stream = ms;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      lc.attrs = at;
      lc.numAttrs = 1;
      cudaLaunchKernelEx(&lc, k_merge_thresh, (const i64*)lists, (int)nlists, (int)k,
                         (const unsigned long long*)(lists + (size_t)nlists * 2 * k), (i64*)out_t, (i64*)out_i);
    }
    else
      launch_merge_any(lists, n > 0 ? nlists : 0, k, out_t, out_i, ms);
    g_trace.post(tq, ms);
    ++launches;
    if (n > 0) {
      cudaEventRecord(pool_event(h, 46), ms);
      cudaStreamWaitEvent(st, pool_event(h, 46), 0);
    }
  }
  call_end(h, st);
  g_trace.dump();
  return finish(h, launches);
}

int launch_count(hsim_handle* h, const Tables* dT, int64_t first, int64_t n, int64_t* d_acc, cudaStream_t st) {
  Cands c{nullptr, first, 0, 0, n, nullptr, 0, 0};
  int launches = 0;
  i64 total = 0;
  call_begin(h, st);
  if (n > 0) {
    const int rc = run_phases(h, dT, c, n, nullptr, 0, nullptr, 1, &total, st, launches);
    if (rc) return rc;
  }
  call_end(h, st);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(cudaGetErrorString(e));
    return HSIM_ECUDA;
  }
  cudaMemcpy(d_acc, &total, 8, cudaMemcpyHostToDevice);
  return 0;
}

}  // namespace hsim
