// flow.cu — SURVEY.md §8(f) f3: flow-level contention re-simulation of the
// gradient synchronisation of k candidates (typically the top-k of a sweep).
// DESIGN.md F.1 states the model; in short ("bandwidth
// contention", :400 FCT per flow, :409-412 "the flow with the highest FCT
// value determines the bottleneck"; SPEC.md:340-373 route / simulate_flows):
//
//   * every collective step of the C.8 sync (a reshard step when some class
//     has tp != t*, then 2(D-1) ring steps per segment) is a set of flows on
//     the rail-only link graph: per GPU an NVLink egress / ingress port, the
//     PCIe path to its rail NIC and back, the NIC's wire to the rail switch and
//     back; Fig 2 case (c) crosses the source node's NVLink to the
//     destination's rank first;
//   * flows share links max-min fairly (progressive filling), each capped by
//     its own path's beta, and complete at drain end + the path's alpha;
//   * a step's flows all start when the previous step's last flow completes;
//     a segment starts when the segment before it on a shared stage group
//     has completed (C.8's FIFO).
//
// One CTA per candidate.  k_flow_count decodes the candidate (the same
// partition code as the sweep), builds its segments and counts its flows;
// the host then sizes the per-candidate scratch and k_flow_sim runs the
// fluid event loop with the whole block (flows in parallel, block-wide min
// reductions); k_flow_stats takes nearest-rank FCT percentiles by an MSB
// radix select.  Arithmetic follows DESIGN F.1's fixed IEEE sequence
// (share = residual / count, residual -= k x s, rem -= rate x delta,
// d = ceil(rem / rate)), so the results equal the oracle's bit for bit.
#include <cuda_runtime.h>

#include "hsim.h"
#include "hsim_core.cuh"

namespace hsim {

int sm_count(const hsim_handle* h);
void set_error(const char* m);
void call_begin(hsim_handle* h, cudaStream_t st);
void call_end(hsim_handle* h, cudaStream_t st);
int ensure_flow_scratch(hsim_handle* h, size_t bytes, void** out);

constexpr int FT = 256;     // threads per candidate
constexpr int FMAXJ = 256;  // segments per candidate (<= layers)
constexpr int FMAXS = MAXC * MAXP;
constexpr i64 FINF = INT64_MAX;
constexpr int NOUT = 8;     // status, sync_ab, sync_flow, n_flows, p50, p99, p99.9, max

struct FlowRec {
  double rem, rate, cap;
  i64 arrive, alpha, d;
  int seg, nl, frz, now;
  int link[6];
};

// per-candidate program in shared memory
struct FlowProg {
  int status, C, J, nst;
  i64 D;
  int P[MAXC], Dc[MAXC], off[MAXC];
  int16_t typ[FMAXS], tp[FMAXS], pos[FMAXS], ct[FMAXS];
  int16_t a[FMAXJ], z[FMAXJ];
  int16_t tstar[FMAXJ];
  uint8_t sc[FMAXJ][MAXC];
  uint8_t rs[FMAXJ], pred[FMAXJ];
  i64 S[FMAXJ];
};

struct SegState {
  int cur, steps, pending, live;
  i64 done_max, completion;
};

__device__ __forceinline__ i64 lmin(i64 a, i64 b) { return a < b ? a : b; }

// group (node, base) of stage s of replica r of class c: every type belongs to
// one class and all of its groups have one tp, so C.3's lowest-free-block rule
// fills the type's nodes in order -- the j-th type-t group sits at block j.
__device__ __forceinline__ void group_of(const Tables& T, const FlowProg& F, int c, int r, int s, int& node, int& base) {
  const int k = F.off[c] + s;
  const int t = F.typ[k], tp = F.tp[k];
  const int per = T.gpn / tp;
  const int j = r * F.ct[k] + F.pos[k];
  node = T.type_nodes[T.type_node_off[t] + j / per];
  base = (j % per) * tp;
}

__device__ __forceinline__ int link_class(const Tables& T, int n1, int r1, int n2, int r2) {
  const int t1 = T.node_type[n1], t2 = T.node_type[n2];
  return n1 == n2 ? T.lc_same[t1][r1][r2] : T.lc_cross[t1][r1][t2][r2];
}

__device__ __forceinline__ int lid(const Tables& T, int kind, int n, int r) { return (n * T.gpn + r) * 6 + kind; }

__device__ __forceinline__ double link_cap(const Tables& T, int id) {
  const int kind = id % 6, g = id / 6, n = g / T.gpn, r = g % T.gpn;
  const int t = T.node_type[n];
  if (kind <= 1) return T.port_cap[t][r][kind];
  if (kind <= 3) return T.pcie_cap[t];
  return T.nic_cap[t];
}

// the flow (n1, r1) -> (n2, r2) of `bytes` (DESIGN F.1 paths)
__device__ void make_flow(const Tables& T, FlowRec& f, int n1, int r1, int n2, int r2, i64 bytes, int seg, i64 now) {
  const int lc = link_class(T, n1, r1, n2, r2);
  f.alpha = T.lc[lc].alpha;
  f.cap = T.lc[lc].beta;
  f.rem = (double)bytes;
  f.arrive = now;
  f.seg = seg;
  f.frz = 0;
  int nl = 0;
  if (n1 == n2 || r1 != r2) {
    f.link[nl++] = lid(T, 0, n1, r1);
    f.link[nl++] = lid(T, 1, n1, r2);
  }
  if (n1 != n2) {
    f.link[nl++] = lid(T, 2, n1, r2);
    f.link[nl++] = lid(T, 4, n1, r2);
    f.link[nl++] = lid(T, 5, n2, r2);
    f.link[nl++] = lid(T, 3, n2, r2);
  }
  f.nl = nl;
}

// ---- block reductions ------------------------------------------------------------
template <typename V, typename Op>
__device__ V block_reduce(V v, Op op, V* sh) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  V r = sh[0];
  for (int q = 1; q < FT / 32; ++q) r = op(r, sh[q]);
  __syncthreads();
  return r;
}
struct MinI { __device__ i64 operator()(i64 a, i64 b) const { return a < b ? a : b; } };
struct MaxI { __device__ i64 operator()(i64 a, i64 b) const { return a > b ? a : b; } };
struct MinD { __device__ double operator()(double a, double b) const { return a < b ? a : b; } };
struct SumI { __device__ int operator()(int a, int b) const { return a + b; } };

// ---- setup: decode, partition, layers, segments (thread 0) ----------------------
__device__ void flow_setup(const Tables& T, i64 i, FlowProg& F) {
  F.status = 0;
  F.J = 0;
  F.D = 1;
  if (i < 0 || i >= T.N) { F.status = INT32_MIN; return; }
  const TplRec& tr = T.tpl[find_template(T, i)];
  ClassSplit cs[MAXC];
  const int st = partition_any(T, tr, i - tr.prefix, cs);
  if (st) { F.status = st; return; }
  F.C = tr.C;
  F.D = tr.D;
  int16_t lay[FMAXS];
  int k = 0;
  for (int c = 0; c < F.C; ++c) {
    const CrecHdr* h = crec_hdr(T, tr.crec[c]);
    const StageRec* sr = crec_stages(T, tr.crec[c]);
    F.P[c] = h->P;
    F.Dc[c] = h->D;
    F.off[c] = k;
    LayerWalk lw = walk(T, h, cs[c].dig);
    for (int s = 0; s < h->P; ++s, ++k) {
      lay[k] = (int16_t)lw.next(sr);
      F.typ[k] = (int16_t)sr[s].type;
      F.tp[k] = (int16_t)sr[s].tp;
      int pos = 0, ct = 0;
      for (int q = 0; q < h->P; ++q)
        if (sr[q].type == sr[s].type) {
          if (q < s) ++pos;
          ++ct;
        }
      F.pos[k] = (int16_t)pos;
      F.ct[k] = (int16_t)ct;
    }
  }
  F.nst = k;
  if (F.D == 1) return;
  // segments: common refinement of the classes' layer boundaries (C.6)
  int sc[MAXC], nxt[MAXC];
  for (int c = 0; c < F.C; ++c) {
    sc[c] = 0;
    nxt[c] = F.P[c] > 1 ? lay[F.off[c]] : (int)T.L;
  }
  int a = 0, J = 0;
  while (a < T.L) {
    int z = (int)T.L;
    for (int c = 0; c < F.C; ++c) z = min(z, nxt[c]);
    F.a[J] = (int16_t)a;
    F.z[J] = (int16_t)z;
    F.S[J] = (i64)(z - a) * T.seg_layer_bytes + (a == 0 ? T.seg_first_bytes : 0) + (z == T.L ? T.seg_last_bytes : 0);
    int ts = 1 << 30;
    for (int c = 0; c < F.C; ++c) {
      F.sc[J][c] = (uint8_t)sc[c];
      ts = min(ts, (int)F.tp[F.off[c] + sc[c]]);
    }
    F.tstar[J] = (int16_t)ts;
    int rs = 0, keep = 0;
    for (int c = 0; c < F.C; ++c) {
      rs |= F.tp[F.off[c] + sc[c]] != ts;
      if (J > 0) keep |= F.sc[J - 1][c] == sc[c];
    }
    F.rs[J] = (uint8_t)rs;
    F.pred[J] = (uint8_t)keep;  // FIFO: waits for segment J-1 iff they share a stage group
    ++J;
    for (int c = 0; c < F.C; ++c)
      if (nxt[c] == z && z < T.L) {
        ++sc[c];
        nxt[c] = sc[c] + 1 < F.P[c] ? nxt[c] + lay[F.off[c] + sc[c]] : (int)T.L;
      }
    a = z;
  }
  F.J = J;
}

__device__ __forceinline__ i64 rs_flows(const FlowProg& F, int j) {
  i64 n = 0;
  for (int c = 0; c < F.C; ++c) {
    const int tp = F.tp[F.off[c] + F.sc[j][c]];
    if (tp != F.tstar[j]) n += (i64)F.Dc[c] * tp;
  }
  return n;
}
__device__ __forceinline__ i64 ring_flows(const FlowProg& F, int j) { return (i64)F.tstar[j] * F.D; }
__device__ __forceinline__ int seg_steps(const FlowProg& F, int j) { return (F.rs[j] ? 1 : 0) + 2 * (int)(F.D - 1); }

// endpoints and bytes of flow x of step `st` of segment j
__device__ void step_flow(const Tables& T, const FlowProg& F, int j, int st, i64 x, int& n1, int& r1, int& n2, int& r2,
                          i64& bytes) {
  const i64 xs = (F.S[j] + F.tstar[j] - 1) / F.tstar[j];
  if (F.rs[j] && st == 0) {  // reshard: every TP-ring edge of every group with tp != t*
    for (int c = 0; c < F.C; ++c) {
      const int tp = F.tp[F.off[c] + F.sc[j][c]];
      if (tp == F.tstar[j]) continue;
      const i64 cnt = (i64)F.Dc[c] * tp;
      if (x < cnt) {
        const int r = (int)(x / tp), q = (int)(x % tp);
        int node, base;
        group_of(T, F, c, r, F.sc[j][c], node, base);
        n1 = n2 = node;
        r1 = base + q;
        r2 = base + (q + 1) % tp;
        bytes = xs;
        return;
      }
      x -= cnt;
    }
  }
  // ring q < t*: position k (class asc, replica asc) -> k + 1 (wrap)
  const int q = (int)(x / F.D);
  const i64 k = x % F.D, k2 = (k + 1) % F.D;
  auto pos = [&](i64 kk, int& node, int& base) {
    int c = 0;
    while (kk >= F.Dc[c]) kk -= F.Dc[c++];
    group_of(T, F, c, (int)kk, F.sc[j][c], node, base);
  };
  int b1, b2;
  pos(k, n1, b1);
  pos(k2, n2, b2);
  r1 = b1 + q;
  r2 = b2 + q;
  bytes = (xs + F.D - 1) / F.D;
}

__device__ __forceinline__ i64 tau_of(const Tables& T, int n1, int r1, int n2, int r2, i64 x) {
  return tau_lc(T, link_class(T, n1, r1, n2, r2), x);
}

// ---- K_flow_count -------------------------------------------------------------------
__global__ void __launch_bounds__(FT) k_flow_count(const Tables* __restrict__ gT, const i64* __restrict__ idx, int k,
                                                   i64* __restrict__ nflows) {
  __shared__ FlowProg F;
  const Tables& T = *gT;
  const int b = blockIdx.x;
  if (threadIdx.x == 0) {
    flow_setup(T, idx[b], F);
    i64 n = 0;
    if (!F.status)
      for (int j = 0; j < F.J; ++j) n += (F.rs[j] ? rs_flows(F, j) : 0) + 2 * (F.D - 1) * ring_flows(F, j);
    nflows[b] = F.status ? 0 : n;
  }
}

// ---- K_flow_sim -----------------------------------------------------------------------
struct FlowScratch {
  FlowRec* fl;   // [nmax] flow records
  int* act;      // [nmax] active flow slots
  int* freel;    // [nmax] free slots
  double* res;   // [nlink] per link
  int* cnt;
  int* took;
  i64* fct;      // [n_flows] of this candidate
};

__device__ void maxmin(const Tables& T, FlowScratch& W, int nact, double* shd, int* shi) {
  for (int q = threadIdx.x; q < nact; q += FT) {
    FlowRec& f = W.fl[W.act[q]];
    f.frz = 0;
    for (int e = 0; e < f.nl; ++e) {
      W.res[f.link[e]] = link_cap(T, f.link[e]);
      W.cnt[f.link[e]] = 0;
      W.took[f.link[e]] = 0;
    }
  }
  __syncthreads();
  for (int q = threadIdx.x; q < nact; q += FT) {
    const FlowRec& f = W.fl[W.act[q]];
    for (int e = 0; e < f.nl; ++e) atomicAdd(&W.cnt[f.link[e]], 1);
  }
  __syncthreads();
  for (;;) {
    double s = 1e300;
    for (int q = threadIdx.x; q < nact; q += FT) {
      const FlowRec& f = W.fl[W.act[q]];
      if (f.frz) continue;
      double v = f.cap;
      for (int e = 0; e < f.nl; ++e) v = fmin(v, __ddiv_rn(W.res[f.link[e]], (double)W.cnt[f.link[e]]));
      s = fmin(s, v);
    }
    s = block_reduce(s, MinD(), shd);
    int left = 0;
    for (int q = threadIdx.x; q < nact; q += FT) {
      FlowRec& f = W.fl[W.act[q]];
      f.now = 0;
      if (f.frz) continue;
      bool hit = f.cap == s;
      for (int e = 0; e < f.nl; ++e) hit = hit || __ddiv_rn(W.res[f.link[e]], (double)W.cnt[f.link[e]]) == s;
      if (hit) {
        f.now = 1;
        f.rate = s;
        for (int e = 0; e < f.nl; ++e) atomicAdd(&W.took[f.link[e]], 1);
      } else {
        ++left;
      }
    }
    __syncthreads();
    for (int q = threadIdx.x; q < nact; q += FT) {
      FlowRec& f = W.fl[W.act[q]];
      if (!f.now) continue;
      f.frz = 1;
      for (int e = 0; e < f.nl; ++e) {
        const int kk = atomicExch(&W.took[f.link[e]], 0);
        if (kk) {  // the first flow to reach a link applies the round's whole update
          W.res[f.link[e]] = __dsub_rn(W.res[f.link[e]], __dmul_rn((double)kk, s));
          W.cnt[f.link[e]] -= kk;
        }
      }
    }
    left = block_reduce(left, SumI(), shi);
    if (!left) break;
  }
}

__global__ void __launch_bounds__(FT) k_flow_sim(const Tables* __restrict__ gT, const i64* __restrict__ idx, int k,
                                                 unsigned char* __restrict__ scratch, size_t per_cand_bytes, int nmax,
                                                 int nlink, const i64* __restrict__ fct_off, i64* __restrict__ out,
                                                 i64* __restrict__ fct_all) {
  __shared__ FlowProg F;
  __shared__ SegState G[FMAXJ];
  __shared__ i64 ab_rs[FMAXJ], ab_ring[FMAXJ];
  __shared__ double shd[FT / 32];
  __shared__ i64 shl[FT / 32];
  __shared__ int shi[FT / 32];
  __shared__ int nact, nfree, nfct, nstart;
  __shared__ int start_seg[FMAXJ], start_step[FMAXJ];
  __shared__ i64 t_now, sync_flow_sh;
  const Tables& T = *gT;
  const int b = blockIdx.x;
  if (threadIdx.x == 0) flow_setup(T, idx[b], F);
  __syncthreads();
  i64* o = out + (i64)b * NOUT;
  if (F.status || F.D == 1) {
    if (threadIdx.x < NOUT) o[threadIdx.x] = threadIdx.x == 0 ? F.status : 0;
    return;
  }
  unsigned char* base = scratch + (size_t)b * per_cand_bytes;
  FlowScratch W;
  W.fl = (FlowRec*)base;
  W.act = (int*)(W.fl + nmax);
  W.freel = W.act + nmax;
  W.res = (double*)(((uintptr_t)(W.freel + nmax) + 15) & ~(uintptr_t)15);
  W.cnt = (int*)(W.res + nlink);
  W.took = W.cnt + nlink;
  W.fct = fct_all + fct_off[b];
  const int J = F.J;

  // alpha-beta schedule of the same steps: a step lasts its slowest flow's tau
  for (int j = 0; j < J; ++j) {
    i64 m = 0;
    if (F.rs[j]) {
      const i64 n = rs_flows(F, j);
      for (i64 x = threadIdx.x; x < n; x += FT) {
        int n1, r1, n2, r2;
        i64 by;
        step_flow(T, F, j, 0, x, n1, r1, n2, r2, by);
        m = max(m, tau_of(T, n1, r1, n2, r2, by));
      }
    }
    m = block_reduce(m, MaxI(), shl);
    i64 mr = 0;
    const i64 n = ring_flows(F, j);
    for (i64 x = threadIdx.x; x < n; x += FT) {
      int n1, r1, n2, r2;
      i64 by;
      step_flow(T, F, j, F.rs[j] ? 1 : 0, x, n1, r1, n2, r2, by);
      mr = max(mr, tau_of(T, n1, r1, n2, r2, by));
    }
    mr = block_reduce(mr, MaxI(), shl);
    if (threadIdx.x == 0) {
      ab_rs[j] = m;
      ab_ring[j] = mr;
    }
  }
  if (threadIdx.x == 0) {
    i64 e = 0, ab = 0;
    for (int j = 0; j < J; ++j) {
      e = (F.pred[j] ? e : 0) + ab_rs[j] + 2 * (F.D - 1) * ab_ring[j];
      ab = max(ab, e);
    }
    o[1] = ab;
    nact = 0;
    nfree = 0;
    nfct = 0;
    t_now = 0;
    sync_flow_sh = 0;
    nstart = 0;
    for (int j = 0; j < J; ++j) {
      G[j].cur = 0;
      G[j].steps = seg_steps(F, j);
      G[j].pending = 0;
      G[j].live = 0;
      G[j].done_max = 0;
      G[j].completion = FINF;
      if (!F.pred[j]) {
        start_seg[nstart] = j;
        start_step[nstart++] = 0;
      }
    }
  }
  __syncthreads();
  int next_slot_base = 0;  // slots [0, next_slot_base) have been handed out (uniform)
  for (;;) {
    // start the queued steps: their flows arrive now
    for (int q = 0; q < nstart; ++q) {
      const int j = start_seg[q], st = start_step[q];
      const i64 n = (F.rs[j] && st == 0) ? rs_flows(F, j) : ring_flows(F, j);
      const int nf0 = nfree;
      for (i64 x = threadIdx.x; x < n; x += FT) {
        int n1, r1, n2, r2;
        i64 by;
        step_flow(T, F, j, st, x, n1, r1, n2, r2, by);
        // slot: reuse a freed one, else a fresh one
        const int slot = x < nf0 ? W.freel[nf0 - 1 - x] : next_slot_base + (int)(x - nf0);
        make_flow(T, W.fl[slot], n1, r1, n2, r2, by, j, t_now);
        W.act[nact + x] = slot;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        G[j].pending = (int)n;
        G[j].live = 1;
        G[j].done_max = 0;
        nact += (int)n;
        nfree = nf0 > n ? nf0 - (int)n : 0;
      }
      next_slot_base += n > nf0 ? (int)(n - nf0) : 0;
      __syncthreads();
    }
    if (threadIdx.x == 0) nstart = 0;
    __syncthreads();
    const int na = nact;
    if (na) maxmin(T, W, na, shd, shi);
    // next drain: d = ceil(rem / rate) per flow
    i64 dmin = FINF;
    for (int q = threadIdx.x; q < na; q += FT) {
      FlowRec& f = W.fl[W.act[q]];
      f.d = f.rem <= 0.0 ? 0 : (i64)ceil(__ddiv_rn(f.rem, f.rate));
      dmin = lmin(dmin, f.d);
    }
    dmin = block_reduce(dmin, MinI(), shl);
    i64 tev = FINF;
    for (int j = threadIdx.x; j < J; j += FT) tev = lmin(tev, G[j].completion);
    tev = block_reduce(tev, MinI(), shl);
    const i64 t = t_now;
    const i64 tdr = dmin == FINF ? FINF : t + dmin;
    if (tdr == FINF && tev == FINF) break;
    if (tdr <= tev) {
      const double delta = (double)dmin;
      for (int q = threadIdx.x; q < na; q += FT) {
        FlowRec& f = W.fl[W.act[q]];
        if (f.d == dmin) {
          const i64 done = tdr + f.alpha;
          W.fct[atomicAdd(&nfct, 1)] = done - f.arrive;
          atomicMax((unsigned long long*)&G[f.seg].done_max, (unsigned long long)done);
          atomicSub(&G[f.seg].pending, 1);
          f.frz = -1;  // finished
        } else {
          f.rem = __dsub_rn(f.rem, __dmul_rn(f.rate, delta));
        }
      }
      __syncthreads();
      // compact the active list (order-free: every reduction is a min / count)
      if (threadIdx.x == 0) {
        int w = 0;
        for (int q = 0; q < na; ++q) {
          const int s = W.act[q];
          if (W.fl[s].frz == -1) W.freel[nfree++] = s;
          else W.act[w++] = s;
        }
        nact = w;
        t_now = tdr;
        for (int j = 0; j < J; ++j)
          if (G[j].live && G[j].pending == 0 && G[j].completion == FINF) G[j].completion = G[j].done_max;
      }
      __syncthreads();
    } else {
      const double delta = (double)(tev - t);
      for (int q = threadIdx.x; q < na; q += FT) {
        FlowRec& f = W.fl[W.act[q]];
        f.rem = __dsub_rn(f.rem, __dmul_rn(f.rate, delta));
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        t_now = tev;
        for (int j = 0; j < J; ++j) {
          if (G[j].completion != tev) continue;
          G[j].completion = FINF;
          G[j].live = 0;
          if (G[j].cur + 1 < G[j].steps) {
            start_seg[nstart] = j;
            start_step[nstart++] = ++G[j].cur;
          } else {
            sync_flow_sh = max(sync_flow_sh, tev);
            if (j + 1 < J && F.pred[j + 1]) {
              start_seg[nstart] = j + 1;
              start_step[nstart++] = 0;
            }
          }
        }
      }
      __syncthreads();
    }
  }
  if (threadIdx.x == 0) {
    o[0] = 0;
    o[2] = sync_flow_sh;
    o[3] = nfct;
  }
}

// ---- K_flow_stats: nearest-rank percentiles (MSB radix select) -------------------------
__device__ i64 radix_select(const i64* v, i64 n, i64 rank /* 0-based */, int* hist, i64* shl, int* shsel) {
  u64 prefix = 0;
  i64 need = rank;
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int q = threadIdx.x; q < 256; q += FT) hist[q] = 0;
    __syncthreads();
    const u64 hi_mask = shift == 56 ? 0 : (~0ull << (shift + 8));
    for (i64 x = threadIdx.x; x < n; x += FT) {
      const u64 u = (u64)v[x];
      if ((u & hi_mask) == prefix) atomicAdd(&hist[(u >> shift) & 255], 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int dgt = 0;
      i64 acc = 0;
      for (; dgt < 256; ++dgt) {
        if (acc + hist[dgt] > need) break;
        acc += hist[dgt];
      }
      shsel[0] = dgt;
      shl[0] = need - acc;
    }
    __syncthreads();
    prefix |= (u64)shsel[0] << shift;
    need = shl[0];
    __syncthreads();
  }
  return (i64)prefix;
}

__global__ void __launch_bounds__(FT) k_flow_stats(const i64* __restrict__ fct_off, const i64* __restrict__ fct_all,
                                                   i64* __restrict__ out) {
  __shared__ int hist[256];
  __shared__ i64 shl[FT / 32];
  __shared__ int shsel[1];
  const int b = blockIdx.x;
  i64* o = out + (i64)b * NOUT;
  const i64 n = o[3];
  if (o[0] != 0 || n == 0) {
    if (threadIdx.x >= 4 && threadIdx.x < NOUT) o[threadIdx.x] = 0;
    return;
  }
  const i64* v = fct_all + fct_off[b];
  // nearest rank r = ceil(p n), p = 50/100, 99/100, 999/1000 (1-based)
  const i64 r50 = (n * 50 + 99) / 100, r99 = (n * 99 + 99) / 100, r999 = (n * 999 + 999) / 1000;
  const i64 p50 = radix_select(v, n, r50 - 1, hist, shl, shsel);
  const i64 p99 = radix_select(v, n, r99 - 1, hist, shl, shsel);
  const i64 p999 = radix_select(v, n, r999 - 1, hist, shl, shsel);
  i64 mx = 0;
  for (i64 x = threadIdx.x; x < n; x += FT) mx = max(mx, v[x]);
  mx = block_reduce(mx, MaxI(), shl);
  if (threadIdx.x == 0) {
    o[4] = p50;
    o[5] = p99;
    o[6] = p999;
    o[7] = mx;
  }
}

// host side of hsim_flow_resim (host.cu does argument checks)
int launch_flow(hsim_handle* h, const Tables* dT, const Tables& hT, const int64_t* idx, int32_t k, int64_t* out,
                int64_t* fct, int64_t fct_cap, cudaStream_t st) {
  call_begin(h, st);
  const int nmax = hT.n_nodes * hT.gpn;  // each GPU sends at most one flow at a time
  const int nlink = nmax * 6;
  const size_t per = ((sizeof(FlowRec) + 12) * (size_t)nmax + 15 + (size_t)nlink * 16 + 255) & ~(size_t)255;
  // flows per candidate (device), then the FCT storage offsets (host)
  void* buf = nullptr;
  if (ensure_flow_scratch(h, (size_t)k * 16 + 64, &buf)) return HSIM_ENOMEM;
  i64* d_n = (i64*)buf;
  k_flow_count<<<k, FT, 0, st>>>(dT, idx, k, d_n);
  i64* hn = new i64[k + 1];
  cudaMemcpyAsync(hn, d_n, (size_t)k * 8, cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) {
    delete[] hn;
    set_error("k_flow_count failed");
    return HSIM_ECUDA;
  }
  i64 tot = 0;
  for (int b = 0; b < k; ++b) {
    const i64 nb = hn[b];
    hn[b] = tot;
    tot += nb;
  }
  hn[k] = tot;
  const size_t need = (size_t)k * per + (size_t)(k + 1) * 8 + (size_t)tot * 8 + 256;
  if (ensure_flow_scratch(h, need, &buf)) {
    delete[] hn;
    return HSIM_ENOMEM;
  }
  unsigned char* sc = (unsigned char*)buf;
  i64* d_off = (i64*)(sc + (size_t)k * per);
  i64* d_fct = d_off + (k + 1);
  cudaMemcpyAsync(d_off, hn, (size_t)(k + 1) * 8, cudaMemcpyHostToDevice, st);
  k_flow_sim<<<k, FT, 0, st>>>(dT, idx, k, sc, per, nmax, nlink, d_off, out, d_fct);
  k_flow_stats<<<k, FT, 0, st>>>(d_off, d_fct, out);
  if (fct && fct_cap > 0) {  // per candidate: its FCTs (up to fct_cap), unordered
    for (int b = 0; b < k; ++b) {
      const i64 nb = hn[b + 1] - hn[b];
      if (nb > 0) cudaMemcpyAsync(fct + (i64)b * fct_cap, d_fct + hn[b], (size_t)(nb < fct_cap ? nb : fct_cap) * 8,
                                  cudaMemcpyDeviceToDevice, st);
    }
  }
  cudaStreamSynchronize(st);  // hn is freed below; the copies above are enqueued with it alive
  delete[] hn;
  call_end(h, st);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(cudaGetErrorString(e));
    return HSIM_ECUDA;
  }
  return HSIM_OK;
}

}  // namespace hsim
