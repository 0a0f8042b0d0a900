// hsim_core.cuh — product-side data layout and per-candidate arithmetic.
//
// Device tables built by host.cu (hsim_create) and the __host__ __device__
// functions that evaluate one candidate: decode (DESIGN.md C.2), partition
// (C.4), stage durations (C.5), 1F1B max-plus (C.7),
// gradient sync with reshard (C.6/C.8).  The kernels in
// kernels.cu call these; host.cu calls the partition part only to render
// hsim_decode's JSON (never to produce a timing: there is no CPU path).
//
// Exactness (DESIGN.md C.0): durations are ceil((double)x / r), one IEEE RN
// division (__ddiv_rn on the device; host built with -ffp-contract=off), the
// rest int64 + / max.  Device code is compiled with -fmad=false.
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define HD __host__ __device__ __forceinline__
#define HDN static __host__ __device__ __noinline__   // one copy of large per-candidate bodies (I-cache)
#else
#define HD inline
#define HDN static
#endif
#ifndef HSIM_FASTP
#define HSIM_FASTP 8   // deepest pipeline evaluated register-resident (compile-time P)
#endif

namespace hsim {

typedef int64_t i64;
typedef uint64_t u64;
typedef uint32_t u32;

constexpr int MAXT = 4;      // device types
constexpr int MAXG = 8;      // GPUs per node
constexpr int MAXC = 4;      // classes per template
constexpr int MAXP = 64;     // stages per pipeline
constexpr int MAXLC = 64;    // distinct link classes
constexpr int FASTP = HSIM_FASTP;
constexpr int CHUNK = 32;    // candidates per scheduling chunk (one warp)

struct Link { i64 alpha; double beta; };  // alpha ns, beta B/ns

// One stage of a class record (crec).  128 B, 8-byte aligned.
struct StageRec {
  i64 layer_f, layer_b;   // per-layer fwd / bwd incl. TP all-reduce / EP all-to-all (C.5)
  i64 tcomp;              // compute-only fwd+bwd of one layer: partition weight input (C.4)
  i64 fext, gext;         // emb (stage 0) + head (stage P-1) fwd / bwd
  i64 wext;               // emb+head fwd+bwd for the batch weight (C.4)
  u64 tp_mask;            // link classes of this stage group's TP ring (reshard, A14)
  u64 dp_mask[4];         // link classes of intra-class DP ring edges, rings q < 2^k (C.6)
  int32_t type, tp, l0, lg_tp;          // device type, TP, base layer split, log2(tp)
  int32_t first_node, first_base, last_node, last_base;  // replica 0 / replica D-1 group
  int32_t _pad[2];
};
static_assert(sizeof(StageRec) == 128, "StageRec layout");

struct CrecHdr {
  int32_t P, D, U, nd;    // stages, replicas, sub-classes, #layer digits
  u32 pw;                 // (2 r_layer + 1)^nd: radix of the class's digit block
  int32_t _pad[3];
};
static_assert(sizeof(CrecHdr) == 32, "CrecHdr layout");
// crec layout in the int64 pool: CrecHdr (4 x i64) | StageRec[P] (16 x i64 each) | U x (i64 k_u, i64 c[P-1])
constexpr int HDR_WORDS = 4;

struct TplRec {
  i64 prefix;             // first candidate index
  int32_t b, M, C, D;     // micro-batch size, #micro-batches, classes, total replicas
  int32_t crec[MAXC];     // int64-offsets of the class records in the pool
};

struct Tables {
  // model-derived
  i64 L;
  i64 seg_layer_bytes;    // W_layer * bpe_grad
  i64 seg_first_bytes;    // V*h*bpe_grad (embedding with layer 0)
  i64 seg_last_bytes;     // (V*h*!tied + h)*bpe_grad (head + final norm with layer L-1)
  int32_t r_layer, r_batch;
  // templates
  i64 n_tpl, N, n_chunks;
  const i64* tpl_prefix;  // [n_tpl + 1] first candidate of each template
  const i64* tpl_cprefix; // [n_tpl + 1] first chunk of each template (chunks never straddle templates)
  const TplRec* tpl;      // [n_tpl]
  const i64* pool;        // crec pool
  // links
  int32_t n_lc, n_nodes;
  Link lc[MAXLC];
  int8_t lc_same[MAXT][MAXG][MAXG];               // same node: link class of i -> j
  int8_t lc_cross[MAXT][MAXG][MAXT][MAXG];        // different nodes: (t1, r1) -> (t2, r2)
  const int8_t* node_type;                        // [n_nodes]
};

// --- C.0 --------------------------------------------------------------------
HD i64 ceilq(i64 x, double r) {
#ifdef __CUDA_ARCH__
  return x == 0 ? 0 : (i64)ceil(__ddiv_rn((double)x, r));
#else
  return x == 0 ? 0 : (i64)__builtin_ceil((double)x / r);
#endif
}
HD i64 ceil_div(i64 a, i64 b) { return (a + b - 1) / b; }
HD i64 imax(i64 a, i64 b) { return a > b ? a : b; }
HD i64 imin(i64 a, i64 b) { return a < b ? a : b; }

// max over the link classes in `mask` of alpha + ceil(x / beta)  (C.6 tau_e)
HD i64 eval_mask(const Tables& T, u64 mask, i64 x) {
  i64 best = 0;
  while (mask) {
#ifdef __CUDA_ARCH__
    int b = __ffsll((long long)mask) - 1;
#else
    int b = __builtin_ctzll(mask);
#endif
    mask &= mask - 1;
    best = imax(best, T.lc[b].alpha + ceilq(x, T.lc[b].beta));
  }
  return best;
}

HD const CrecHdr* crec_hdr(const Tables& T, int32_t off) { return (const CrecHdr*)(T.pool + off); }
HD const StageRec* crec_stages(const Tables& T, int32_t off) { return (const StageRec*)(T.pool + off + HDR_WORDS); }
HD const i64* crec_sub(const Tables& T, int32_t off, int P, int u) {
  return T.pool + off + HDR_WORDS + 16 * P + (i64)u * P;  // (k_u, c[0..P-2]) = P int64
}

// upper_bound(x) - 1 over a sorted int64 array of n+1 entries (first entry 0)
HD i64 bsearch_le(const i64* a, i64 n, i64 x) {
  i64 lo = 0, hi = n;
  while (hi - lo > 1) {
    i64 mid = (lo + hi) >> 1;
    if (a[mid] <= x) lo = mid; else hi = mid;
  }
  return lo;
}
HD i64 find_template(const Tables& T, i64 i) { return bsearch_le(T.tpl_prefix, T.n_tpl, i); }

// Decoded + partitioned candidate (steps a0 + a1), without per-stage arrays:
// layer counts are re-derived from the class's digit block when needed.
struct Split {
  u32 dig[MAXC];             // digit block of each class (boundary digits, LSB = boundary 0)
  i64 q[MAXC];               // Hamilton floor per replica of class c
  i64 seats[MAXC];           // replicas 0..seats-1 of class c get +1
  i64 add[MAXC];             // epsilon (c < C-1) or floor(R / D_last)
  i64 rm;                    // last class: replicas < rm get +1
  int32_t C;
};
HD i64 replica_mb(const Split& s, int c, i64 k) {
  i64 m = s.q[c] + (k < s.seats[c] ? 1 : 0) + s.add[c];
  if (c == s.C - 1) m += (k < s.rm ? 1 : 0);
  return m;
}

// Sequential walk over one class's stages: l_s = l0_s + delta_s - delta_{s-1}
// with delta_s = digit_s - r (DESIGN.md C.2/C.4).
struct LayerWalk {
  u32 dig;
  int nd, dprev, s;
  u32 bl;
  int r;
  HD int next(const StageRec* st) {
    int d = 0;
    if (s < nd) { d = (int)(dig % bl) - r; dig /= bl; }
    int l = st[s].l0 + d - dprev;
    dprev = d;
    ++s;
    return l;
  }
};
HD LayerWalk walk(const Tables& T, const CrecHdr* h, u32 dig) {
  return LayerWalk{dig, h->nd, 0, 0, (u32)(2 * T.r_layer + 1), T.r_layer};
}

// Digits are least-significant first: class 0's boundaries, class 1's, ...,
// then the batch digits of classes 0..C-2.  Layer split = template base split
// + deltas; batch split = Hamilton over all replicas with weights
// floor(2^40 / slowest stage) (C.4).  Returns 0, -1 (layer) or -2 (batch).
HDN int partition(const Tables& T, const TplRec& tp, i64 local, Split& sp) {
  const int C = tp.C;
  sp.C = C;
  const u32 bb = (u32)(2 * T.r_batch + 1);
  u32 loc = (u32)local;  // radix < 2^31 (validated at create)
  i64 w[MAXC];
  int status = 0;
  for (int c = 0; c < C; ++c) {
    const CrecHdr* h = crec_hdr(T, tp.crec[c]);
    const StageRec* st = crec_stages(T, tp.crec[c]);
    sp.dig[c] = loc % h->pw;
    loc /= h->pw;
    LayerWalk lw = walk(T, h, sp.dig[c]);
    i64 worst = 0;
    for (int s = 0; s < h->P; ++s) {
      const int l = lw.next(st);
      if (l < 1) status = -1;
      worst = imax(worst, (i64)l * st[s].tcomp + st[s].wext);
    }
    w[c] = ((i64)1 << 40) / worst;
  }
  if (status) return status;
  i64 W = 0, eps[MAXC], R = 0;
  for (int c = 0; c < C; ++c) W += (i64)crec_hdr(T, tp.crec[c])->D * w[c];
  for (int c = 0; c < C - 1; ++c) { eps[c] = (i64)(loc % bb) - T.r_batch; loc /= bb; }
  i64 left = tp.M, rem[MAXC];
  for (int c = 0; c < C; ++c) {
    sp.q[c] = (i64)tp.M * w[c] / W;
    rem[c] = (i64)tp.M * w[c] % W;
    left -= (i64)crec_hdr(T, tp.crec[c])->D * sp.q[c];
    sp.seats[c] = 0;
  }
  // leftover seats to the largest remainders; ties -> lower (class-major) replica
  bool done[MAXC] = {false, false, false, false};
  for (int pass = 0; pass < C && left > 0; ++pass) {
    int best = -1;
    for (int c = 0; c < C; ++c)
      if (!done[c] && (best < 0 || rem[c] > rem[best])) best = c;
    done[best] = true;
    const i64 D = crec_hdr(T, tp.crec[best])->D;
    sp.seats[best] = imin(D, left);
    left -= sp.seats[best];
  }
  for (int c = 0; c < C - 1; ++c) {
    sp.add[c] = eps[c];
    R -= (i64)crec_hdr(T, tp.crec[c])->D * eps[c];
  }
  const i64 Dl = crec_hdr(T, tp.crec[C - 1])->D;
  const i64 fl = R >= 0 ? R / Dl : -((-R + Dl - 1) / Dl);
  sp.add[C - 1] = fl;
  sp.rm = R - fl * Dl;
  for (int c = 0; c < C; ++c)
    if (replica_mb(sp, c, crec_hdr(T, tp.crec[c])->D - 1) < 1) return -2;  // m non-increasing in k
  return 0;
}

// --- step a4: non-interleaved 1F1B as a level-synchronous max-plus sweep -----
// Level of F(s,j): s+j if j <= P-1-s else 2j+s; of B(s,j): 2P-1-s+2j
// (DESIGN.md C.7).  Every op's inputs were produced at an earlier level, at
// most one op per stage per level, and the only same-level hazard is F(s-1)
// next to F(s) in the warm-up, so stages are visited in descending order.
// State per stage: X = end of its last op, R = last F end + c_s (what stage
// s+1 receives), Lb = last B end + c_{s-1} (what stage s-1 receives).
HD i64 level_F(int P, int s, i64 j) { return j <= P - 1 - s ? s + j : 2 * j + s; }
HD i64 level_B(int P, int s, i64 j) { return 2 * P - 1 - s + 2 * j; }

// generic depth (P <= MAXP), per-thread arrays
HD i64 pipeline_generic(int P, i64 m, const i64* f, const i64* g, const i64* c) {
  i64 X[MAXP], R[MAXP], Lb[MAXP];
  i64 lastF = 0;
  for (int s = 0; s < P; ++s) X[s] = R[s] = Lb[s] = 0;
  const i64 levels = 2 * (m + P - 1);
  for (i64 lv = 0; lv < levels; ++lv) {
    for (int s = P - 1; s >= 0; --s) {
      const i64 jw = lv - s, js = lv - s, jb = lv - (2 * P - 1 - s);
      const bool isF = (jw >= 0 && lv <= P - 1 && jw < m) || (lv >= 2 * P - s && !(js & 1) && (js >> 1) < m);
      const bool isB = jb >= 0 && !(jb & 1) && (jb >> 1) < m;
      if (isF) {
        const i64 e = imax(X[s], s == 0 ? 0 : R[s - 1]) + f[s];
        X[s] = e;
        if (s < P - 1) R[s] = e + c[s]; else lastF = e;
      } else if (isB) {
        const i64 e = imax(X[s], s == P - 1 ? lastF : Lb[s + 1]) + g[s];
        X[s] = e;
        if (s > 0) Lb[s] = e + c[s - 1];
      }
    }
  }
  return X[0];
}

// compile-time depth: every array is register-resident; the steady phase
// (levels [2P-1, 2m), every stage busy, F iff level = s mod 2) has no
// per-cell bookkeeping: one int64 max and two int64 adds per cell.
template <int P>
struct Pipe {
  i64 f[P], g[P], c[P], X[P], R[P], Lb[P], lastF;

  HD void generic_level(i64 lv, i64 m) {
#pragma unroll
    for (int s = P - 1; s >= 0; --s) {
      const i64 js = lv - s, jb = lv - (2 * P - 1 - s);
      const bool isF = (js >= 0 && lv <= P - 1 && js < m) || (lv >= 2 * P - s && !(js & 1) && (js >> 1) < m);
      const bool isB = jb >= 0 && !(jb & 1) && (jb >> 1) < m;
      if (isF) {
        const i64 e = imax(X[s], s == 0 ? (i64)0 : R[s == 0 ? 0 : s - 1]) + f[s];
        X[s] = e;
        if (s < P - 1) R[s] = e + c[s]; else lastF = e;
      } else if (isB) {
        const i64 e = imax(X[s], s == P - 1 ? lastF : Lb[s == P - 1 ? s : s + 1]) + g[s];
        X[s] = e;
        if (s > 0) Lb[s] = e + c[s == 0 ? 0 : s - 1];
      }
    }
  }
  // one steady level of parity par: stages with s % 2 == par run F, the others B
  template <int par>
  HD void steady_level() {
#pragma unroll
    for (int s = P - 1; s >= 0; --s) {
      if ((s & 1) == par) {
        const i64 e = imax(X[s], s == 0 ? (i64)0 : R[s == 0 ? 0 : s - 1]) + f[s];
        X[s] = e;
        if (s < P - 1) R[s] = e + c[s]; else lastF = e;
      } else {
        const i64 e = imax(X[s], s == P - 1 ? lastF : Lb[s == P - 1 ? s : s + 1]) + g[s];
        X[s] = e;
        if (s > 0) Lb[s] = e + c[s == 0 ? 0 : s - 1];
      }
    }
  }
  HD i64 run(i64 m) {
#pragma unroll
    for (int s = 0; s < P; ++s) X[s] = R[s] = Lb[s] = 0;
    lastF = 0;
    const i64 total = 2 * (m + P - 1);
    const i64 lo = 2 * P - 1;
    const i64 hi = m >= P ? 2 * m : lo;
    const i64 e1 = lo < total ? lo : total;
    for (i64 lv = 0; lv < e1; ++lv) generic_level(lv, m);
    if (hi > lo) {
      steady_level<1>();  // level 2P-1 is odd
      for (i64 k = 0; k < m - P; ++k) {
        steady_level<0>();
        steady_level<1>();
      }
    }
    for (i64 lv = hi > lo ? hi : lo; lv < total; ++lv) generic_level(lv, m);
    return X[0];
  }
};

// T_pipe of every sub-class of class c, max-reduced into T0; adds the cells.
template <int P>
HDN void class_pipes(const Tables& T, const TplRec& tp, const Split& sp, int c, i64& T0, i64& cells) {
  const int32_t off = tp.crec[c];
  const CrecHdr* h = crec_hdr(T, off);
  const StageRec* st = crec_stages(T, off);
  Pipe<P> p;
  LayerWalk lw = walk(T, h, sp.dig[c]);
#pragma unroll
  for (int s = 0; s < P; ++s) {
    const i64 l = lw.next(st);
    p.f[s] = l * st[s].layer_f + st[s].fext;
    p.g[s] = l * st[s].layer_b + st[s].gext;
  }
  for (int u = 0; u < h->U; ++u) {
    const i64* sub = crec_sub(T, off, P, u);
#pragma unroll
    for (int s = 0; s + 1 < P; ++s) p.c[s] = sub[1 + s];
    const i64 m = replica_mb(sp, c, sub[0]);
    cells += 2 * P * m;
    T0 = imax(T0, p.run(m));
  }
}

HDN void class_pipes_generic(const Tables& T, const TplRec& tp, const Split& sp, int c, i64& T0, i64& cells) {
  const int32_t off = tp.crec[c];
  const CrecHdr* h = crec_hdr(T, off);
  const StageRec* st = crec_stages(T, off);
  const int P = h->P;
  i64 f[MAXP], g[MAXP];
  LayerWalk lw = walk(T, h, sp.dig[c]);
  for (int s = 0; s < P; ++s) {
    const i64 l = lw.next(st);
    f[s] = l * st[s].layer_f + st[s].fext;
    g[s] = l * st[s].layer_b + st[s].gext;
  }
  for (int u = 0; u < h->U; ++u) {
    const i64* sub = crec_sub(T, off, P, u);
    const i64 m = replica_mb(sp, c, sub[0]);
    cells += 2 * P * m;
    T0 = imax(T0, pipeline_generic(P, m, f, g, sub + 1));
  }
}

// --- step a5: gradient sync (C.6, C.8) -----------------------------------------
// Segments = common refinement of the classes' layer boundaries, in ascending
// layer order, list-scheduled FIFO per (class, stage) group from T0.
HDN i64 grad_sync(const Tables& T, const TplRec& tp, const Split& sp, i64 T0) {
  const int C = tp.C;
  int sc[MAXC];
  i64 nextcut[MAXC], cur_free[MAXC];
  LayerWalk lw[MAXC];
  const StageRec* st[MAXC];
  for (int c = 0; c < C; ++c) {
    const CrecHdr* h = crec_hdr(T, tp.crec[c]);
    st[c] = crec_stages(T, tp.crec[c]);
    lw[c] = walk(T, h, sp.dig[c]);
    sc[c] = 0;
    const i64 l0 = lw[c].next(st[c]);
    nextcut[c] = h->P > 1 ? l0 : T.L;
    cur_free[c] = T0;
  }
  i64 a = 0, Titer = T0;
  while (a < T.L) {
    i64 z = T.L;
    for (int c = 0; c < C; ++c) z = imin(z, nextcut[c]);
    const i64 S = (z - a) * T.seg_layer_bytes + (a == 0 ? T.seg_first_bytes : 0) + (z == T.L ? T.seg_last_bytes : 0);
    int tstar = 1 << 30, lg = 0;
    for (int c = 0; c < C; ++c) {
      const StageRec& s = st[c][sc[c]];
      if (s.tp < tstar) { tstar = s.tp; lg = s.lg_tp; }
    }
    const i64 xs = ceil_div(S, tstar);
    i64 RS = 0;
    u64 mask = 0;
    for (int c = 0; c < C; ++c) {
      const StageRec& s = st[c][sc[c]];
      if (s.tp != tstar) RS = imax(RS, eval_mask(T, s.tp_mask, xs));  // reshard (A14)
      mask |= s.dp_mask[lg];
      // edge from the last replica of class c to the first replica of the next
      // class (wrap: class C-1 -> class 0), ring q through device base + q
      const int cn = c + 1 < C ? c + 1 : 0;
      const StageRec& t = st[cn][sc[cn]];
      const int n1 = s.last_node, n2 = t.first_node;
      const int t1 = T.node_type[n1], t2 = T.node_type[n2];
      for (int q = 0; q < tstar; ++q) {
        const int r1 = s.last_base + q, r2 = t.first_base + q;
        const int id = n1 == n2 ? T.lc_same[t1][r1][r2] : T.lc_cross[t1][r1][t2][r2];
        mask |= (u64)1 << id;
      }
    }
    const i64 chunk = ceil_div(xs, (i64)tp.D);
    const i64 AR = 2 * (i64)(tp.D - 1) * eval_mask(T, mask, chunk);
    i64 start = 0;
    for (int c = 0; c < C; ++c) start = imax(start, cur_free[c]);
    const i64 end = start + RS + AR;
    for (int c = 0; c < C; ++c) cur_free[c] = end;
    Titer = imax(Titer, end);
    for (int c = 0; c < C; ++c) {  // advance classes whose stage ends at z
      if (nextcut[c] == z && z < T.L) {
        sc[c]++;
        const int P = crec_hdr(T, tp.crec[c])->P;
        const i64 l = lw[c].next(st[c]);
        nextcut[c] = sc[c] + 1 < P ? nextcut[c] + l : T.L;
        cur_free[c] = T0;
      }
    }
    a = z;
  }
  return Titer;
}

// --- whole candidate (steps a0-a5) ---------------------------------------------
// Returns the iteration time in ns or a negative status; *cells (if non-null)
// receives sum_u 2 * P_u * m_u (the 1F1B cells simulated).
HDN i64 eval_in_template(const Tables& T, const TplRec& tp, i64 local, i64* cells) {
  Split sp;
  const int st = partition(T, tp, local, sp);
  if (st) return st;
  i64 T0 = 0, ncell = 0;
  for (int c = 0; c < tp.C; ++c) {
    switch (crec_hdr(T, tp.crec[c])->P) {
      case 1: class_pipes<1>(T, tp, sp, c, T0, ncell); break;
      case 2: class_pipes<2>(T, tp, sp, c, T0, ncell); break;
#if HSIM_FASTP >= 3
      case 3: class_pipes<3>(T, tp, sp, c, T0, ncell); break;
#endif
#if HSIM_FASTP >= 4
      case 4: class_pipes<4>(T, tp, sp, c, T0, ncell); break;
#endif
#if HSIM_FASTP >= 5
      case 5: class_pipes<5>(T, tp, sp, c, T0, ncell); break;
#endif
#if HSIM_FASTP >= 6
      case 6: class_pipes<6>(T, tp, sp, c, T0, ncell); break;
#endif
#if HSIM_FASTP >= 7
      case 7: class_pipes<7>(T, tp, sp, c, T0, ncell); break;
#endif
#if HSIM_FASTP >= 8
      case 8: class_pipes<8>(T, tp, sp, c, T0, ncell); break;
#endif
      default: class_pipes_generic(T, tp, sp, c, T0, ncell); break;
    }
  }
  if (cells) *cells = ncell;
  if (tp.D == 1) return T0;
  return grad_sync(T, tp, sp, T0);
}

#ifdef __CUDACC__
// --- warp-cooperative path for deep pipelines (FASTP < P <= 32) ----------------
// Lanes sweep the 1F1B anti-diagonal wavefront (BASELINE north_star): lane =
// one stage s of one pipeline "job" (candidate x sub-class), floor(32 / P)
// jobs per pass.  Every lane exports one value, the output of its most
// recent op (F: end + c_s, B: end + c_{s-1}); an F reads its left
// neighbour's export, a B its right neighbour's, as of the previous level --
// in 1F1B the producer's most recent op is always the right one (DESIGN.md
// C.7), so one 64-bit __shfl per level suffices.  Warm-up / cool-down levels
// use the closed-form op levels; the steady levels [2P-1, 2m) alternate F/B by
// parity with no bookkeeping.
__device__ __forceinline__ i64 shfl64(i64 v, int src) { return __shfl_sync(0xffffffffu, v, src); }

__device__ __forceinline__ int nth_set_lane(unsigned mask, int n) {
  for (int q = 0; q < n; ++q) mask &= mask - 1;
  return __ffs(mask) - 1;
}

struct LanePipe {
  int P, s, lane;
  i64 m, f, g, cR, cL;  // cR = c_s (0 on the last stage), cL = c_{s-1}
  i64 X, out;
  // one level; every lane of the warp must call it (it shuffles).  In the
  // steady range the op is given by the parity constants, else by the
  // closed-form levels of F(s,j) / B(s,j).
  __device__ __forceinline__ void level(i64 lv, bool steady, int srcS, i64 durS, i64 cS, i64 zS) {
    int src = srcS;
    i64 dur = durS, cc = cS, z = zS;
    bool doOp = true;
    if (!steady) {
      const i64 js = lv - s, jb = lv - (2 * P - 1 - s);
      const bool isF = (js >= 0 && lv <= P - 1 && js < m) || (lv >= 2 * P - s && !(js & 1) && (js >> 1) < m);
      const bool isB = jb >= 0 && !(jb & 1) && (jb >> 1) < m;
      doOp = isF || isB;
      src = isF ? lane - 1 : lane + 1;
      dur = isF ? f : g;
      cc = isF ? cR : cL;
      z = (isF && s == 0) || (isB && s == P - 1) ? 0 : -1;  // stage-0 input / B right after own F
    }
    const i64 v = shfl64(out, src) & z;
    if (doOp) {
      const i64 e = imax(X, v) + dur;
      X = e;
      out = e + cc;
    }
  }
};

// All 32 lanes call it.  `ok` marks lanes whose candidate (this warp's
// template) has a valid split; T0 / cells of those lanes are updated.
static __device__ __noinline__ void warp_class_pipes(const Tables& T, const TplRec& tp, const Split& sp, int c, bool ok,
                                                     i64& T0, i64& cells) {
  const int lane = threadIdx.x & 31;
  const int32_t off = tp.crec[c];
  const CrecHdr* h = crec_hdr(T, off);
  const StageRec* st = crec_stages(T, off);
  const int P = h->P, U = h->U;
  const int nseg = 32 / P;
  const unsigned vmask = __ballot_sync(0xffffffffu, ok);
  const int nv = __popc(vmask);
  const int myrank = __popc(vmask & ((1u << lane) - 1));
  const int seg = lane / P, s = lane - seg * P;
  if (ok)
    for (int u = 0; u < U; ++u) cells += 2 * P * replica_mb(sp, c, crec_sub(T, off, P, u)[0]);
  // this lane's stage layer count is the same for every job of one candidate;
  // it is recomputed per job from the candidate's digit block
  const int njobs = U * nv;
  for (int base = 0; base < njobs; base += nseg) {
    const int q = base + seg;
    const bool act = seg < nseg && q < njobs;
    const int u = act ? q / nv : 0, rank = act ? q - u * nv : 0;
    const int jl = act ? nth_set_lane(vmask, rank) : 0;
    // fetch the job's candidate split from its lane
    Split sj;
    sj.C = tp.C;  // warp-uniform (this lane's own split may be unset)
    sj.q[c] = shfl64(sp.q[c], jl);
    sj.seats[c] = shfl64(sp.seats[c], jl);
    sj.add[c] = shfl64(sp.add[c], jl);
    sj.rm = shfl64(sp.rm, jl);
    const u32 dig = (u32)__shfl_sync(0xffffffffu, (int)sp.dig[c], jl);
    const i64* sub = crec_sub(T, off, P, u);
    LanePipe lp;
    lp.P = P; lp.s = s; lp.lane = lane;
    lp.m = act ? replica_mb(sj, c, sub[0]) : 0;
    LayerWalk lw = walk(T, h, dig);
    int l = 0;
    for (int k = 0; k <= s; ++k) l = lw.next(st);
    lp.f = act ? (i64)l * st[s].layer_f + st[s].fext : 0;
    lp.g = act ? (i64)l * st[s].layer_b + st[s].gext : 0;
    lp.cR = act && s + 1 < P ? sub[1 + s] : 0;
    lp.cL = act && s > 0 ? sub[s] : 0;
    lp.X = 0;
    lp.out = 0;
    // level ranges: warm-up [0, lo), steady [lo, hi) per job, cool-down to total
    const i64 lo = 2 * P - 1;
    const i64 hi = lp.m >= P ? 2 * lp.m : lo;
    const i64 total = act ? 2 * (lp.m + P - 1) : 0;
    i64 totMax = total;
    for (int o = 16; o > 0; o >>= 1) totMax = imax(totMax, (i64)__shfl_xor_sync(0xffffffffu, (long long)totMax, o));
    i64 hiMin = act ? hi : INT64_MAX;
    for (int o = 16; o > 0; o >>= 1) hiMin = imin(hiMin, (i64)__shfl_xor_sync(0xffffffffu, (long long)hiMin, o));
    // per-lane constants of the two steady level parities (lo = 2P-1 is odd)
    const bool oddS = s & 1;
    const int srcO = oddS ? lane - 1 : lane + 1, srcE = oddS ? lane + 1 : lane - 1;
    const i64 durO = oddS ? lp.f : lp.g, durE = oddS ? lp.g : lp.f;
    const i64 cO = oddS ? lp.cR : lp.cL, cE = oddS ? lp.cL : lp.cR;
    const i64 zO = (!oddS && s == P - 1) ? 0 : -1;
    const i64 zE = (oddS ? s == P - 1 : s == 0) ? 0 : -1;
    i64 lv = 0;
    for (; lv < lo && lv < totMax; ++lv) lp.level(lv, false, 0, 0, 0, 0);
    // every job is in its steady range: no bookkeeping, one shuffle per level
    for (; lv + 1 < hiMin; lv += 2) {
      {
        const i64 v = shfl64(lp.out, srcO) & zO;
        const i64 e = imax(lp.X, v) + durO;
        lp.X = e;
        lp.out = e + cO;
      }
      {
        const i64 v = shfl64(lp.out, srcE) & zE;
        const i64 e = imax(lp.X, v) + durE;
        lp.X = e;
        lp.out = e + cE;
      }
    }
    // jobs leaving their steady range at different levels, then cool-down
    for (; lv < totMax; ++lv) {
      const bool odd = lv & 1;
      lp.level(lv, lv >= lo && lv < hi, odd ? srcO : srcE, odd ? durO : durE, odd ? cO : cE, odd ? zO : zE);
    }
    // candidate lane L: its job (u, rank) sits in segment u*nv + rank - base
    for (int uu = 0; uu < U; ++uu) {
      const int qq = uu * nv + myrank;
      const bool mine = ok && qq >= base && qq < base + nseg;
      const i64 got = shfl64(lp.X, mine ? (qq - base) * P : 0);
      if (mine) T0 = imax(T0, got);
    }
  }
}

// Evaluates the candidates of one template held by the lanes with in_g set
// (all 32 lanes call it; the template is warp-uniform).
__device__ __forceinline__ i64 eval_group(const Tables& T, const TplRec& tp, i64 local, bool in_g) {
  Split sp;
  int stt = 1;
  if (in_g) stt = partition(T, tp, local, sp);
  const bool ok = in_g && stt == 0;
  i64 T0 = 0, ncell = 0;
  for (int c = 0; c < tp.C; ++c) {
    const int P = crec_hdr(T, tp.crec[c])->P;
    if (P > FASTP && P <= 32) {
      warp_class_pipes(T, tp, sp, c, ok, T0, ncell);
    } else if (ok) {
      switch (P) {
        case 1: class_pipes<1>(T, tp, sp, c, T0, ncell); break;
        case 2: class_pipes<2>(T, tp, sp, c, T0, ncell); break;
#if HSIM_FASTP >= 3
        case 3: class_pipes<3>(T, tp, sp, c, T0, ncell); break;
#endif
#if HSIM_FASTP >= 4
        case 4: class_pipes<4>(T, tp, sp, c, T0, ncell); break;
#endif
#if HSIM_FASTP >= 5
        case 5: class_pipes<5>(T, tp, sp, c, T0, ncell); break;
#endif
#if HSIM_FASTP >= 6
        case 6: class_pipes<6>(T, tp, sp, c, T0, ncell); break;
#endif
#if HSIM_FASTP >= 7
        case 7: class_pipes<7>(T, tp, sp, c, T0, ncell); break;
#endif
#if HSIM_FASTP >= 8
        case 8: class_pipes<8>(T, tp, sp, c, T0, ncell); break;
#endif
        default: class_pipes_generic(T, tp, sp, c, T0, ncell); break;
      }
    }
  }
  if (!ok) return in_g ? (i64)stt : INT64_MIN;
  if (tp.D == 1) return T0;
  return grad_sync(T, tp, sp, T0);
}
#endif

HD i64 eval_candidate(const Tables& T, i64 i, i64* cells) {
  if (i < 0 || i >= T.N) return INT64_MIN;
  const TplRec tp = T.tpl[find_template(T, i)];
  return eval_in_template(T, tp, i - tp.prefix, cells);
}

}  // namespace hsim
