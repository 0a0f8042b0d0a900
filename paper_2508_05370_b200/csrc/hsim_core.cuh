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
#include <math.h>
#include <stdint.h>

#ifdef __CUDACC__
#define HD __host__ __device__ __forceinline__
#define HDN static __host__ __device__ __noinline__   // one copy of large per-candidate bodies (I-cache)
#else
#define HD inline
#define HDN static
#endif
#ifndef HSIM_WHOLE_MAXP
#define HSIM_WHOLE_MAXP 16  // deepest register-resident pipeline with the cyclic c | BL check
#endif
#ifndef HSIM_AFFINE_MAXP
#define HSIM_AFFINE_MAXP 8  // deepest register-resident pipeline with the affine-regime jump
#endif
#ifndef HSIM_UNROLL_MAXP
#define HSIM_UNROLL_MAXP 16  // deepest pipeline whose 1F1B warm-up / cool-down levels are fully unrolled
#endif
#ifndef HSIM_FASTP
#define HSIM_FASTP 16  // deepest pipeline evaluated register-resident (compile-time P): 8 or 16
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
  int16_t first_node, first_base, last_node, last_base;  // replica 0 / replica D-1 group
  int32_t type2;          // V.1 mixed TP group: its second device type (-1: homogeneous)
  int32_t _pad;
  i64 emb_b;              // B.1: embedding backward of stage 0 (0 elsewhere)
};
static_assert(sizeof(StageRec) == 128, "StageRec layout");

// n / d for 0 <= n < 2^31 as ((u64)n * m) >> sh with l = ceil(log2 d),
// m = floor(2^(31+l) / d) + 1 < 2^32, sh = 31 + l (Granlund-Montgomery, N = 31)
struct FastDiv {
  u32 m, sh;
  HD u32 div(u32 n) const { return (u32)(((u64)n * m) >> sh); }
};
inline FastDiv make_fastdiv(u32 d) {
  u32 l = 0;
  while (((u64)1 << l) < d) ++l;
  return FastDiv{(u32)((((u64)1 << (31 + l)) / d) + 1), 31 + l};
}

struct CrecHdr {
  int32_t P, D, U, nd;    // stages, replicas, sub-classes, #layer digits
  u32 pw;                 // (2 r_layer + 1)^nd: radix of the class's digit block
  FastDiv pwdiv;          // division by pw
  int32_t woff;           // offset of the class's rows in Tables.wtab, -1 = none
};
static_assert(sizeof(CrecHdr) == 32, "CrecHdr layout");
// crec layout in the int64 pool: CrecHdr (4 x i64) | StageRec[P] (16 x i64 each) |
// U x (i64 k_u, i64 c[P-1], i64 c_wrap): sub-class records of P + 1 words; c_wrap
// = the stage P-1 -> stage 0 p2p cost of the interleaved schedule (V.2; else 0)
constexpr int HDR_WORDS = 4;

struct TplRec {
  i64 prefix;             // first candidate index
  int32_t b, M, C, D;     // micro-batch size, #micro-batches, classes, total replicas
  int32_t crec[MAXC];     // int64-offsets of the class records in the pool
  uint32_t pmask;         // bit min(P, 31) set for every class depth P (V.2: P >= 2 -> bit 0)
  int32_t flags;          // bit 0: V.3 expert parallelism across the replicas (dense-only gradient sync);
                          // bit 1: V.1 mixed TP groups (the DP ring's wrap edge is in dp_mask)
  double rD;              // 1.0 / D (ring chunk: ceil division by D with exact fix-up)
};

struct Tables {
  // model-derived
  i64 L;
  i64 seg_layer_bytes;    // W_layer * bpe_grad
  i64 seg_first_bytes;    // V*h*bpe_grad (embedding with layer 0)
  i64 seg_last_bytes;     // (V*h*!tied + h)*bpe_grad (head + final norm with layer L-1)
  int32_t r_layer, r_batch;
  FastDiv ldiv, bdiv;     // division by 2 r_layer + 1 / 2 r_batch + 1
  // templates
  i64 n_tpl, N, n_bucket;
  const i64* tpl_prefix;  // [n_tpl + 1] first candidate of each template
  const int32_t* tpl_bucket;  // [n_bucket + 1] template of candidate b << bucket_shift (coarse index)
  const i64* tpl_cprefix;     // [n_tpl + 1] first 32-candidate chunk of each template (chunks never straddle)
  const int32_t* tpl_cbucket; // [n_cbucket + 1] template of chunk b << cbucket_shift (coarse index)
  i64 n_cbucket;
  int32_t cbucket_shift, _pad5;
  int32_t bucket_shift, _pad2;
  const TplRec* tpl;      // [n_tpl]
  const i64* pool;        // crec pool
  // links
  int32_t n_lc, n_nodes;
  Link lc[MAXLC];
  // exact integer form of tau (DESIGN.md C.0): when beta = G / 2^k exactly and
  // every x << k < 2^52 (checked at create), ceil(RN(x / beta)) ==
  // ceil_div(x << k, G), computed from a reciprocal estimate + exact fix-up
  i64 lc_G[MAXLC];
  double lc_rG[MAXLC];     // 1.0 / G (floor estimate, then exact integer fix-up)
  double lc_rb[MAXLC];     // RN(1 / beta) (device ceil division by beta = G / 2^k)
  u64 lc_up[MAXLC];       // classes after this one (ids sorted by beta asc, alpha desc) with a larger alpha
  int8_t lc_k[MAXLC], _pad4[MAXLC];
  int32_t lc_exact, _pad3;
  const u64* xmask_cross;  // [MAXT][MAXG][MAXT][MAXG][4] link classes of edges (t1, b1+q) -> (t2, b2+q), q < 2^lg
  const u64* xmask_same;   // [MAXT][MAXG][MAXG][4] same node
  int8_t lc_same[MAXT][MAXG][MAXG];               // same node: link class of i -> j
  int8_t lc_cross[MAXT][MAXG][MAXT][MAXG];        // different nodes: (t1, r1) -> (t2, r2)
  const int8_t* node_type;                        // [n_nodes]
  // memory feasibility (DESIGN.md M.1), per lg = log2(tp): bytes of state per
  // layer / for the embedding / for the head on one device, and
  // K[lg] = s h (10 t + 24) (activation bytes per layer = ceil(b K / t))
  int32_t mem_check, sync_overlap;
  int32_t interleave, ep_dp;  // DESIGN.md V.2 (v chunks per stage; 1 = off), V.3
  int32_t buckets, _pad7;     // DESIGN.md B.1: 2 = two gradient buckets per stage group
  i64 seg_layer_dense;        // V.3: W_layer without the expert matrices, x bpe_grad
  i64 mem_layer[4], mem_emb[4], mem_head[4], mem_K[4];
  i64 mem_cap[MAXT];
  // f3 flow-level re-simulation (DESIGN.md F.1): rail-only link graph
  const int32_t* type_nodes;       // node ids grouped by device type (placement order)
  int32_t type_node_off[MAXT + 1]; // type t's nodes: type_nodes[off[t] .. off[t+1])
  int32_t gpn, _pad6;              // GPUs per node (every node type)
  double port_cap[MAXT][MAXG][2];  // NVLink egress / ingress port of local rank r, B/ns
  double pcie_cap[MAXT];           // GPU <-> rail NIC path, B/ns
  double nic_cap[MAXT];            // NIC <-> rail switch port, min(NIC, rail), B/ns
  // pipeline dedupe: a class pipeline is a function of (template,
  // class, boundary digits, the class's sub-class micro-batch vector) only; the
  // vector is base + [u < a] + [u < b] (m non-increasing in the replica, at most
  // two +1 steps).  Key = tau | c << wt | dig << (wt + 2) | base << .. | a | b,
  // plus 1 (0 = empty), with the field widths below; dd_ok = 0 when they
  // exceed 63 bits (dedupe then off).
  int32_t dd_ok, dd_wt, dd_wd, dd_wm, dd_wu, _pad8;
  // partition weight table (device only; host: nullptr): for class record h
  // and boundary digits dig, wtab[h.woff + dig] = floor(2^40 / max_s(l_s
  // tcomp_s + wext_s)) | min_s(l_s) << 48 (w = 0 and min 0 when some l_s < 1)
  // -- the per-candidate stage walk of step a1 precomputed per (class, digits)
  const i64* wtab;
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

// ceil(n / d) for 0 <= n < 2^52, 1 <= d < 2^31: floor estimate in fp64 from the
// reciprocal (|error| < 1), then an exact integer fix-up of the remainder
#ifdef __CUDA_ARCH__
// Device form, all in fp64: n < 2^52 and d < 2^31 are exact doubles, the
// truncated estimate q is within 1 of n / d, and the remainder n - q d is an
// integer below 2^33 in magnitude, so one explicit FMA computes it exactly
// (an exact integer result -- no contraction of a rounded expression).
__device__ __forceinline__ i64 ceil_div_rcp_d(double n, double d, double rd) {
  double q = trunc(n * rd);
  double r = fma(-q, d, n);
  if (r < 0.0) { q -= 1.0; r += d; }
  if (r >= d) { q += 1.0; r -= d; }
  return (i64)q + (r != 0.0 ? 1 : 0);
}
#endif
HD i64 ceil_div_rcp(i64 n, i64 d, double rd) {
#ifdef __CUDA_ARCH__
  return ceil_div_rcp_d((double)n, (double)d, rd);
#else
  i64 q = (i64)((double)n * rd);
  i64 r = n - q * d;
  if (r < 0) { q -= 1; r += d; }
  if (r >= d) { q += 1; r -= d; }
  return q + (r != 0 ? 1 : 0);
#endif
}
// alpha_e + ceil(x / beta_e) of link class b (C.6 tau_e)
HD i64 tau_lc(const Tables& T, int b, i64 x) {
#ifdef __CUDA_ARCH__
  // ceil(x / beta) with beta = G / 2^k itself: x / beta = (x << k) / G < 2^52
  // keeps the truncated estimate within 1, and x - q beta = (x 2^k - q G) / 2^k
  // has under 33 significant bits, so the FMA remainder is exact
  if (T.lc_exact) return T.lc[b].alpha + ceil_div_rcp_d((double)x, T.lc[b].beta, T.lc_rb[b]);
#else
  if (T.lc_exact) return T.lc[b].alpha + ceil_div_rcp(x << T.lc_k[b], T.lc_G[b], T.lc_rG[b]);
#endif
  return T.lc[b].alpha + ceilq(x, T.lc[b].beta);
}

// max over the link classes in `mask` of alpha + ceil(x / beta)  (C.6 tau_e).
// Class ids are sorted by (beta ascending, alpha descending), so the lowest bit
// is the slowest class; every later class with alpha <= its alpha is dominated
// (tau never larger) and dropped: the walk visits only the mask's Pareto front.
HD int ffs64(u64 m) {
#ifdef __CUDA_ARCH__
  return __ffsll((long long)m) - 1;
#else
  return __builtin_ctzll(m);
#endif
}
HD i64 eval_mask(const Tables& T, u64 mask, i64 x) {
  i64 best = 0;
  while (mask) {
    const int b = ffs64(mask);
    best = imax(best, tau_lc(T, b, x));
    mask &= T.lc_up[b];
  }
  return best;
}

HD const CrecHdr* crec_hdr(const Tables& T, int32_t off) { return (const CrecHdr*)(T.pool + off); }
HD const StageRec* crec_stages(const Tables& T, int32_t off) { return (const StageRec*)(T.pool + off + HDR_WORDS); }
HD const i64* crec_sub(const Tables& T, int32_t off, int P, int u) {
  return T.pool + off + HDR_WORDS + 16 * P + (i64)u * (P + 1);  // (k_u, c[0..P-2], c_wrap)
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
// template of candidate i: max{tau : prefix[tau] <= i}; the coarse bucket
// table narrows the binary search to the templates of one bucket
// template of chunk g (chunks of 32 candidates never straddle templates)
HD i64 find_template_of_chunk(const Tables& T, i64 g) {
  const i64 b = g >> T.cbucket_shift;
  i64 lo = T.tpl_cbucket[b], hi = (i64)T.tpl_cbucket[b + 1] + 1;
  if (hi > T.n_tpl) hi = T.n_tpl;
  while (hi - lo > 1) {
    const i64 mid = (lo + hi) >> 1;
    if (T.tpl_cprefix[mid] <= g) lo = mid; else hi = mid;
  }
  return lo;
}
HD i64 find_template(const Tables& T, i64 i) {
  const i64 b = i >> T.bucket_shift;
  i64 lo = T.tpl_bucket[b], hi = (i64)T.tpl_bucket[b + 1] + 1;
  if (hi > T.n_tpl) hi = T.n_tpl;
  while (hi - lo > 1) {
    const i64 mid = (lo + hi) >> 1;
    if (T.tpl_prefix[mid] <= i) lo = mid; else hi = mid;
  }
  return lo;
}

// floor(n / d) and n mod d for 0 <= n < 2^63, 0 < d, quotient < 2^40: on the
// device an fp64 estimate (relative error < 2^-51, so within 1 of the true
// quotient) fixed up with one exact int64 remainder -- no 64-bit division
// subroutine; on the host the plain operators.  Exact either way.
HD void divmod_est(i64 n, i64 d, i64& q, i64& r) {
#ifdef __CUDA_ARCH__
  // 1/d from the hardware approximation (~2^-20) and two explicit Newton
  // steps (error ~1 ulp; explicit fma, no contraction), so n * (1/d) is
  // within 2^-11 of n / d for quotients < 2^40: the floor is off by at most
  // one and the exact int64 remainder below fixes it
  const double dd = (double)d;
  double rc;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rc) : "d"(dd));
  double e = fma(-dd, rc, 1.0);
  rc = fma(rc, e, rc);
  e = fma(-dd, rc, 1.0);
  rc = fma(rc, e, rc);
  q = (i64)floor((double)n * rc);
  r = n - q * d;
  if (r < 0) { q -= 1; r += d; }
  if (r >= d) { q += 1; r -= d; }
#else
  q = n / d;
  r = n % d;
#endif
}

// Decoded + partitioned candidate, per class (steps a0 + a1), without
// per-stage arrays: layer counts are re-derived from the class's digit block.
// Replica k of the class gets m_k = q + [k < seats] + add + [k < rm]
// (rm = 0 except for the last class), non-increasing in k.
struct ClassSplit {
  u32 dig;     // boundary digits of this class (LSB = boundary 0)
  i64 q;       // Hamilton floor per replica
  i64 seats;   // replicas 0..seats-1 get +1 (largest remainders)
  i64 add;     // epsilon (c < C-1) or floor(R / D_last) (last class)
  i64 rm;      // last class: replicas < rm get +1
};
HD i64 mb_of(const ClassSplit& cs, i64 k) { return cs.q + (k < cs.seats ? 1 : 0) + cs.add + (k < cs.rm ? 1 : 0); }

// Sequential walk over one class's stages: l_s = l0_s + delta_s - delta_{s-1}
// with delta_s = digit_s - r (DESIGN.md C.2/C.4).
struct LayerWalk {
  u32 dig;
  int nd, dprev, s;
  u32 bl;
  int r;
  FastDiv dv;
  HD int next(const StageRec* st) {
    int d = 0;
    if (s < nd) {
      const u32 qd = dv.div(dig);
      d = (int)(dig - qd * bl) - r;
      dig = qd;
    }
    int l = st[s].l0 + d - dprev;
    dprev = d;
    ++s;
    return l;
  }
};
HD LayerWalk walk(const Tables& T, const CrecHdr* h, u32 dig) {
  return LayerWalk{dig, h->nd, 0, 0, (u32)(2 * T.r_layer + 1), T.r_layer, T.ldiv};
}

// Digits are least-significant first: class 0's boundaries, class 1's, ...,
// then the batch digits of classes 0..C-2.  Layer split = template base split
// + deltas; batch split = Hamilton over all replicas with weights
// floor(2^40 / slowest stage) (C.4).  Returns 0, -1 (layer) or -2 (batch).
// ILV: the V.2 rules (T.interleave > 1) are compiled in (K_split<true>).
template <int C, bool ILV = false>
HD int partition_c(const Tables& T, const TplRec& tp, i64 local, ClassSplit (&cs)[C]) {
  const u32 bb = (u32)(2 * T.r_batch + 1);
  u32 loc = (u32)local;  // radix < 2^31 (validated at create)
  i64 w[C], D[C];
  int status = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) {
    const CrecHdr* h = crec_hdr(T, tp.crec[c]);
    const StageRec* st = crec_stages(T, tp.crec[c]);
    D[c] = h->D;
    const u32 lq = h->pwdiv.div(loc);
    cs[c].dig = loc - lq * h->pw;
    loc = lq;
    const int lmin = ILV && h->P >= 2 ? T.interleave : 1;  // V.2: every chunk holds a layer
#ifdef __CUDA_ARCH__
    if (T.wtab && h->woff >= 0) {  // precomputed per (class, digits)
      const i64 e = __ldg(&T.wtab[h->woff + cs[c].dig]);
      if ((int)(e >> 48) < lmin) status = -1;
      w[c] = e & (((i64)1 << 48) - 1);
      continue;
    }
#endif
    LayerWalk lw = walk(T, h, cs[c].dig);
    i64 worst = 0;
    for (int s = 0; s < h->P; ++s) {
      const int l = lw.next(st);
      if (l < lmin) status = -1;
      worst = imax(worst, (i64)l * st[s].tcomp + st[s].wext);
    }
    i64 wr;
    divmod_est((i64)1 << 40, worst, w[c], wr);
  }
  if (status) return status;
  i64 W = 0, R = 0, left = tp.M, rem[C];
#pragma unroll
  for (int c = 0; c < C; ++c) W += D[c] * w[c];
#pragma unroll
  for (int c = 0; c < C; ++c) {
    divmod_est((i64)tp.M * w[c], W, cs[c].q, rem[c]);
    left -= D[c] * cs[c].q;
    cs[c].seats = 0;
    cs[c].rm = 0;
    if (c < C - 1) {
      const u32 lq = T.bdiv.div(loc);
      cs[c].add = (i64)(loc - lq * bb) - T.r_batch;
      loc = lq;
      R -= D[c] * cs[c].add;
    }
  }
  // leftover seats (left < sum D) to the largest remainders; ties -> lower
  // (class-major) replica index: rank of class c = #classes ahead of it
#pragma unroll
  for (int c = 0; c < C; ++c) {
    i64 before = 0;
#pragma unroll
    for (int o = 0; o < C; ++o)
      if (o != c && (rem[o] > rem[c] || (rem[o] == rem[c] && o < c))) before += D[o];
    cs[c].seats = imax(0, imin(D[c], left - before));
  }
  const i64 Dl = D[C - 1];
  // |R| <= sum_c D_c r_batch and D_l are small: 32-bit floor division
  const int32_t R32 = (int32_t)R, D32 = (int32_t)Dl;
#ifdef __CUDA_ARCH__
  // floor(R / D): fp32 estimate (|R| < 2^24, off by at most one) + exact fix-up
  int32_t f32 = (int32_t)floorf(__fdividef((float)R32, (float)D32));
  const int32_t rr = R32 - f32 * D32;
  if (rr < 0) f32 -= 1;
  else if (rr >= D32) f32 += 1;
  const i64 fl = f32;
#else
  const i64 fl = R32 >= 0 ? R32 / D32 : -((-R32 + D32 - 1) / D32);
#endif
  cs[C - 1].add = fl;
  cs[C - 1].rm = R - fl * Dl;
#pragma unroll
  for (int c = 0; c < C; ++c)
    if (mb_of(cs[c], D[c] - 1) < 1) return -2;  // m non-increasing in k
  if (ILV) {
    // V.2: every replica's m must be a multiple of its depth; the distinct m
    // of a class occur at k = 0, D-1 and next to the seats / rm thresholds
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const i64 P = crec_hdr(T, tp.crec[c])->P;
      if (P < 2) continue;
      const i64 ks[6] = {0, D[c] - 1, cs[c].seats - 1, cs[c].seats, cs[c].rm - 1, cs[c].rm};
      for (int q = 0; q < 6; ++q)
        if (ks[q] >= 0 && ks[q] < D[c] && mb_of(cs[c], ks[q]) % P) return -2;
    }
  }
  if (T.mem_check) {
    // DESIGN.md M.1: every device of every stage fits; replica 0 has the most
    // micro-batches (m non-increasing in k) and need is non-decreasing in m
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const CrecHdr* h = crec_hdr(T, tp.crec[c]);
      const StageRec* st = crec_stages(T, tp.crec[c]);
      const i64 m0 = mb_of(cs[c], 0);
      LayerWalk lw = walk(T, h, cs[c].dig);
      for (int s = 0; s < h->P; ++s) {
        const i64 l = lw.next(st);
        const int lg = st[s].lg_tp;
        const i64 act = ((i64)tp.b * T.mem_K[lg] + st[s].tp - 1) >> lg;
        const i64 fl = imin((i64)(h->P - s), m0);
        i64 need = l * T.mem_layer[lg] + fl * l * act;
        if (s == 0) need += T.mem_emb[lg];
        if (s == h->P - 1) need += T.mem_head[lg];
        if (need > T.mem_cap[st[s].type]) return -3;
      }
    }
  }
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

// compile-time depth: every array is register-resident.  Clocks are kept in
// offset coordinates X_s = end_s - o_s with o_s = c_0 + ... + c_{s-1}: then
// the F message of stage s-1 arrives at X_{s-1} (no add), the B message of
// stage s+1 at X_{s+1} + 2 c_s, stage 0's F input (time 0) and the last
// stage's B input (its own F) never exceed the stage clock, and
// T_pipe = end(B(0, m-1)) = X_0.  Every input is the neighbour's clock as of
// the previous level (its most recent op is the one consumed, C.7), so a
// level is computed from the previous level's clocks.
// m >= P: warm-up levels [0, 2P-1) and cool-down levels [2m, 2m+2P-2) have a
// fixed op pattern (unrolled, no bookkeeping); the steady levels [2P-1, 2m)
// alternate F (s = level mod 2) / B.  m < P: closed-form levels at run time.
// Lane compaction: a register-resident lane whose pipeline has
// not settled after the first block re-queues its (slot, sub-class, class) to
// a dense list of its depth and moves on; K_pipe_cont<P> re-runs those jobs 32
// per warp, so a warp's easy jobs no longer wait for its one hard job.
#ifndef HSIM_DEFER_MIN
#define HSIM_DEFER_MIN 16  // re-queue only with at least this many steady pairs left
#endif
struct DeferCtx {
  i64* list;                   // items slot << 16 | u << 4 | class
  unsigned long long* counter;
  i64 cap;
  i64 item;                    // slot << 16 | class (the sub-class is or'ed in)
};

template <int P>
struct Pipe {
  // Times are exact integers held in doubles (all < 2^52, checked at create):
  // the max-plus cell then runs on the fp64 pipe (DSETP + DADD) with the
  // selects on the ALU pipe, about half the ALU-pipe work of int64 max/add.
  double f[P], g[P], c[P], X[P];  // c[s] = 2 * (p2p cost of boundary s -> s+1)

  // op of stage s at level lv: +1 F, -1 B, 0 none
  HD static int op_at(i64 lv, int s, i64 m) {
    const i64 js = lv - s, jb = lv - (2 * P - 1 - s);
    if ((js >= 0 && lv <= P - 1 && js < m) || (lv >= 2 * P - s && !(js & 1) && (js >> 1) < m)) return 1;
    if (jb >= 0 && !(jb & 1) && (jb >> 1) < m) return -1;
    return 0;
  }
  HD static double dmax(double a, double b) { return a > b ? a : b; }
  HD double fop(const double (&old)[P], int s) const {
    return s == 0 ? old[0] + f[0] : dmax(old[s], old[s == 0 ? 0 : s - 1]) + f[s];
  }
  HD double bop(const double (&old)[P], int s) const {
    return s == P - 1 ? old[s] + g[s] : dmax(old[s], old[s == P - 1 ? s : s + 1] + c[s]) + g[s];
  }
  HD void level_rt(i64 lv, i64 m) {  // run-time ops
    double old[P];
#pragma unroll
    for (int s = 0; s < P; ++s) old[s] = X[s];
#pragma unroll
    for (int s = 0; s < P; ++s) {
      const int o = op_at(lv, s, m);
      if (o > 0) X[s] = fop(old, s);
      else if (o < 0) X[s] = bop(old, s);
    }
  }
  // m >= P: ops of warm-up level lv (compile-time after unrolling)
  HD void level_warm(int lv) {
    double old[P];
#pragma unroll
    for (int s = 0; s < P; ++s) old[s] = X[s];
#pragma unroll
    for (int s = 0; s < P; ++s) {
      const int js = lv - s, jb = lv - (2 * P - 1 - s);
      if ((js >= 0 && lv <= P - 1) || (lv >= 2 * P - s && !(js & 1))) X[s] = fop(old, s);
      else if (jb >= 0 && !(jb & 1)) X[s] = bop(old, s);
    }
  }
  // m >= P: ops of cool-down level 2m + d
  HD void level_cool(int d) {
    double old[P];
#pragma unroll
    for (int s = 0; s < P; ++s) old[s] = X[s];
#pragma unroll
    for (int s = 0; s < P; ++s) {
      if (d < s && !((d - s) & 1)) X[s] = fop(old, s);
      else if (d < 2 * P - 1 - s && !((d + 1 + s) & 1)) X[s] = bop(old, s);
    }
  }
  // one steady level of parity par: stages with s % 2 == par run F, the others B
  template <int par>
  HD void steady_level() {
    double old[P];
#pragma unroll
    for (int s = 0; s < P; ++s) old[s] = X[s];
#pragma unroll
    for (int s = 0; s < P; ++s) X[s] = (s & 1) == par ? fop(old, s) : bop(old, s);
  }
  HD void steady_pair() {
    steady_level<1>();
    steady_level<0>();
  }
  // --- exact acceleration of the steady regime ------------------------------
  // Levels [2P-1, 2m) form (odd, even) pairs, each the same max-plus map A with
  // per-stage constants, so X(k+1) = A(X(k)) and A(x + d) = A(x) + d.
  //
  // Affine regime (AFF): with d = X(k) - X(k-1), evaluate the next pair on
  // (value, slope d) operands.  Every max keeps the operand that wins now
  // (ties: the one growing faster); the pair is then the fixed selection
  // X' = Pi X + w for as long as no losing operand that grows faster has
  // caught up -- H pairs (a safe lower bound, see sym_cell).  If that pair
  // moves X by exactly d and Pi d = d (slopes reproduce), then
  // X(k + t) = X(k) + t d for t <= H: a transient in which different stages
  // advance at different rates (balanced stages of unequal speed) is crossed
  // in one multiply-add per stage, exactly (integers < 2^52 in fp64).  A
  // uniform d is the periodic regime of cyclicity 1 (H infinite).
  // Cyclic regime (WHOLE): X moved by the same d over a whole block of BL
  // pairs -> cyclicity c | BL: X(k + q BL) = X(k) + q d.
  HD static void sym_cell(double a, double sa, double b, double sb, double dur, double& x, double& sl, double& H) {
    const bool bw = b > a || (b == a && sb > sa);
    const double w = bw ? b : a, sw = bw ? sb : sa, l = bw ? a : b, sL = bw ? sa : sb;
    // the loser overtakes after (w - l) / (sL - sw) pairs: RN quotient of exact
    // integers < 2^52 is within 1 of the true one, so floor - 1 is safe
    if (sL > sw) H = fmin(H, floor((w - l) / (sL - sw)) - 1.0);
    x = w + dur;
    sl = sw;
  }
  template <int par>
  HD void sym_level(double (&x)[P], double (&sl)[P], double& H) const {
    double ox[P], os[P];
#pragma unroll
    for (int s = 0; s < P; ++s) { ox[s] = x[s]; os[s] = sl[s]; }
#pragma unroll
    for (int s = 0; s < P; ++s) {
      if ((s & 1) == par) {  // F
        if (s == 0) { x[0] = ox[0] + f[0]; sl[0] = os[0]; }
        else sym_cell(ox[s], os[s], ox[s == 0 ? 0 : s - 1], os[s == 0 ? 0 : s - 1], f[s], x[s], sl[s], H);
      } else {               // B
        if (s == P - 1) { x[s] = ox[s] + g[s]; sl[s] = os[s]; }
        else sym_cell(ox[s], os[s], ox[s == P - 1 ? s : s + 1] + c[s], os[s == P - 1 ? s : s + 1], g[s], x[s], sl[s], H);
      }
    }
  }
  // horizon H >= 1 of the affine regime with increments d, or < 1 if none
  HD double affine_horizon(const double (&d)[P]) const {
    double x[P], sl[P], H = 1e300;
#pragma unroll
    for (int s = 0; s < P; ++s) { x[s] = X[s]; sl[s] = d[s]; }
    sym_level<1>(x, sl, H);
    sym_level<0>(x, sl, H);
    bool ok = true;
#pragma unroll
    for (int s = 0; s < P; ++s) ok = ok && x[s] - X[s] == d[s] && sl[s] == d[s];
    return ok ? H : 0.0;
  }
  // One block of BL steady pairs, then the checks above.  Returns true when
  // the remaining steady pairs are settled (the caller runs the leftovers).
  template <int BL, bool WHOLE, bool AFF>
  HD bool block(int& k, int kn, i64& skipped) {
    double o0[P], o1[P];
#pragma unroll
    for (int s = 0; s < P; ++s) o0[s] = X[s];
#pragma unroll 1
    for (int b = 0; b < BL - 1; ++b) steady_pair();
#pragma unroll
    for (int s = 0; s < P; ++s) o1[s] = X[s];
    steady_pair();
    k += BL;
#ifndef HSIM_NOSKIP
    if (AFF) {
      double d[P];
#pragma unroll
      for (int s = 0; s < P; ++s) d[s] = X[s] - o1[s];
      const double H = affine_horizon(d);
      if (H >= 1.0) {
        const int t = (int)fmin(H, (double)(kn - k));
#pragma unroll
        for (int s = 0; s < P; ++s) X[s] += (double)t * d[s];
        skipped += t;
        k += t;
        return k == kn;
      }
    } else {
      const double d = X[0] - o1[0];
      bool per = true;
#pragma unroll
      for (int s = 1; s < P; ++s) per = per && (X[s] - o1[s] == d);
      if (per) {
        const int r = kn - k;
        const double rd = (double)r * d;
#pragma unroll
        for (int s = 0; s < P; ++s) X[s] += rd;
        skipped += r;
        k = kn;
        return true;
      }
    }
    if (WHOLE) {
      const double d = X[0] - o0[0];
      bool per = true;
#pragma unroll
      for (int s = 1; s < P; ++s) per = per && (X[s] - o0[s] == d);
      if (per) {
        const int q = (kn - k) / BL;
        const double qd = (double)q * d;
#pragma unroll
        for (int s = 0; s < P; ++s) X[s] += qd;
        skipped += (i64)q * BL;
        k += q * BL;
        return true;
      }
    }
#endif
    return false;
  }
  // T_pipe; `skipped` = steady level pairs not executed (periodic regime).
  // T_pipe; with dc (device): -1 if the job was re-queued for K_pipe_cont
  HD i64 run(i64 m, i64& skipped, const DeferCtx* dc = nullptr, int u = 0) {
#pragma unroll
    for (int s = 0; s < P; ++s) X[s] = 0;
    skipped = 0;
    if (m >= P) {
      // warm-up levels [0, 2P-1): unrolled (compile-time op pattern) for
      // shallow pipelines; deeper ones loop over levels with run-time ops so the
      // kernel's straight-line code stays within the instruction cache
      if (P <= HSIM_UNROLL_MAXP) {
#pragma unroll
        for (int lv = 0; lv < 2 * P - 1; ++lv) level_warm(lv);
      } else {
#pragma unroll 1
        for (int lv = 0; lv < 2 * P - 1; ++lv) level_rt(lv, m);
      }
      // steady pairs: a first block of 4, then blocks of 12 (P <= HSIM_WHOLE_MAXP)
      // or 4; after each, the affine check (P <= HSIM_AFFINE_MAXP; else only
      // the uniform-increment case) and, for P <= HSIM_WHOLE_MAXP, the cyclic
      // c | BL check (deeper pipelines: the snapshot would not fit the registers)
      constexpr bool EXT = P <= HSIM_WHOLE_MAXP, AFF = P <= HSIM_AFFINE_MAXP;
      constexpr int BLK = EXT ? 12 : 4;
      const int kn = (int)(m - P);
      int k = 0;
      // with the cyclic check (P >= 5), block lengths cycle 24, 28, 20 so that
      // c | 24 (c = 8: two runs of eight identical stages), c | 28 (c = 7:
      // seven identical consecutive stages) and c | 20 (c = 5) are all caught
      // within about one cycle after the transient
      if (kn >= 4 && !block<4, EXT, AFF>(k, kn, skipped)) {
#ifdef __CUDA_ARCH__
        if (dc && kn - k >= HSIM_DEFER_MIN) {
          const unsigned long long q = atomicAdd(dc->counter, 1ull);
          if ((i64)q < dc->cap) {
            dc->list[q] = dc->item | (i64)u << 4;
            skipped = kn - k;  // executed here: warm-up + the first block
            return -1;
          }
        }
#endif
        if (EXT && P >= 5) {
          for (;;) {
            if (k + 24 > kn || block<24, EXT, AFF>(k, kn, skipped)) break;
            if (k + 28 > kn || block<28, EXT, AFF>(k, kn, skipped)) break;
            if (k + 20 > kn || block<20, EXT, AFF>(k, kn, skipped)) break;
          }
        } else {
          while (k + BLK <= kn && !block<BLK, EXT, AFF>(k, kn, skipped)) {
          }
        }
      }
      for (; k < kn; ++k) steady_pair();
      steady_level<1>();  // level 2m-1
      if (P <= HSIM_UNROLL_MAXP) {
#pragma unroll
        for (int d = 0; d < 2 * P - 2; ++d) level_cool(d);
      } else {
#pragma unroll 1
        for (int d = 0; d < 2 * P - 2; ++d) level_rt(2 * m + d, m);
      }
    } else {
      const i64 total = 2 * (m + P - 1);
      for (i64 lv = 0; lv < total; ++lv) level_rt(lv, m);
    }
    return (i64)X[0];
  }
};

#ifdef HSIM_DIAG
__device__ unsigned long long g_diag[17][16];
#endif
// T_pipe of every sub-class of a class (compile-time depth), max-reduced.
struct PipeOut { i64 T0, cells; };

// R (S.1, overlap mode only; else nullptr): R[s * rs] = max over sub-classes
// of the end of stage s's last op (its last backward) in real time
// dc (device): re-queue context or nullptr (a re-queued sub-class contributes
// 0 here; K_pipe_cont<P> max's its exact T_pipe and stage ends in).
// only_u >= 0: evaluate that sub-class alone (K_pipe_cont).
template <int P>
HD PipeOut class_pipes_inl(const Tables& T, int32_t off, const ClassSplit& cs, i64* R = nullptr, i64 rs = 0,
                           const DeferCtx* dc = nullptr, int only_u = -1) {
  const CrecHdr* h = crec_hdr(T, off);
  const StageRec* st = crec_stages(T, off);
  Pipe<P> p;
  LayerWalk lw = walk(T, h, cs.dig);
#pragma unroll
  for (int s = 0; s < P; ++s) {
    const i64 l = lw.next(st);
    p.f[s] = (double)(l * st[s].layer_f + st[s].fext);
    p.g[s] = (double)(l * st[s].layer_b + st[s].gext);
  }
  PipeOut r{0, 0};
  const int u0 = only_u >= 0 ? only_u : 0, u1 = only_u >= 0 ? only_u + 1 : h->U;
  for (int u = u0; u < u1; ++u) {
    const i64* sub = crec_sub(T, off, P, u);
#pragma unroll
    for (int s = 0; s + 1 < P; ++s) p.c[s] = (double)(2 * sub[1 + s]);
    const i64 m = mb_of(cs, sub[0]);
    i64 sk;
    const i64 tp = p.run(m, sk, dc, u);
    r.T0 = imax(r.T0, tp);
    // cells executed; a re-queued job is counted once, by its complete run in
    // K_pipe_cont (the cells of the abandoned first attempt are not counted)
    r.cells += tp < 0 ? 0 : 2 * P * (m - sk);
    if (R) {  // offset coordinates -> real ends: end_s = X_s + c_0 + ... + c_{s-1}
      double o = 0;
#pragma unroll
      for (int s = 0; s < P; ++s) {
        const i64 e = tp < 0 ? 0 : (i64)(p.X[s] + o);
#ifdef __CUDA_ARCH__
        if (only_u >= 0) atomicMax((unsigned long long*)&R[s * rs], (unsigned long long)e);
        else
#endif
          R[s * rs] = u == 0 ? e : imax(R[s * rs], e);
        if (s + 1 < P) o += 0.5 * p.c[s];
      }
    }
#if defined(HSIM_DIAG) && defined(__CUDA_ARCH__)
    {  // histogram of executed steady pairs in units of P; bucket 7 = not detected
      const i64 kn = m >= P ? m - P : 0, ex = kn - sk;
      const int bk = sk > 0 ? (int)imin(ex / P, 6) : 7;
      atomicAdd(&g_diag[P][bk], 1ull);
      atomicAdd(&g_diag[P][8], (unsigned long long)ex);
      atomicAdd(&g_diag[P][9], (unsigned long long)kn);
    }
#endif
  }
  return r;
}

// --- step a5: gradient sync (C.6, C.8) -----------------------------------------
// RS_j + AR_j of the segment [a, z) whose layers sit in stage sc[c] of every
// class c: reshard (A14) over the TP rings of groups with tp != t*, then the
// DP ring all-reduce over all replicas (class asc, replica asc, wrap), rings
// through device base + q, q < t*.
template <int C>
HD i64 seg_cost_c(const Tables& T, const TplRec& tp, const StageRec* const (&st)[C], const int (&sc)[C], i64 a, i64 z) {
  // V.3 (tp.flags bit 0): the expert weights are sharded over the replicas, so
  // only the dense parameters are all-reduced
  const i64 lb = (tp.flags & 1) ? T.seg_layer_dense : T.seg_layer_bytes;
  const i64 S = (z - a) * lb + (a == 0 ? T.seg_first_bytes : 0) + (z == T.L ? T.seg_last_bytes : 0);
  int tstar = 1 << 30, lg = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) {
    const int tpc = st[c][sc[c]].tp;
    if (tpc < tstar) { tstar = tpc; lg = st[c][sc[c]].lg_tp; }
  }
  const i64 xs = (S + tstar - 1) >> lg;  // t* is a power of two
  u64 rsmask = 0, mask = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) {
    const StageRec& s = st[c][sc[c]];
    if (s.tp != tstar) rsmask |= s.tp_mask;  // reshard over this group's TP ring (A14)
    mask |= s.dp_mask[lg];
    if (tp.flags & 2) continue;  // V.1: single class, the wrap edge is in dp_mask
    // edge from the last replica of class c to the first replica of the next
    // class (wrap: class C-1 -> class 0), ring q through device base + q
    const StageRec& t = st[c + 1 < C ? c + 1 : 0][sc[c + 1 < C ? c + 1 : 0]];
    const int n1 = s.last_node, n2 = t.first_node;
    const int t1 = s.type, t2 = t.type;  // a node's type is its devices' type (C.1)
    mask |= n1 == n2 ? T.xmask_same[((t1 * MAXG + s.last_base) * MAXG + t.first_base) * 4 + lg]
                     : T.xmask_cross[(((t1 * MAXG + s.last_base) * MAXT + t2) * MAXG + t.first_base) * 4 + lg];
  }
  const i64 RS = rsmask ? eval_mask(T, rsmask, xs) : 0;
  const i64 AR = 2 * (i64)(tp.D - 1) * eval_mask(T, mask, ceil_div_rcp(xs, tp.D, tp.rD));
  return RS + AR;
}

// C.8: segments = common refinement of the classes' layer boundaries, in
// ascending layer order, list-scheduled FIFO per (class, stage) group from T0:
// a segment starts when every group it uses is free (all classes take part).
// BK (DESIGN.md B.1, Tables.buckets = 2): each stage's l layers are also cut
// after its lower ceil(l/2) -- two buckets on the same group.
HD i64 lower_half(i64 l) { return (l + 1) >> 1; }
template <int C, bool BK = false>
HD i64 grad_sync_c(const Tables& T, const TplRec& tp, const ClassSplit (&cs)[C], i64 T0) {
  int sc[C], P[C];
  i64 nextcut[C], cur_free[C];
  i64 sa[C], ls[C];  // BK: start and layers of the current stage
  int bk[C];         // BK: 0 lower bucket, 1 upper
  LayerWalk lw[C];
  const StageRec* st[C];
#pragma unroll
  for (int c = 0; c < C; ++c) {
    const CrecHdr* h = crec_hdr(T, tp.crec[c]);
    P[c] = h->P;
    st[c] = crec_stages(T, tp.crec[c]);
    lw[c] = walk(T, h, cs[c].dig);
    sc[c] = 0;
    const i64 l0 = lw[c].next(st[c]);
    nextcut[c] = P[c] > 1 ? l0 : T.L;
    if constexpr (BK) {
      sa[c] = 0;
      ls[c] = P[c] > 1 ? l0 : T.L;
      bk[c] = 0;
      if (lower_half(ls[c]) < ls[c]) nextcut[c] = lower_half(ls[c]);
    }
    cur_free[c] = T0;
  }
  i64 a = 0, Titer = T0;
  while (a < T.L) {
    i64 z = T.L;
#pragma unroll
    for (int c = 0; c < C; ++c) z = imin(z, nextcut[c]);
    const i64 cost = seg_cost_c<C>(T, tp, st, sc, a, z);
    i64 start = 0;
#pragma unroll
    for (int c = 0; c < C; ++c) start = imax(start, cur_free[c]);
    const i64 end = start + cost;
    Titer = imax(Titer, end);
#pragma unroll
    for (int c = 0; c < C; ++c) {  // advance classes whose stage (or lower bucket) ends at z
      cur_free[c] = end;
      if (nextcut[c] == z && z < T.L) {
        if constexpr (BK) {
          if (bk[c] == 0 && lower_half(ls[c]) < ls[c]) {  // into the upper bucket: same group
            bk[c] = 1;
            nextcut[c] = sa[c] + ls[c];
            continue;
          }
        }
        sc[c]++;
        const i64 l = lw[c].next(st[c]);
        nextcut[c] = sc[c] + 1 < P[c] ? nextcut[c] + l : T.L;
        if constexpr (BK) {
          sa[c] = z;
          ls[c] = nextcut[c] - z;
          bk[c] = 0;
          if (lower_half(ls[c]) < ls[c]) nextcut[c] = z + lower_half(ls[c]);
        }
        cur_free[c] = T0;
      }
    }
    a = z;
  }
  return Titer;
}

// S.1: no barrier.  Segment j is ready when every group
// holding its layers has ended its last backward -- R[coff_c + s] = max over
// the class's replicas of that stage's end (written by the 1F1B kernels,
// row stride rs) -- and segments are issued in descending layer order (the
// order backward produces gradients), FIFO per group: a class entering a new
// stage meets a group that has not synchronised yet.  BK (B.1): a stage's
// upper bucket (its top l - ceil(l/2) layers, + the head) is ready earlier by
// the lower bucket's share of the last backward, ceil(l/2) x layer_b (+ the
// embedding on stage 0).
template <int C, bool BK = false>
HD i64 grad_sync_overlap_c(const Tables& T, const TplRec& tp, const ClassSplit (&cs)[C], const i64* R, i64 rs,
                           i64 T0) {
  int sc[C], coff[C], bk[C];
  int16_t start[C][MAXP + 1];
  i64 cur_free[C];
  const StageRec* st[C];
  int off = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) {
    const CrecHdr* h = crec_hdr(T, tp.crec[c]);
    st[c] = crec_stages(T, tp.crec[c]);
    LayerWalk lw = walk(T, h, cs[c].dig);
    int a = 0;
    for (int s = 0; s < h->P; ++s) {
      start[c][s] = (int16_t)a;
      a += lw.next(st[c]);
    }
    start[c][h->P] = (int16_t)T.L;
    sc[c] = h->P - 1;
    coff[c] = off;
    off += h->P;
    cur_free[c] = 0;
    bk[c] = 0;
    if constexpr (BK) {
      const i64 l = start[c][sc[c] + 1] - start[c][sc[c]];
      bk[c] = lower_half(l) < l ? 1 : 0;
    }
  }
  i64 z = T.L, Titer = T0;
  while (z > 0) {
    i64 a = 0, ready = 0, begin = 0;
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const int s = sc[c];
      i64 lo = start[c][s], rd = R[(i64)(coff[c] + s) * rs];
      if constexpr (BK) {
        if (bk[c]) {
          const i64 l = start[c][s + 1] - start[c][s];
          lo += lower_half(l);
          rd -= lower_half(l) * st[c][s].layer_b + (s == 0 ? st[c][s].emb_b : 0);
        }
      }
      a = imax(a, lo);
      ready = imax(ready, rd);
      begin = imax(begin, cur_free[c]);
    }
    const i64 end = imax(begin, ready) + seg_cost_c<C>(T, tp, st, sc, a, z);
    Titer = imax(Titer, end);
#pragma unroll
    for (int c = 0; c < C; ++c) {
      cur_free[c] = end;
      if constexpr (BK) {
        if (bk[c]) {
          const i64 l = start[c][sc[c] + 1] - start[c][sc[c]];
          if (start[c][sc[c]] + lower_half(l) == a) bk[c] = 0;  // down into the lower bucket: same group
          continue;
        }
      }
      if (a > 0 && start[c][sc[c]] == a) {
        sc[c]--;
        cur_free[c] = 0;
        if constexpr (BK) {
          const i64 l = start[c][sc[c] + 1] - start[c][sc[c]];
          bk[c] = lower_half(l) < l ? 1 : 0;
        }
      }
    }
    z = a;
  }
  return Titer;
}

// V.2 (interleaved 1F1B): stage s of a class holds v layer ranges (virtual
// stage k P + s = chunk k of stage s, chunk k of l layers = l / v + [k < l mod
// v]), so a (class, stage) group is revisited by later segments: the group
// clocks are explicit.  C.8 (R == nullptr): segments in ascending layer order
// from T0; S.1: descending, each ready when its groups' last backward ended
// (R[(coff_c + s) * rs]).  FIFO per group either way.
template <int C>
HD i64 grad_sync_ilv_c(const Tables& T, const TplRec& tp, const ClassSplit (&cs)[C], const i64* R, i64 rs, i64 T0) {
  const StageRec* st[C];
  int P[C], v[C], coff[C], x[C], sc[C];
  int16_t lay[C][MAXP];
  i64 fr[C][MAXP], lo[C], hi[C];
  const bool desc = R != nullptr;
  int off = 0;
  for (int c = 0; c < C; ++c) {
    const CrecHdr* h = crec_hdr(T, tp.crec[c]);
    st[c] = crec_stages(T, tp.crec[c]);
    P[c] = h->P;
    v[c] = h->P >= 2 ? T.interleave : 1;
    coff[c] = off;
    off += h->P;
    LayerWalk lw = walk(T, h, cs[c].dig);
    for (int q = 0; q < h->P; ++q) {
      lay[c][q] = (int16_t)lw.next(st[c]);
      fr[c][q] = desc ? 0 : T0;
    }
    x[c] = desc ? v[c] * P[c] - 1 : 0;
  }
  auto chunk = [&](int c, int xx) {  // layers of virtual stage xx of class c
    const int s = xx % P[c], k = xx / P[c], l = lay[c][s];
    return (i64)(l / v[c] + (k < l % v[c] ? 1 : 0));
  };
  for (int c = 0; c < C; ++c) {
    sc[c] = x[c] % P[c];
    if (desc) { hi[c] = T.L; lo[c] = T.L - chunk(c, x[c]); }
    else { lo[c] = 0; hi[c] = chunk(c, 0); }
  }
  // segment = [max lo, min hi): the common refinement at the cursors
  i64 Titer = T0;
  for (;;) {
    i64 sa = 0, sz = T.L, ready = 0, begin = 0;
    for (int c = 0; c < C; ++c) {
      sa = imax(sa, lo[c]);
      sz = imin(sz, hi[c]);
      begin = imax(begin, fr[c][sc[c]]);
      if (desc) ready = imax(ready, R[(i64)(coff[c] + sc[c]) * rs]);
    }
    const i64 end = imax(begin, ready) + seg_cost_c<C>(T, tp, st, sc, sa, sz);
    Titer = imax(Titer, end);
    for (int c = 0; c < C; ++c) fr[c][sc[c]] = end;
    if (desc ? sa == 0 : sz == T.L) break;
    for (int c = 0; c < C; ++c) {
      if (desc && lo[c] == sa) {
        --x[c];
        hi[c] = lo[c];
        lo[c] = hi[c] - chunk(c, x[c]);
      } else if (!desc && hi[c] == sz) {
        ++x[c];
        lo[c] = hi[c];
        hi[c] = lo[c] + chunk(c, x[c]);
      }
      sc[c] = x[c] % P[c];
    }
  }
  return Titer;
}

// host-side rendering of a candidate's split (hsim_decode)
template <bool ILV>
HD int partition_any_t(const Tables& T, const TplRec& tp, i64 local, ClassSplit* out) {
  int st = 0;
  switch (tp.C) {
    case 1: { ClassSplit cs[1]; st = partition_c<1, ILV>(T, tp, local, cs); for (int c = 0; c < 1; ++c) out[c] = cs[c]; break; }
    case 2: { ClassSplit cs[2]; st = partition_c<2, ILV>(T, tp, local, cs); for (int c = 0; c < 2; ++c) out[c] = cs[c]; break; }
    case 3: { ClassSplit cs[3]; st = partition_c<3, ILV>(T, tp, local, cs); for (int c = 0; c < 3; ++c) out[c] = cs[c]; break; }
    default: { ClassSplit cs[4]; st = partition_c<4, ILV>(T, tp, local, cs); for (int c = 0; c < 4; ++c) out[c] = cs[c]; break; }
  }
  return st;
}
HD int partition_any(const Tables& T, const TplRec& tp, i64 local, ClassSplit* out) {
  return T.interleave > 1 ? partition_any_t<true>(T, tp, local, out) : partition_any_t<false>(T, tp, local, out);
}

#ifdef __CUDACC__
// --- lane-per-stage 1F1B wavefront (deep pipelines), used by kernels.cu ---------
__device__ __forceinline__ i64 shfl64(i64 v, int src) { return __shfl_sync(0xffffffffu, v, src); }

__device__ __forceinline__ int nth_set_lane(unsigned mask, int n) {
  for (int q = 0; q < n; ++q) mask &= mask - 1;
  return __ffs(mask) - 1;
}

// Times as exact integers in doubles (< 2^52, checked at create): fp64 max/add.
__device__ __forceinline__ double shfl_d(double v, int src) { return __shfl_sync(0xffffffffu, v, src); }
__device__ __forceinline__ double dmax2(double a, double b) { return a > b ? a : b; }

struct LanePipe {
  int P, s, lane;
  i64 m;
  double f, g, cR, cL;  // cR = c_s (0 on the last stage), cL = c_{s-1}
  double X, out;
  // one level; every lane of the warp must call it (it shuffles).  In the
  // steady range the op is given by the parity constants, else by the
  // closed-form levels of F(s,j) / B(s,j).
  __device__ __forceinline__ void level(i64 lv, bool steady, int srcS, double durS, double cS, bool keepS) {
    int src = srcS;
    double dur = durS, cc = cS;
    bool keep = keepS, doOp = true;
    if (!steady) {
      const i64 js = lv - s, jb = lv - (2 * P - 1 - s);
      const bool isF = (js >= 0 && lv <= P - 1 && js < m) || (lv >= 2 * P - s && !(js & 1) && (js >> 1) < m);
      const bool isB = jb >= 0 && !(jb & 1) && (jb >> 1) < m;
      doOp = isF || isB;
      src = isF ? lane - 1 : lane + 1;
      dur = isF ? f : g;
      cc = isF ? cR : cL;
      keep = !((isF && s == 0) || (isB && s == P - 1));  // stage-0 input / B right after own F
    }
    const double v0 = shfl_d(out, src);
    const double v = keep ? v0 : 0.0;
    if (doOp) {
      const double e = dmax2(X, v) + dur;
      X = e;
      out = e + cc;
    }
  }
};

#endif

}  // namespace hsim
