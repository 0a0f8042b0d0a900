// oracle/oracle.cpp — TEST INFRASTRUCTURE ONLY.
//
// A plain, slow, CPU, event-driven implementation of what the hot path
// computes: for one candidate mapping (a linear index into the search space)
// it predicts one training-iteration time in int64 ns.  Only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
// may load it.  It shares no code, header, table or constant generator with
// the product (paper_2508_05370_b200/); its input structs are its own.
//
// It follows PAPER.md (arXiv 2508.05370) and the readings recorded in
// DESIGN.md §2 (the paper gives no cost formulas beyond the link delay; every
// other formula is a reading, listed there with its id A1..A24 / C.x).
//
// Variants (off by default): V.2 interleaved 1F1B
// (orc_input.interleave = v model chunks per stage, Megatron-LM's virtual
// pipeline) and V.3 expert parallelism across the DP replicas (ep_dp); both
// are stated where they act (op_order / run_pipelines, layer_chain,
// ep_alltoall_x, segments) and in DESIGN.md.
//
// Two modes (SURVEY.md §8(c) "It runs in two modes ... The two modes must agree"):
//  * literal (default): every replica of every class is simulated; every stage
//    is its own resource in a (time, seq)-ordered event queue;
//    stage durations are sums over their layers' op durations; every
//    collective (TP all-reduce, DP ring all-reduce) is simulated send by send
//    on its ring.  No closed forms, no sub-classing, no precomputed tables.
//  * compact: one pipeline per sub-class of isomorphic replicas (replicas of a
//    class with equal p2p cost vectors; m = the largest m among them, DESIGN
//    A13), stage durations as l_s x (one layer's op chain) + emb/head, and
//    every ring collective as steps x (slowest edge) (the closed form the
//    literal async ring reaches, pinned in tests/test_oracle_pins.py).  Same
//    event engine, same decode / placement / partition.  It exists so the
//    exhaustive parity runs on configs 3 and 5 fit in host-core minutes; the
//    literal == compact equivalence is tested (tests/test_oracle_compact.py).
//
// Exactness rules (DESIGN.md C.0): durations are ceil((double)x / r) with x an
// int64 < 2^53 and r a double; everything else is int64 + and max.  Built with
// -ffp-contract=off, no fast-math.
//
// Pins (tests/test_oracle_pins.py): Table 4 delays, ring all-reduce and 1F1B
// closed forms, DAG longest path, Hamilton / Fig 3 shares, Table 1 payload,
// parameter counts, brute-force tiny spaces, invariants; the memory-feasibility
// row (DESIGN M.1) in tests/test_memory_pins.py.  Absolute iteration
// times are "parity unpinned" (the paper prints none).

#include <algorithm>
#include <array>
#include <map>
#include <mutex>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <queue>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

typedef int64_t i64;

// ----------------------------------------------------------------------------
// Input structs (the oracle's own; built by oracle/oracle.py from the shared
// workload dicts in hsim_inputs/ — field copies only).
// ----------------------------------------------------------------------------
extern "C" {
struct orc_hop { double gbps; int32_t bidir; int32_t pad; };
struct orc_path { int32_t n; int32_t pad; orc_hop hop[4]; };
struct orc_type {
  double peak_flop_per_ns, hbm_bytes_per_ns;
  double eff_flop[5], eff_mem[5];
  i64 mem_bytes;
  int32_t gpus_per_node, n_link_kinds;
  orc_path link_kind[4];
  int32_t intra_kind[8][8];
  orc_path gpu_nic;
  double nic_gbps;
  i64 nic_delay_ns;
};
struct orc_input {
  int32_t n_types, n_nodes;
  const orc_type* types;
  const int32_t* node_type;
  i64 rail_alpha_ns;
  double rail_gbps;
  i64 frame_bytes;
  // model (Table 5 row + DESIGN A3 fields)
  i64 L, h, heads, kv_heads, ffn, nm, seq, V, tied, E, topk, bpe_act, bpe_grad, B;
  // search space (framework description as a space; DESIGN C.2)
  int32_t n_b, bset[8];
  int32_t n_tp[8], tpset[8][8];
  int32_t n_p, pset[16];
  int32_t homo, mixed, use_all, r_layer, pmax, r_batch;
  int32_t mem_check;  // prune candidates that do not fit (status -3, DESIGN M.1)
  int32_t sync_overlap;  // gradient sync overlapped with the backward (DESIGN S.1)
  int32_t interleave;    // v model chunks per stage, interleaved 1F1B (DESIGN V.2); 1 = off
  int32_t ep_dp;         // expert parallelism across the DP replicas (DESIGN V.3)
  int32_t mixtp;         // mixed-type TP groups, the MIXTP family (DESIGN V.1)
  int32_t sync_buckets;  // 2 = two gradient buckets per stage group (DESIGN B.1); 0/1 = one
};
}

namespace {

enum { ATTN = 0, MLP = 1, MOE = 2, EMB = 3, HEAD = 4 };

// --- C.0 exactness ----------------------------------------------------------
i64 ceilq(i64 x, double r) {  // one IEEE RN division, then ceil
  if (x == 0) return 0;
  return (i64)std::ceil((double)x / r);
}
i64 ceil_div(i64 a, i64 b) { return (a + b - 1) / b; }

// --- links: PAPER.md:394-396 (delay = jumbo*8 / uni-dir Gbps), Table 4 ------
struct Link { i64 alpha; double beta; };  // alpha ns, beta B/ns

double uni_gbps(const orc_hop& hp) { return hp.bidir ? hp.gbps / 2.0 : hp.gbps; }

// A path of hops: alpha = sum of per-hop delays (each ceil'd, A9), beta = the
// slowest hop (uni Gbps / 8 = B/ns).
Link path_link(const orc_path& p, i64 frame) {
  Link l{0, 1e300};
  for (int k = 0; k < p.n; ++k) {
    double u = uni_gbps(p.hop[k]);
    l.alpha += ceilq(frame * 8, u);
    l.beta = std::min(l.beta, u / 8.0);
  }
  return l;
}
Link join(Link a, Link b) { return Link{a.alpha + b.alpha, std::min(a.beta, b.beta)}; }
i64 tau(const Link& e, i64 x) { return e.alpha + ceilq(x, e.beta); }

struct Cluster {
  const orc_input* in;
  std::vector<int> gpn;            // gpus per node, per node
  std::vector<int> ntype;          // device type per node
  std::vector<i64> n_of_type;      // total GPUs per type
  std::vector<std::vector<int>> nodes_of_type;

  const orc_type& T(int node) const { return in->types[ntype[node]]; }

  // Fig 2 cases (a)(b)(c); DESIGN A10-A12.
  Link gpu_to_gpu(int n1, int r1, int n2, int r2) const {
    const i64 fr = in->frame_bytes;
    if (n1 == n2) {
      const orc_type& t = T(n1);
      return path_link(t.link_kind[t.intra_kind[r1][r2]], fr);
    }
    // rail path GPU -> PCIe -> NIC -> rail switch -> NIC -> PCIe -> GPU
    const orc_type& a = T(n1);
    const orc_type& b = T(n2);
    Link rail = path_link(a.gpu_nic, fr);
    rail = join(rail, Link{a.nic_delay_ns, a.nic_gbps / 8.0});
    rail = join(rail, Link{in->rail_alpha_ns, in->rail_gbps / 8.0});
    rail = join(rail, Link{b.nic_delay_ns, b.nic_gbps / 8.0});
    rail = join(rail, path_link(b.gpu_nic, fr));
    if (r1 == r2) return rail;                                          // case (b)
    return join(path_link(a.link_kind[a.intra_kind[r1][r2]], fr), rail);  // case (c)
  }
};

// --- C.5: per-device FLOPs and bytes of one layer op -------------------------
struct Cost { i64 flop, bytes; };
// g = the devices the experts are sharded over (MOE weight bytes; 0 = t, the
// TP group, A17); DESIGN V.3 shards them over every replica's group (g = D t)
Cost op_cost(const orc_input& m, int kind, i64 t, i64 b, i64 g = 0) {
  const i64 T = b * m.seq, h = m.h, bpe = m.bpe_act;
  if (g == 0) g = t;
  const i64 hkv = m.kv_heads * h / m.heads;
  switch (kind) {
    case ATTN:
      return {ceil_div(2 * T * h * (2 * h + 2 * hkv) + 4 * b * m.seq * m.seq * h, t),
              ceil_div(bpe * h * (2 * h + 2 * hkv), t) + 2 * T * h * bpe};
    case MLP:
      return {ceil_div(2 * T * m.nm * h * m.ffn, t), ceil_div(bpe * m.nm * h * m.ffn, t) + 2 * T * h * bpe};
    case MOE:
      return {ceil_div(2 * T * m.topk * m.nm * h * m.ffn, t),
              ceil_div(bpe * m.E * m.nm * h * m.ffn, g) + 2 * T * h * bpe};
    case EMB:
      return {0, 2 * T * h * bpe};
    default:  // HEAD
      return {ceil_div(2 * T * h * m.V, t), ceil_div(bpe * m.V * h, t) + T * h * bpe + ceil_div(T * m.V * bpe, t)};
  }
}
// roofline duration; backward = 2x FLOP and 2x bytes, rounded on its own (A6)
i64 op_dur(const orc_input& m, const orc_type& ty, int kind, bool bwd, i64 t, i64 b, i64 g = 0) {
  Cost c = op_cost(m, kind, t, b, g);
  i64 mul = bwd ? 2 : 1;
  double rf = ty.peak_flop_per_ns * ty.eff_flop[kind];
  double rm = ty.hbm_bytes_per_ns * ty.eff_mem[kind];
  return std::max(ceilq(mul * c.flop, rf), ceilq(mul * c.bytes, rm));
}

// --- literal async ring (DESIGN C.11): rank r sends to r+1 over edge r --------
// send(r,k).start = max(send(r,k-1).end, send(r-1,k-1).end)
i64 ring_sim(const std::vector<i64>& edge_tau, int steps) {
  const int n = (int)edge_tau.size();
  std::vector<i64> end(n, 0), nxt(n);
  for (int k = 0; k < steps; ++k) {
    for (int r = 0; r < n; ++r) nxt[r] = std::max(end[r], end[(r + n - 1) % n]) + edge_tau[r];
    end.swap(nxt);
  }
  i64 t = 0;
  for (i64 e : end) t = std::max(t, e);
  return t;
}

// --- f3 progressive filling (DESIGN F.1): nf flows over links; flow f uses
// links inc[f][0..nfl[f]) of capacity linkcap[e] and is capped at cap[f]
// (its own path); rates out.  share_e = residual_e / unfrozen_e (one IEEE
// division); s = min(share over links with unfrozen flows, unfrozen caps);
// every unfrozen flow on an argmin link or with cap == s freezes at s; each
// link's residual -= (flows frozen on it) x s.
void maxmin_fill(int nf, const std::vector<std::vector<int>>& inc, const std::map<int, double>& linkcap,
                 const std::vector<double>& cap, std::vector<double>& rate) {
  std::map<int, double> res;
  std::map<int, int> cnt;
  for (int f = 0; f < nf; ++f)
    for (int e : inc[f]) {
      res[e] = linkcap.at(e);
      cnt[e] += 1;
    }
  std::vector<char> frozen(nf, 0);
  int left = nf;
  rate.assign(nf, 0.0);
  while (left) {
    double s = 1e300;
    for (auto& kv : cnt)
      if (kv.second > 0) s = std::min(s, res[kv.first] / kv.second);
    for (int f = 0; f < nf; ++f)
      if (!frozen[f]) s = std::min(s, cap[f]);
    std::vector<int> fz;
    for (int f = 0; f < nf; ++f) {
      if (frozen[f]) continue;
      bool hit = cap[f] == s;
      for (int e : inc[f]) hit = hit || (cnt[e] > 0 && res[e] / cnt[e] == s);
      if (hit) fz.push_back(f);
    }
    std::map<int, int> took;
    for (int f : fz) {
      frozen[f] = 1;
      rate[f] = s;
      for (int e : inc[f]) took[e] += 1;
      --left;
    }
    for (auto& kv : took) {
      res[kv.first] = res[kv.first] - (double)kv.second * s;
      cnt[kv.first] -= kv.second;
    }
  }
}

// --- Hamilton / largest remainder (DESIGN C.4): ties -> lower index ----------
std::vector<i64> hamilton(i64 n, const std::vector<i64>& w) {
  const int k = (int)w.size();
  i64 W = 0;
  for (i64 x : w) W += x;
  std::vector<i64> q(k), rem(k);
  i64 given = 0;
  for (int i = 0; i < k; ++i) {
    q[i] = n * w[i] / W;
    rem[i] = n * w[i] % W;
    given += q[i];
  }
  std::vector<int> order(k);
  for (int i = 0; i < k; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return rem[a] > rem[b]; });
  for (i64 s = 0; s < n - given; ++s) q[order[s]] += 1;
  return q;
}

// --- candidate space (DESIGN C.2) --------------------------------------------
// type2 >= 0: a mixed-type TP group (DESIGN V.1): tp/2 devices of `type` and
// tp/2 of `type2`
struct StageSpec { int type; int tp; int type2 = -1; };
struct ClassSpec { std::vector<StageSpec> st; int D; };
struct Template { int b; std::vector<ClassSpec> cls; i64 radix; i64 prefix; };

bool tp_ok(const orc_input& in, int type, int tp) {
  return in.types[type].gpus_per_node % tp == 0 && in.heads % tp == 0 && in.kv_heads % tp == 0;
}

i64 ipow(i64 a, i64 e) { i64 r = 1; while (e-- > 0) r *= a; return r; }

std::vector<Template> enumerate(const orc_input& in, const Cluster& cl) {
  std::vector<Template> out;
  std::vector<int> bs(in.bset, in.bset + in.n_b), ps(in.pset, in.pset + in.n_p);
  std::sort(bs.begin(), bs.end());
  std::sort(ps.begin(), ps.end());
  const int nt = in.n_types;
  for (int b : bs) {
    if (in.B % b) continue;
    const i64 M = in.B / b;
    auto emit = [&](std::vector<ClassSpec> cls) {
      i64 D = 0;
      for (auto& c : cls) D += c.D;
      if (M < D) return;  // the only structural filter
      Template t{b, cls, 1, 0};
      for (auto& c : cls) {
        int P = (int)c.st.size();
        if (P <= in.pmax) t.radix *= ipow(2 * in.r_layer + 1, P - 1);
      }
      t.radix *= ipow(2 * in.r_batch + 1, (i64)cls.size() - 1);
      out.push_back(t);
    };
    if (in.homo) {
      // per type: "unused" then (tp, P, D) ascending
      struct Opt { int tp, P, D; };
      std::vector<std::vector<Opt>> opts(nt);
      for (int t = 0; t < nt; ++t) {
        opts[t].push_back({0, 0, 0});
        std::vector<int> tps(in.tpset[t], in.tpset[t] + in.n_tp[t]);
        std::sort(tps.begin(), tps.end());
        for (int tp : tps) {
          if (!tp_ok(in, t, tp)) continue;
          for (int P : ps) {
            if (P > in.L) continue;
            for (i64 D = 1; D * P * tp <= cl.n_of_type[t]; ++D) {
              if (in.use_all && D * P * tp != cl.n_of_type[t]) continue;
              opts[t].push_back({tp, P, (int)D});
            }
          }
        }
      }
      std::vector<int> pick(nt, 0);
      while (true) {
        bool any = false;
        for (int t = 0; t < nt; ++t) any |= pick[t] != 0;
        if (any) {
          std::vector<ClassSpec> cls;
          for (int t = 0; t < nt; ++t) {
            if (!pick[t]) continue;
            Opt o = opts[t][pick[t]];
            ClassSpec c;
            c.D = o.D;
            for (int s = 0; s < o.P; ++s) c.st.push_back({t, o.tp});
            cls.push_back(c);
          }
          emit(cls);
        }
        int t = nt - 1;  // odometer, type 0 most significant
        while (t >= 0 && ++pick[t] == (int)opts[t].size()) { pick[t] = 0; --t; }
        if (t < 0) break;
      }
    }
    if (in.mixed && nt >= 2) {
      struct Opt { int tp, P; };
      std::vector<std::vector<Opt>> opts(nt);
      for (int t = 0; t < nt; ++t) {
        std::vector<int> tps(in.tpset[t], in.tpset[t] + in.n_tp[t]);
        std::sort(tps.begin(), tps.end());
        for (int tp : tps) {
          if (!tp_ok(in, t, tp)) continue;
          for (int P : ps) opts[t].push_back({tp, P});
        }
      }
      bool empty = false;
      for (int t = 0; t < nt; ++t) empty |= opts[t].empty();
      if (!empty) {
        std::vector<int> pick(nt, 0);
        while (true) {
          int sumP = 0;
          i64 Dmax = INT64_MAX;
          for (int t = 0; t < nt; ++t) {
            Opt o = opts[t][pick[t]];
            sumP += o.P;
            Dmax = std::min(Dmax, cl.n_of_type[t] / ((i64)o.P * o.tp));
          }
          if (sumP <= in.L && Dmax >= 1) {
            for (i64 D = in.use_all ? Dmax : 1; D <= Dmax; ++D) {
              ClassSpec c;
              c.D = (int)D;
              for (int t = 0; t < nt; ++t)
                for (int s = 0; s < opts[t][pick[t]].P; ++s) c.st.push_back({t, opts[t][pick[t]].tp});
              emit({c});
            }
          }
          int t = nt - 1;
          while (t >= 0 && ++pick[t] == (int)opts[t].size()) { pick[t] = 0; --t; }
          if (t < 0) break;
        }
      }
    }
    if (in.mixtp && nt >= 2) {
      // V.1 (DESIGN): one class whose every stage is a mixed TP group of tp
      // devices, tp/2 of type a and tp/2 of type a2 (a < a2); tp >= 2 in both
      // types' TP sets, tp | heads and kv heads, tp/2 | GPUs per node (each
      // half fits a node); D replicas of P stages need
      // D P tp/2 GPUs of each type (use_all: exactly all of both)
      for (int a = 0; a < nt; ++a)
        for (int a2 = a + 1; a2 < nt; ++a2) {
          std::vector<int> tps;
          for (int q = 0; q < in.n_tp[a]; ++q) tps.push_back(in.tpset[a][q]);
          std::sort(tps.begin(), tps.end());
          for (int tp : tps) {
            bool in2 = false;
            for (int q = 0; q < in.n_tp[a2]; ++q) in2 |= in.tpset[a2][q] == tp;
            if (tp < 2 || !in2 || in.heads % tp || in.kv_heads % tp || in.types[a].gpus_per_node % (tp / 2) ||
                in.types[a2].gpus_per_node % (tp / 2))
              continue;
            for (int P : ps) {
              if (P > in.L) continue;
              for (i64 D = 1; D * P * (tp / 2) <= std::min(cl.n_of_type[a], cl.n_of_type[a2]); ++D) {
                if (in.use_all && (D * P * (tp / 2) != cl.n_of_type[a] || D * P * (tp / 2) != cl.n_of_type[a2])) continue;
                ClassSpec c;
                c.D = (int)D;
                for (int st = 0; st < P; ++st) c.st.push_back(StageSpec{a, tp, a2});
                emit({c});
              }
            }
          }
        }
    }
  }
  i64 acc = 0;
  for (auto& t : out) { t.prefix = acc; acc += t.radix; }
  return out;
}

// --- one decoded, placed and partitioned candidate ---------------------------
// a stage group: tp GPUs [base, base+tp) on node; V.1 mixed group: tp/2 GPUs
// [base, base+tp/2) on node and tp/2 at the same base on node2
struct Group { int node, base, node2 = -1; };

struct Plan {
  const Template* tpl;
  std::vector<std::vector<int>> delta;  // per class, per boundary (P-1)
  std::vector<int> eps;                 // per class (C-1)
  std::vector<std::vector<std::vector<Group>>> place;  // [class][replica][stage]
  std::vector<std::vector<i64>> layers;  // [class][stage]
  std::vector<std::vector<i64>> mb;      // [class][replica] micro-batches
  int status = 0;
};

struct Oracle {
  orc_input in;
  std::vector<orc_type> types;
  std::vector<int32_t> node_type;
  Cluster cl;
  std::vector<Template> tpls;
  i64 N = 0;
  int compact_mode = 0;  // 0 literal, 1 compact (see the header)

  void init() {
    in.types = types.data();
    in.node_type = node_type.data();
    cl.in = &in;
    cl.n_of_type.assign(in.n_types, 0);
    cl.nodes_of_type.assign(in.n_types, {});
    for (int n = 0; n < in.n_nodes; ++n) {
      int t = node_type[n];
      cl.ntype.push_back(t);
      cl.gpn.push_back(types[t].gpus_per_node);
      cl.n_of_type[t] += types[t].gpus_per_node;
      cl.nodes_of_type[t].push_back(n);
    }
    tpls = enumerate(in, cl);
    N = tpls.empty() ? 0 : tpls.back().prefix + tpls.back().radix;
  }

  // C.2 decode: template = max{tau : prefix <= i}; digits LSB first
  Plan decode(i64 i) const {
    Plan p;
    size_t lo = 0, hi = tpls.size();
    while (hi - lo > 1) {
      size_t mid = (lo + hi) / 2;
      if (tpls[mid].prefix <= i) lo = mid; else hi = mid;
    }
    p.tpl = &tpls[lo];
    i64 local = i - p.tpl->prefix;
    const int C = (int)p.tpl->cls.size();
    p.delta.resize(C);
    for (int c = 0; c < C; ++c) {
      int P = (int)p.tpl->cls[c].st.size();
      p.delta[c].assign(P > 0 ? P - 1 : 0, 0);
      if (P <= in.pmax)
        for (int s = 0; s < P - 1; ++s) {
          p.delta[c][s] = (int)(local % (2 * in.r_layer + 1)) - in.r_layer;
          local /= (2 * in.r_layer + 1);
        }
    }
    p.eps.assign(C, 0);
    for (int c = 0; c < C - 1; ++c) {
      p.eps[c] = (int)(local % (2 * in.r_batch + 1)) - in.r_batch;
      local /= (2 * in.r_batch + 1);
    }
    return p;
  }

  // C.3 placement: class-major, replica-major, stage-major; lowest-id node of
  // the stage's type with a free tp-aligned block, lowest block.
  void place(Plan& p) const {
    std::vector<std::vector<char>> used(in.n_nodes);
    for (int n = 0; n < in.n_nodes; ++n) used[n].assign(cl.gpn[n], 0);
    const auto& cls = p.tpl->cls;
    p.place.resize(cls.size());
    for (size_t c = 0; c < cls.size(); ++c) {
      p.place[c].resize(cls[c].D);
      for (int r = 0; r < cls[c].D; ++r) {
        for (const StageSpec& s : cls[c].st) {
          // V.1: a mixed group takes tp/2-blocks; the a2 half sits at the same
          // base on the lowest node of type a2 where that block is free
          const int w = s.type2 >= 0 ? s.tp / 2 : s.tp;
          Group g{-1, -1};
          for (int n : cl.nodes_of_type[s.type]) {
            for (int k = 0; k * w < cl.gpn[n] && g.node < 0; ++k) {
              bool fr = true;
              for (int q = 0; q < w; ++q) fr &= !used[n][k * w + q];
              if (fr) g = Group{n, k * w};
            }
            if (g.node >= 0) break;
          }
          if (g.node >= 0 && s.type2 >= 0) {
            for (int n : cl.nodes_of_type[s.type2]) {
              bool fr = true;
              for (int q = 0; q < w; ++q) fr &= !used[n][g.base + q];
              if (fr) { g.node2 = n; break; }
            }
            if (g.node2 < 0) g.node = -1;
          }
          if (g.node < 0) { std::fprintf(stderr, "oracle: placement failed\n"); std::abort(); }
          for (int q = 0; q < w; ++q) used[g.node][g.base + q] = 1;
          if (g.node2 >= 0)
            for (int q = 0; q < w; ++q) used[g.node2][g.base + q] = 1;
          p.place[c][r].push_back(g);
        }
      }
    }
  }

  // device q of a group of t GPUs as (node, local rank); V.1: devices
  // [0, t/2) on node, [t/2, t) on node2, both from base
  static std::pair<int, int> dev(const Group& g, int t, int q) {
    if (g.node2 < 0) return {g.node, g.base + q};
    return q < t / 2 ? std::make_pair(g.node, g.base + q) : std::make_pair(g.node2, g.base + q - t / 2);
  }
  Link link_dd(const Group& g1, int t1, int q1, const Group& g2, int t2, int q2) const {
    const auto a = dev(g1, t1, q1), z = dev(g2, t2, q2);
    return cl.gpu_to_gpu(a.first, a.second, z.first, z.second);
  }
  // TP ring of a stage group: device 0 -> 1 -> ... -> t-1 -> 0
  std::vector<Link> tp_ring(const Group& g, int t) const {
    std::vector<Link> e;
    for (int q = 0; q < t; ++q) e.push_back(link_dd(g, t, q, g, t, (q + 1) % t));
    return e;
  }
  i64 act_bytes(int b) const { return (i64)b * in.seq * in.h * in.bpe_act; }  // A5

  // TP all-reduce after attention / MLP (A16): literal ring, 2(t-1) steps
  i64 tp_allreduce(const Group& g, int t, int b) const {
    if (t == 1) return 0;
    std::vector<i64> taus;
    for (const Link& e : tp_ring(g, t)) taus.push_back(tau(e, ceil_div(act_bytes(b), t)));
    return ring_sim(taus, 2 * (t - 1));
  }
  // EP all-to-all (A17): g-1 rounds, each bounded by the slowest pair of the group
  i64 ep_alltoall(const Group& g, int t, int b) const {
    if (t == 1) return 0;
    i64 per = ceil_div(act_bytes(b) * in.topk, (i64)t * t);
    i64 slow = 0;
    for (int x = 0; x < t; ++x)
      for (int y = 0; y < t; ++y)
        if (x != y) slow = std::max(slow, tau(link_dd(g, t, x, g, t, y), per));
    return (i64)(t - 1) * slow;
  }

  // --- SURVEY §8(f) f4 variants --------------------------------------------------
  // V.2 (DESIGN): a class with P >= 2 stages runs the interleaved 1F1B with v =
  // in.interleave model chunks per stage; chunk k of a stage with l layers has
  // floor(l / v) + [k < l mod v] layers.
  int vchunks(const ClassSpec& c) const { return in.interleave > 1 && c.st.size() >= 2 ? in.interleave : 1; }
  static i64 chunk_layers(i64 l, int v, int k) { return l / v + (k < l % v ? 1 : 0); }
  // V.3 (DESIGN): in a single-class MoE template, the expert-parallel group of a
  // stage is the union of every replica's TP group of that stage (g = D tp).
  bool ep_class(const Template& t) const { return in.ep_dp && in.E > 1 && t.cls.size() == 1; }
  i64 ep_g(const Template& t, const StageSpec& s) const { return ep_class(t) ? (i64)t.cls[0].D * s.tp : 0; }

  // compute-only fwd+bwd of one layer (C.4); g: expert divisor (V.3, 0 = tp)
  // V.3: all-to-all over the union of the groups' devices (g = n tp): g - 1
  // rounds, each bounded by the slowest ordered pair, message ceil(A k / (t g))
  // per pair (A17 is the one-group case, g = t)
  // (memoised per (groups, t, b): the group-wide pair scan is O(g^2))
  mutable std::mutex a2a_mu;
  mutable std::map<std::tuple<std::vector<std::pair<int, int>>, int, int>, i64> a2a_memo;
  i64 ep_alltoall_x(const std::vector<Group>& gs, int t, int b) const {
    std::vector<std::pair<int, int>> key;
    for (const Group& g : gs) key.push_back({g.node, g.base});
    {
      std::lock_guard<std::mutex> lk(a2a_mu);
      auto it = a2a_memo.find(std::make_tuple(key, t, b));
      if (it != a2a_memo.end()) return it->second;
    }
    const i64 v = ep_alltoall_x_scan(gs, t, b);
    std::lock_guard<std::mutex> lk(a2a_mu);
    a2a_memo[std::make_tuple(key, t, b)] = v;
    return v;
  }
  i64 ep_alltoall_x_scan(const std::vector<Group>& gs, int t, int b) const {
    std::vector<std::pair<int, int>> dev;
    for (const Group& g : gs)
      for (int q = 0; q < t; ++q) dev.push_back({g.node, g.base + q});
    const i64 g = (i64)dev.size();
    if (g == 1) return 0;
    const i64 per = ceil_div(act_bytes(b) * in.topk, (i64)t * g);
    i64 slow = 0;
    for (size_t x = 0; x < dev.size(); ++x)
      for (size_t y = 0; y < dev.size(); ++y)
        if (x != y) slow = std::max(slow, tau(cl.gpu_to_gpu(dev[x].first, dev[x].second, dev[y].first, dev[y].second), per));
    return (g - 1) * slow;
  }

  // duration of one op on one device of stage group ss; V.1: a mixed group's
  // devices hold equal shards and every op ends with a TP collective, so the
  // op lasts as long as on its slower device type -- "the bottleneck device"
  // (PAPER.md:280 C4)
  i64 sdur(const StageSpec& ss, int kind, bool bwd, int b, i64 g = 0) const {
    i64 d = op_dur(in, types[ss.type], kind, bwd, ss.tp, b, g);
    if (ss.type2 >= 0) d = std::max(d, op_dur(in, types[ss.type2], kind, bwd, ss.tp, b, g));
    return d;
  }
  // compute-only fwd+bwd of one layer (C.4); g: expert divisor (V.3, 0 = tp)
  i64 tcomp(const StageSpec& s, int b, i64 g = 0) const {
    int mk = in.E > 1 ? MOE : MLP;
    return sdur(s, ATTN, false, b) + sdur(s, mk, false, b, g) + sdur(s, ATTN, true, b) + sdur(s, mk, true, b, g);
  }
  i64 extra_fb(const StageSpec& s, int b, int kind) const { return sdur(s, kind, false, b) + sdur(s, kind, true, b); }

  // C.4 step 1: non-uniform partition
  void partition(Plan& p) const {
    const auto& cls = p.tpl->cls;
    const int C = (int)cls.size(), b = p.tpl->b;
    const i64 M = in.B / b;
    p.layers.resize(C);
    std::vector<i64> repl_w;  // class-major replica weights
    for (int c = 0; c < C; ++c) {
      const int P = (int)cls[c].st.size();
      std::vector<i64> w(P);
      for (int s = 0; s < P; ++s) w[s] = (i64(1) << 40) / tcomp(cls[c].st[s], b, ep_g(*p.tpl, cls[c].st[s]));
      std::vector<i64> l = hamilton(in.L, w);
      for (int s = 0; s < P; ++s) {
        i64 d_here = s < P - 1 ? p.delta[c][s] : 0;
        i64 d_prev = s > 0 ? p.delta[c][s - 1] : 0;
        l[s] += d_here - d_prev;
        if (l[s] < 1) p.status = -1;
        if (l[s] < vchunks(cls[c])) p.status = -1;  // V.2: every chunk holds a layer
      }
      p.layers[c] = l;
      if (p.status) return;
      i64 worst = 0;
      for (int s = 0; s < P; ++s) {
        i64 t = l[s] * tcomp(cls[c].st[s], b, ep_g(*p.tpl, cls[c].st[s]));
        if (s == 0) t += extra_fb(cls[c].st[s], b, EMB);
        if (s == P - 1) t += extra_fb(cls[c].st[s], b, HEAD);
        worst = std::max(worst, t);
      }
      for (int r = 0; r < cls[c].D; ++r) repl_w.push_back((i64(1) << 40) / worst);
    }
    std::vector<i64> m = hamilton(M, repl_w);
    p.mb.resize(C);
    size_t k = 0;
    i64 R = 0;
    for (int c = 0; c < C; ++c) {
      for (int r = 0; r < cls[c].D; ++r) {
        i64 v = m[k++];
        if (c < C - 1) v += p.eps[c];
        p.mb[c].push_back(v);
      }
      if (c < C - 1) R -= (i64)cls[c].D * p.eps[c];
    }
    const i64 Dl = cls[C - 1].D;
    i64 q = R >= 0 ? R / Dl : -((-R + Dl - 1) / Dl);  // floor
    i64 rm = R - q * Dl;                               // in [0, Dl)
    for (int r = 0; r < Dl; ++r) p.mb[C - 1][r] += q + (r < rm ? 1 : 0);
    for (int c = 0; c < C; ++c)
      for (i64 v : p.mb[c])
        if (v < 1) p.status = -2;
    // V.2: the interleaved schedule needs every replica's micro-batch count to
    // be a multiple of its depth (Megatron-LM's rule for virtual pipelines)
    for (int c = 0; c < C; ++c)
      if (vchunks(cls[c]) > 1)
        for (i64 v : p.mb[c])
          if (v % (i64)cls[c].st.size()) p.status = -2;
  }

  // --- f2 / DESIGN M.1: memory feasibility -------------------------------------
  // The paper never gates on memory (SPEC.md:104 makes it a warning); this row
  // follows SURVEY §8(f) f2: "params + grads + optimizer + 1F1B in-flight
  // activations <= capacity", read as follows, for one device of every stage
  // group of every replica:
  //   params  = l_s * ceil(W_layer / t) + [s = 0] ceil(V h / t)
  //             + [s = P-1] ceil((V h [!tied] + h) / t)          (C.6's W_layer)
  //   static  = params * (bpe_act + bpe_grad + 12)   weights, gradients (A7), and
  //             Adam's fp32 master copy + two moments (4 + 4 + 4 bytes)
  //   act     = b s h (10 + 24/t) bytes per layer and in-flight micro-batch
  //             (Korthikanti et al. 2022, TP without sequence parallelism,
  //             16-bit, attention scores recomputed -- their "selective
  //             recomputation", i.e. no 5 a s^2 b term), as one integer
  //             ceil(b s h (10 t + 24) / t)
  //   in flight = min(P - s, m_r): 1F1B's warm-up depth of stage s
  //   need    = static + in_flight * l_s * act  <=  mem_bytes(type)
  // Any device over capacity -> -3.  Checked after the layer / batch split
  // (-1 / -2 take precedence).
  i64 device_bytes(const StageSpec& ss, int P, int s, i64 l, i64 m, int b) const {
    const i64 t = ss.tp, h = in.h, S = in.seq;
    const i64 hkv = in.kv_heads * h / in.heads;
    const i64 Wlayer = h * (2 * h + 2 * hkv) + in.nm * h * in.ffn * in.E + (in.E > 1 ? h * in.E : 0) + 2 * h;
    i64 params = l * ceil_div(Wlayer, t);
    if (s == 0) params += ceil_div(in.V * h, t);
    if (s == P - 1) params += ceil_div(in.V * h * (in.tied ? 0 : 1) + h, t);
    const i64 stat = params * (in.bpe_act + in.bpe_grad + 12);
    const i64 act = ceil_div((i64)b * S * h * (10 * t + 24), t);
    const i64 inflight = std::min((i64)(P - s), m);
    return stat + inflight * l * act;
  }
  void check_memory(Plan& p) const {
    if (!in.mem_check || p.status) return;
    const auto& cls = p.tpl->cls;
    for (size_t c = 0; c < cls.size(); ++c) {
      const int P = (int)cls[c].st.size();
      for (int r = 0; r < cls[c].D; ++r)
        for (int s = 0; s < P; ++s) {
          const StageSpec& ss = cls[c].st[s];
          if (device_bytes(ss, P, s, p.layers[c][s], p.mb[c][r], p.tpl->b) > types[ss.type].mem_bytes) {
            p.status = -3;
            return;
          }
        }
    }
  }

  // --- C.7 / C.11: event-driven 1F1B over every replica ------------------------
  // A stage group runs its op list in order; an op starts when the previous op
  // of the group has ended and its input has arrived.  Ops are (fwd?, chunk k,
  // micro-batch j); v = 1 (every chunk index 0) is C.7's non-interleaved 1F1B.
  struct Op { bool fwd; int k, j; };
  struct SimGroup {
    int P, s, m, v = 1;
    std::vector<i64> f, g;     // per chunk: forward / backward duration
    i64 c_prev, c_next;        // c_prev: boundary s-1 -> s, c_next: s -> s+1
    i64 c_wrap = 0;            // V.2: stage P-1 -> stage 0 (next chunk) and back
    i64 lowb = 0;              // B.1: backward work of the lower bucket (its last ceil(l/2) layers + embedding)
    std::vector<Op> ops;
    size_t next = 0;
    bool busy = false;
    i64 done = 0;  // end of the group's last op (its last backward, C.7)
    std::vector<char> inF, inB;  // [k * m + j]
  };
  struct Ev {
    i64 t, seq;
    int kind;  // 0 = op done, 1 = F input arrives, 2 = B input arrives
    int grp, key;
    bool operator>(const Ev& o) const { return std::tie(t, seq) > std::tie(o.t, o.seq); }
  };

  // C.7: warm-up w = min(P-1-s, m) forwards, then (F, B) pairs, then the rest.
  // V.2 (Megatron-LM's interleaved schedule, Narayanan et al. 2021): the
  // forward table visits micro-batches in groups of P -- for each group, chunk
  // 0..v-1, the group's micro-batches in order; the backward table is the same
  // with the chunks in reverse order; warm-up w = min(2(P-1-s) + (v-1) P, m v)
  // table forwards, then (F_tab[w+i], B_tab[i]) pairs, then the remaining
  // backwards.  Needs m mod P = 0 (partition gives -2 otherwise).
  static std::vector<Op> op_order(int P, int s, int m, int v = 1) {
    std::vector<Op> o;
    if (v == 1) {
      int w = std::min(P - 1 - s, m);
      for (int j = 0; j < w; ++j) o.push_back({true, 0, j});
      for (int i = 0; i < m - w; ++i) { o.push_back({true, 0, w + i}); o.push_back({false, 0, i}); }
      for (int j = m - w; j < m; ++j) o.push_back({false, 0, j});
      return o;
    }
    std::vector<Op> F, B;
    for (int g0 = 0; g0 < m; g0 += P) {
      for (int k = 0; k < v; ++k)
        for (int j = g0; j < std::min(g0 + P, m); ++j) F.push_back({true, k, j});
      for (int k = v - 1; k >= 0; --k)
        for (int j = g0; j < std::min(g0 + P, m); ++j) B.push_back({false, k, j});
    }
    const int n = m * v;
    const int w = std::min(2 * (P - 1 - s) + (v - 1) * P, n);
    for (int i = 0; i < w; ++i) o.push_back(F[i]);
    for (int i = 0; i < n - w; ++i) { o.push_back(F[w + i]); o.push_back(B[i]); }
    for (int i = n - w; i < n; ++i) o.push_back(B[i]);
    return o;
  }

  // Runs the listed pipelines (each a consecutive run of P groups); returns the
  // time of the last event (T0).
  static i64 run_pipelines(std::vector<SimGroup>& G) {
    std::priority_queue<Ev, std::vector<Ev>, std::greater<Ev>> q;
    i64 seq = 0, last = 0;
    auto try_start = [&](int gi, i64 t) {
      SimGroup& g = G[gi];
      if (g.busy || g.next >= g.ops.size()) return;
      const Op op = g.ops[g.next];
      const int key = op.k * g.m + op.j;
      bool ready = op.fwd ? g.inF[key] : g.inB[key];
      if (!ready) return;
      g.busy = true;
      q.push(Ev{t + (op.fwd ? g.f[op.k] : g.g[op.k]), seq++, 0, gi, key});
    };
    for (size_t gi = 0; gi < G.size(); ++gi) {
      SimGroup& g = G[gi];
      g.inF.assign((size_t)g.v * g.m, 0);
      g.inB.assign((size_t)g.v * g.m, 0);
      if (g.s == 0)
        for (int j = 0; j < g.m; ++j) g.inF[j] = 1;  // chunk 0 of stage 0: the data loader
      g.ops = op_order(g.P, g.s, g.m, g.v);
    }
    for (size_t gi = 0; gi < G.size(); ++gi) try_start((int)gi, 0);
    while (!q.empty()) {
      Ev e = q.top();
      q.pop();
      last = std::max(last, e.t);
      SimGroup& g = G[e.grp];
      if (e.kind == 0) {
        const Op op = g.ops[g.next];
        g.busy = false;
        g.done = e.t;
        g.next++;
        const int s0 = e.grp - g.s, sl = s0 + g.P - 1;  // stage 0 / stage P-1 of this pipeline
        if (op.fwd) {
          if (g.s < g.P - 1) q.push(Ev{e.t + g.c_next, seq++, 1, e.grp + 1, e.key});
          else if (op.k < g.v - 1) q.push(Ev{e.t + g.c_wrap, seq++, 1, s0, e.key + g.m});  // V.2 wrap
          else g.inB[e.key] = 1;  // last virtual stage: B follows its own F
        } else if (g.s > 0) {
          q.push(Ev{e.t + g.c_prev, seq++, 2, e.grp - 1, e.key});
        } else if (op.k > 0) {
          q.push(Ev{e.t + g.c_wrap, seq++, 2, sl, e.key - g.m});  // V.2 wrap back
        }
        try_start(e.grp, e.t);
      } else {
        (e.kind == 1 ? g.inF : g.inB)[e.key] = 1;
        try_start(e.grp, e.t);
      }
    }
    for (const SimGroup& g : G)
      if (g.next != g.ops.size()) { std::fprintf(stderr, "oracle: 1F1B deadlock\n"); std::abort(); }
    return last;
  }

  // TP all-reduce, compact form: 2(t-1) steps x the slowest ring edge (the
  // value the literal async ring reaches; pinned by the ring closed forms)
  i64 tp_allreduce_compact(const Group& g, int t, int b) const {
    if (t == 1) return 0;
    i64 slow = 0;
    for (const Link& e : tp_ring(g, t)) slow = std::max(slow, tau(e, ceil_div(act_bytes(b), t)));
    return 2 * (i64)(t - 1) * slow;
  }

  // One layer's forward (bwd = 0) or backward (bwd = 1) op chain on stage
  // group gr: attn + AR + mlp + AR (dense) or attn + AR + A2A + moe + A2A (MoE)
  // (DESIGN C.5, A16, A17).
  // V.3: epg = every replica's group of this stage (the expert-parallel group),
  // or nullptr (A17: the TP group)
  i64 layer_chain(const StageSpec& ss, const Group& gr, int b, int bwd, bool compact,
                  const std::vector<Group>* epg = nullptr) const {
    const i64 ar = compact ? tp_allreduce_compact(gr, ss.tp, b) : tp_allreduce(gr, ss.tp, b);
    i64 chain = sdur(ss, ATTN, bwd, b) + ar;
    if (in.E > 1) {
      const i64 a2a = epg ? ep_alltoall_x(*epg, ss.tp, b) : ep_alltoall(gr, ss.tp, b);
      const i64 g = epg ? (i64)epg->size() * ss.tp : 0;
      chain += a2a + sdur(ss, MOE, bwd, b, g) + a2a;
    } else {
      chain += sdur(ss, MLP, bwd, b) + ar;
    }
    return chain;
  }

  // --- C.6: gradient-sync segments ------------------------------------------------
  struct Seg {
    i64 a, z, S, RS, AR;
    int tstar;
    std::vector<int> sc;  // stage of every class holding layers [a, z)
    std::vector<int> bk;  // B.1: bucket of that stage holding them (0 lower, 1 upper)
  };
  // B.1 (DESIGN): with two buckets a stage's l layers split into the lower
  // ceil(l/2) (+ the embedding on stage 0) and the upper rest (+ the head)
  bool two_buckets() const { return in.sync_buckets == 2; }
  static i64 lower_half(i64 l) { return (l + 1) / 2; }
  std::vector<Seg> segments(const Plan& p, bool compact) const {
    const auto& cls = p.tpl->cls;
    const int C = (int)cls.size();
    i64 D = 0;
    for (auto& c : cls) D += c.D;
    // layer ranges of each class in model order: (first layer, stage).  V.2:
    // virtual stage k P + s = chunk k of stage s, so a stage holds v ranges.
    std::vector<i64> cuts{0, in.L};
    std::vector<std::vector<std::pair<i64, int>>> start(C);
    for (int c = 0; c < C; ++c) {
      const int P = (int)cls[c].st.size(), v = vchunks(cls[c]);
      i64 a = 0;
      for (int k = 0; k < v; ++k)
        for (int s = 0; s < P; ++s) {
          start[c].push_back({a, s});
          cuts.push_back(a);
          const i64 l = chunk_layers(p.layers[c][s], v, k);
          if (two_buckets() && lower_half(l) < l) cuts.push_back(a + lower_half(l));  // B.1
          a += l;
        }
    }
    std::sort(cuts.begin(), cuts.end());
    cuts.erase(std::unique(cuts.begin(), cuts.end()), cuts.end());
    const i64 hkv = in.kv_heads * in.h / in.heads;
    // V.3: expert weights are sharded over the replicas (one copy per class), so
    // a single-class EP template synchronises only the dense parameters
    const i64 Wexp = ep_class(*p.tpl) ? 0 : in.nm * in.h * in.ffn * in.E;
    const i64 Wlayer = in.h * (2 * in.h + 2 * hkv) + Wexp + (in.E > 1 ? in.h * in.E : 0) + 2 * in.h;
    std::vector<Seg> out;
    for (size_t j = 0; j + 1 < cuts.size(); ++j) {
      Seg sg;
      sg.a = cuts[j];
      sg.z = cuts[j + 1];
      sg.S = (sg.z - sg.a) * Wlayer * in.bpe_grad;
      if (sg.a == 0) sg.S += in.V * in.h * in.bpe_grad;
      if (sg.z == in.L) sg.S += (in.V * in.h * (in.tied ? 0 : 1) + in.h) * in.bpe_grad;
      sg.sc.assign(C, 0);
      sg.tstar = 1 << 30;
      sg.bk.assign(C, 0);
      for (int c = 0; c < C; ++c) {
        size_t x = 0;
        while (x + 1 < start[c].size() && start[c][x + 1].first <= sg.a) ++x;
        const int s = start[c][x].second;
        sg.sc[c] = s;
        sg.bk[c] = two_buckets() && sg.a >= start[c][x].first + lower_half(p.layers[c][s]) ? 1 : 0;
        sg.tstar = std::min(sg.tstar, cls[c].st[s].tp);
      }
      // reshard (A14): every group with tp != t* re-lays S into t* shards over its ring
      sg.RS = 0;
      for (int c = 0; c < C; ++c) {
        const int tp = cls[c].st[sg.sc[c]].tp;
        if (tp == sg.tstar) continue;
        for (int r = 0; r < cls[c].D; ++r)
          for (const Link& e : tp_ring(p.place[c][r][sg.sc[c]], tp)) sg.RS = std::max(sg.RS, tau(e, ceil_div(sg.S, sg.tstar)));
      }
      // DP ring all-reduce: ring order class asc, replica asc, wrap; ring q < t*
      std::vector<Group> ring;
      std::vector<int> ring_c;  // class of each ring position
      for (int c = 0; c < C; ++c)
        for (int r = 0; r < cls[c].D; ++r) {
          ring.push_back(p.place[c][r][sg.sc[c]]);
          ring_c.push_back(c);
        }
      const i64 chunk = ceil_div(ceil_div(sg.S, sg.tstar), D);
      sg.AR = 0;
      for (int q = 0; q < sg.tstar; ++q) {
        std::vector<i64> taus;
        for (size_t k = 0; k < ring.size(); ++k) {
          const Group& u = ring[k];
          const Group& v = ring[(k + 1) % ring.size()];
          taus.push_back(tau(link_dd(u, cls[ring_c[k]].st[sg.sc[ring_c[k]]].tp, q, v, cls[ring_c[(k + 1) % ring.size()]].st[sg.sc[ring_c[(k + 1) % ring.size()]]].tp, q), chunk));
        }
        if (compact) {
          i64 slow = 0;
          for (i64 x : taus) slow = std::max(slow, x);
          sg.AR = std::max(sg.AR, 2 * (D - 1) * slow);
        } else {
          sg.AR = std::max(sg.AR, ring_sim(taus, (int)(2 * (D - 1))));
        }
      }
      out.push_back(sg);
    }
    return out;
  }

  Plan plan_of(i64 i) const {
    Plan p = decode(i);
    place(p);
    partition(p);
    check_memory(p);
    return p;
  }

  i64 eval(i64 i) const { return eval_mode(i, compact_mode != 0); }
  i64 eval_mode(i64 i, bool compact, i64* T0_out = nullptr) const {
    if (i < 0 || i >= N) return INT64_MIN;
    Plan p = plan_of(i);
    if (p.status) return p.status;
    const auto& cls = p.tpl->cls;
    const int C = (int)cls.size(), b = p.tpl->b;

    // steps 2-4: stage durations (C.5), p2p costs (C.6), 1F1B (C.7).
    // literal: every replica, stage time = the sum over its layers of the
    // layer-op chain.  compact: one pipeline per sub-class (replicas of the
    // class with equal p2p vectors), m = the largest m of its replicas, stage
    // time = l x chain.  owner[c][r] = index of the simulated pipeline that
    // stands for replica r of class c.
    std::vector<SimGroup> G;
    std::vector<std::vector<size_t>> owner(C);
    const bool ep = ep_class(*p.tpl);
    for (int c = 0; c < C; ++c) {
      const int P = (int)cls[c].st.size(), v = vchunks(cls[c]);
      // p2p per boundary: rank pairs q < min(t_s, t_{s+1}) in parallel (A8);
      // V.2 adds the wrap boundary stage P-1 -> stage 0 (last entry)
      auto p2p = [&](const Group& x, int tx, const Group& y, int ty) {
        i64 cs = 0;
        for (int q = 0; q < std::min(tx, ty); ++q) cs = std::max(cs, tau(link_dd(x, tx, q, y, ty, q), act_bytes(b)));
        return cs;
      };
      std::vector<std::vector<i64>> cv(cls[c].D, std::vector<i64>(P > 1 ? P - 1 : 0));
      std::vector<i64> mrep(cls[c].D);
      for (int r = 0; r < cls[c].D; ++r) {
        for (int s = 0; s + 1 < P; ++s)
          cv[r][s] = p2p(p.place[c][r][s], cls[c].st[s].tp, p.place[c][r][s + 1], cls[c].st[s + 1].tp);
        if (v > 1) cv[r].push_back(p2p(p.place[c][r][P - 1], cls[c].st[P - 1].tp, p.place[c][r][0], cls[c].st[0].tp));
        mrep[r] = p.mb[c][r];
      }
      // V.3: the all-to-alls couple the replicas into lockstep -- every replica
      // runs the class's largest micro-batch count and, per boundary, the
      // slowest replica's p2p cost
      std::vector<std::vector<Group>> epg;
      if (ep) {
        std::vector<i64> cmax(cv[0].size(), 0);
        i64 mmax = 0;
        for (int r = 0; r < cls[c].D; ++r) {
          for (size_t k = 0; k < cmax.size(); ++k) cmax[k] = std::max(cmax[k], cv[r][k]);
          mmax = std::max(mmax, mrep[r]);
        }
        for (int r = 0; r < cls[c].D; ++r) { cv[r] = cmax; mrep[r] = mmax; }
        epg.resize(P);
        for (int s = 0; s < P; ++s)
          for (int r = 0; r < cls[c].D; ++r) epg[s].push_back(p.place[c][r][s]);
      }
      owner[c].assign(cls[c].D, 0);
      std::vector<int> rep;  // compact: first replica of each sub-class
      for (int r = 0; r < cls[c].D; ++r) {
        int u = -1;
        if (compact)
          for (int k : rep)
            if (cv[k] == cv[r]) u = k;
        if (u >= 0) {  // replica r joins sub-class of replica u: the pipeline runs the larger m
          const size_t base = owner[c][u];
          owner[c][r] = base;
          for (int s = 0; s < P; ++s) G[base + s].m = std::max(G[base + s].m, (int)mrep[r]);
          continue;
        }
        rep.push_back(r);
        owner[c][r] = G.size();
        for (int s = 0; s < P; ++s) {
          const StageSpec& ss = cls[c].st[s];
          const Group& gr = p.place[c][r][s];
          const std::vector<Group>* eg = ep ? &epg[s] : nullptr;
          SimGroup g{};
          g.P = P; g.s = s; g.m = (int)mrep[r]; g.v = v;
          g.f.assign(v, 0);
          g.g.assign(v, 0);
          for (int k = 0; k < v; ++k) {
            const i64 lk = chunk_layers(p.layers[c][s], v, k);
            if (compact) {
              g.f[k] = lk * layer_chain(ss, gr, b, 0, true, eg);
              g.g[k] = lk * layer_chain(ss, gr, b, 1, true, eg);
              g.lowb = lower_half(lk) * layer_chain(ss, gr, b, 1, true, eg);
            } else {
              for (i64 l = 0; l < lk; ++l) {
                g.f[k] += layer_chain(ss, gr, b, 0, false, eg);
                const i64 gb = layer_chain(ss, gr, b, 1, false, eg);
                g.g[k] += gb;
                if (l < lower_half(lk)) g.lowb += gb;
              }
            }
          }
          if (s == 0) g.lowb += sdur(ss, EMB, true, b);
          // the embedding runs with the first chunk of stage 0, the head with the
          // last chunk of stage P-1
          if (s == 0) { g.f[0] += sdur(ss, EMB, false, b); g.g[0] += sdur(ss, EMB, true, b); }
          if (s == P - 1) { g.f[v - 1] += sdur(ss, HEAD, false, b); g.g[v - 1] += sdur(ss, HEAD, true, b); }
          g.c_prev = s > 0 ? cv[r][s - 1] : 0;
          g.c_next = s + 1 < P ? cv[r][s] : 0;
          g.c_wrap = v > 1 ? cv[r][P - 1] : 0;
          G.push_back(g);
        }
      }
    }
    const i64 T0 = run_pipelines(G);
    if (T0_out) *T0_out = T0;

    // step 5: gradient sync (A19, C.8; S.1 when sync_overlap)
    i64 D = 0;
    for (auto& c : cls) D += c.D;
    if (D == 1) return T0;
    const std::vector<Seg> sg = segments(p, compact);
    const int J = (int)sg.size();
    // FIFO per stage group: free time of stage s of replica r of class c.  In
    // compact mode the replicas of a class share one clock per stage (every
    // segment involves every replica).
    std::vector<std::vector<std::vector<i64>>> freet(C);
    i64 Titer = T0;
    for (int c = 0; c < C; ++c)
      freet[c].assign(compact ? 1 : cls[c].D, std::vector<i64>(cls[c].st.size(), in.sync_overlap ? 0 : T0));
    // S.1: a bucket is ready when its gradients are: the lower one at the end
    // of the group's last backward, the upper one (B.1) that much earlier than
    // the lower bucket's share of that backward (the backward runs head, layers
    // top-down, embedding)
    auto ready = [&](int c, int r, int s, int bk) -> i64 {
      if (!in.sync_overlap) return 0;
      const SimGroup& g = G[owner[c][r] + s];
      return bk ? g.done - g.lowb : g.done;
    };
    auto run_seg = [&](int j) {
      i64 st = 0;
      for (int c = 0; c < C; ++c)
        for (int r = 0; r < cls[c].D; ++r) {
          const int s = sg[j].sc[c];
          st = std::max(st, std::max(ready(c, r, s, sg[j].bk[c]), freet[c][compact ? 0 : r][s]));
        }
      const i64 en = st + sg[j].RS + sg[j].AR;
      for (int c = 0; c < C; ++c)
        for (auto& fr : freet[c]) fr[sg[j].sc[c]] = en;
      Titer = std::max(Titer, en);
    };
    if (!in.sync_overlap) {
      // C.8: barrier at T0, segments in ascending layer order
      for (int j = 0; j < J; ++j) run_seg(j);
    } else {
      // S.1 (Table 1: DP sync is exposed in the backward pass,
      // PAPER.md:100-101): no barrier -- segment j is ready once every group
      // holding its layers, in every replica, has ended its last backward op;
      // segments are issued in descending layer order (the order backward
      // produces gradients), FIFO per group.
      for (int j = J - 1; j >= 0; --j) run_seg(j);
    }
    return Titer;
  }

  // =====================================================================
  // f3 (DESIGN F.1): flow-level contention re-simulation of
  // a candidate's gradient synchronisation.  Every collective step of C.6 /
  // C.8 becomes a set of flows on the rail-only link graph (SPEC.md:340-373
  // build_topology / route / simulate_flows; "bandwidth
  // contention", :400 FCT per flow, :409-412 the slowest flow gates a
  // blocking collective) sharing directed links by progressive-filling
  // max-min fairness.
  //
  // Links (directed, B/ns): per GPU (n, r) an NVLink egress and ingress port
  // (capacity = the fastest intra-node path out of / into it), the PCIe path
  // to its rail NIC and back (the gpu_nic path's beta), and the NIC's wire to
  // the rail switch and back (min(NIC, rail port)); the NVSwitch and the rail
  // fabric are non-blocking.  A flow from (n1, r1) to (n2, r2) uses: same node
  // -> egress(n1,r1), ingress(n1,r2); other node, same rank -> pcie_up, nic_tx
  // at (n1,r1), nic_rx, pcie_dn at (n2,r1); other node and rank (Fig 2 (c))
  // -> egress(n1,r1), ingress(n1,r2), then the rail path of rank r2.  Its own
  // path caps it at the alpha-beta link's beta (a private link), and its fixed
  // latency is the link's alpha.
  //
  // Rates: progressive filling over the active flows -- share_e = residual_e
  // / (unfrozen flows on e) (one IEEE division); s = min over links with
  // unfrozen flows and over unfrozen flows' private caps; every unfrozen flow
  // on an argmin link, or whose cap equals s, is frozen at rate s; each link's
  // residual -= (number of flows frozen on it) x s; repeat.
  // Time (integer ns): each active flow's time to drain d_f = max(0,
  // ceil(rem_f / rate_f)); the next drain event is t + min d_f; at an event
  // every flow with d_f == the minimum finishes (drain end = that time),
  // every other flow keeps rem_f - rate_f x delta.  A flow's completion =
  // drain end + alpha; FCT = completion - arrival.  Without contention a flow
  // drains in ceilq(bytes, beta), so its FCT is the alpha-beta tau exactly.
  //
  // Schedule: C.8 (barrier at T0, segments FIFO per stage group in ascending
  // layer order).  A segment is a sequence of synchronous steps -- the
  // reshard step (when some class has tp != t*: every group with tp != t*
  // sends ceil(S/t*) bytes over each of its TP-ring edges) and the 2(D-1)
  // ring steps (for each ring q < t*, every ring position sends the chunk to
  // the next) -- and a step's flows all arrive when the previous step's last
  // flow completes (the blocking collective).  A segment starts when
  // the previous segment of each of its groups has completed.  Output, time
  // relative to T0: sync_ab (the same schedule with every step lasting its
  // slowest flow's tau: the C.8 extra T_iter - T0) and sync_flow (the flow
  // level schedule), plus every flow's FCT.
  // =====================================================================
  struct FFlow {
    i64 bytes, alpha, arrive;
    double cap, rem, rate;
    int link[6], nl;
    int step;       // global step id
  };
  struct FStep {
    int seg, k;     // segment, index within it
    std::vector<std::array<int, 4>> pairs;  // (n1, r1, n2, r2)
    i64 bytes;
  };

  int gpn0() const { return cl.gpn[0]; }
  int lid(int kind, int n, int r) const { return ((n * gpn0() + r) * 6) + kind; }  // 0 eg 1 in 2 up 3 dn 4 tx 5 rx
  std::vector<double> ext_linkcap;  // orc_flow_sim only: explicit link capacities
  double link_cap(int id) const {
    if (!ext_linkcap.empty()) return ext_linkcap[id];
    const int kind = id % 6, g = id / 6, n = g / gpn0(), r = g % gpn0();
    const orc_type& t = T(n);
    const i64 fr = in.frame_bytes;
    if (kind <= 1) {
      double c = 0;
      for (int j = 0; j < t.gpus_per_node; ++j)
        if (j != r) c = std::max(c, path_link(t.link_kind[kind == 0 ? t.intra_kind[r][j] : t.intra_kind[j][r]], fr).beta);
      return c;
    }
    if (kind <= 3) return path_link(t.gpu_nic, fr).beta;
    return std::min(t.nic_gbps / 8.0, in.rail_gbps / 8.0);
  }
  const orc_type& T(int n) const { return types[node_type[n]]; }
  FFlow make_flow(int n1, int r1, int n2, int r2, i64 bytes) const {
    FFlow f{};
    const Link l = cl.gpu_to_gpu(n1, r1, n2, r2);
    f.bytes = bytes;
    f.alpha = l.alpha;
    f.cap = l.beta;
    f.rem = (double)bytes;
    f.nl = 0;
    if (n1 == n2) {
      f.link[f.nl++] = lid(0, n1, r1);
      f.link[f.nl++] = lid(1, n1, r2);
    } else {
      if (r1 != r2) {
        f.link[f.nl++] = lid(0, n1, r1);
        f.link[f.nl++] = lid(1, n1, r2);
      }
      f.link[f.nl++] = lid(2, n1, r2);
      f.link[f.nl++] = lid(4, n1, r2);
      f.link[f.nl++] = lid(5, n2, r2);
      f.link[f.nl++] = lid(3, n2, r2);
    }
    return f;
  }

  // progressive filling (maxmin_fill) over the flows in `act`
  void maxmin(std::vector<FFlow>& fl, const std::vector<int>& act) const {
    std::vector<std::vector<int>> inc(act.size());
    std::map<int, double> cap_of;
    std::vector<double> cap(act.size()), rate;
    for (size_t k = 0; k < act.size(); ++k) {
      const FFlow& f = fl[act[k]];
      inc[k].assign(f.link, f.link + f.nl);
      for (int e : inc[k])
        if (!cap_of.count(e)) cap_of[e] = link_cap(e);
      cap[k] = f.cap;
    }
    maxmin_fill((int)act.size(), inc, cap_of, cap, rate);
    for (size_t k = 0; k < act.size(); ++k) fl[act[k]].rate = rate[k];
  }

  // The fluid event engine: active flows drain at their max-min rates; timers
  // (time, seq, tag) fire callbacks that may add flows.  At each step the
  // earlier of the next drain completion and the next timer is processed; on
  // a tie drains go first.  on_done(flow, completion) with completion = drain
  // end + alpha; on_timer(tag, now).
  struct FlowEngine {
    const Oracle* o;
    std::vector<FFlow> fl;
    std::vector<int> act;
    std::priority_queue<std::tuple<i64, i64, int>, std::vector<std::tuple<i64, i64, int>>, std::greater<>> tm;
    i64 t = 0, seq = 0;
    bool dirty = true;
    void add(FFlow f, i64 now) {
      f.arrive = now;
      f.rem = (double)f.bytes;
      act.push_back((int)fl.size());
      fl.push_back(f);
      dirty = true;
    }
    void timer(i64 when, int tag) { tm.push({when, seq++, tag}); }
    template <typename OnDone, typename OnTimer>
    void run(OnDone on_done, OnTimer on_timer) {
      while (!act.empty() || !tm.empty()) {
        if (dirty && !act.empty()) o->maxmin(fl, act);
        dirty = false;
        i64 dmin = INT64_MAX;
        std::vector<i64> d(act.size());
        for (size_t k = 0; k < act.size(); ++k) {
          const FFlow& f = fl[act[k]];
          d[k] = f.rem <= 0 ? 0 : (i64)std::ceil(f.rem / f.rate);
          dmin = std::min(dmin, d[k]);
        }
        const i64 t_drain = act.empty() ? INT64_MAX : t + dmin;
        const i64 t_ev = tm.empty() ? INT64_MAX : std::get<0>(tm.top());
        if (t_drain <= t_ev) {
          const double delta = (double)dmin;
          std::vector<int> keep, done;
          for (size_t k = 0; k < act.size(); ++k) {
            FFlow& f = fl[act[k]];
            if (d[k] == dmin) {
              done.push_back(act[k]);
            } else {
              f.rem = f.rem - f.rate * delta;
              keep.push_back(act[k]);
            }
          }
          act.swap(keep);
          t = t_drain;
          dirty = true;
          for (int x : done) on_done(fl[x], t + fl[x].alpha);
        } else {
          const double delta = (double)(t_ev - t);
          for (int x : act) fl[x].rem = fl[x].rem - fl[x].rate * delta;
          t = t_ev;
          dirty = true;
          while (!tm.empty() && std::get<0>(tm.top()) == t) {
            const int tag = std::get<2>(tm.top());
            tm.pop();
            on_timer(tag, t);
          }
        }
      }
    }
  };

  // f3 for candidate i: returns status (0 ok, < 0 invalid); sync_ab, sync_flow
  // relative to T0; fcts appended in completion order
  int flow_resim(i64 i, i64& sync_ab, i64& sync_flow, std::vector<i64>& fcts) const {
    sync_ab = sync_flow = 0;
    if (i < 0 || i >= N) return INT32_MIN;
    Plan p = plan_of(i);
    if (p.status) return p.status;
    const auto& cls = p.tpl->cls;
    const int C = (int)cls.size();
    i64 D = 0;
    for (auto& c : cls) D += c.D;
    if (D == 1) return 0;
    const std::vector<Seg> sg = segments(p, false);
    const int J = (int)sg.size();
    // the steps of every segment
    std::vector<FStep> steps;
    std::vector<int> seg_first(J), seg_n(J);
    for (int j = 0; j < J; ++j) {
      seg_first[j] = (int)steps.size();
      const i64 xs = ceil_div(sg[j].S, sg[j].tstar);
      FStep rs{j, 0, {}, xs};
      for (int c = 0; c < C; ++c) {
        const int s = sg[j].sc[c], tp = cls[c].st[s].tp;
        if (tp == sg[j].tstar) continue;
        for (int r = 0; r < cls[c].D; ++r) {
          const Group& g = p.place[c][r][s];
          for (int q = 0; q < tp; ++q) {
            const auto x = dev(g, tp, q), y = dev(g, tp, (q + 1) % tp);
            rs.pairs.push_back({x.first, x.second, y.first, y.second});
          }
        }
      }
      if (!rs.pairs.empty()) steps.push_back(rs);
      std::vector<Group> ring;
      std::vector<int> rtp;
      for (int c = 0; c < C; ++c)
        for (int r = 0; r < cls[c].D; ++r) {
          ring.push_back(p.place[c][r][sg[j].sc[c]]);
          rtp.push_back(cls[c].st[sg[j].sc[c]].tp);
        }
      FStep st{j, 0, {}, ceil_div(xs, D)};
      for (int q = 0; q < sg[j].tstar; ++q)
        for (size_t k = 0; k < ring.size(); ++k) {
          const Group& u = ring[k];
          const Group& v = ring[(k + 1) % ring.size()];
          const size_t k2 = (k + 1) % ring.size();
          const auto x = dev(u, rtp[k], q), y = dev(v, rtp[k2], q);
          st.pairs.push_back({x.first, x.second, y.first, y.second});
        }
      for (i64 k = 0; k < 2 * (D - 1); ++k) steps.push_back(st);
      seg_n[j] = (int)steps.size() - seg_first[j];
      for (int k = 0; k < seg_n[j]; ++k) steps[seg_first[j] + k].k = k;
    }
    // FIFO predecessors: the previous segment on each of its groups (every
    // segment involves every replica of every class, so a group is (c, stage))
    std::vector<std::vector<int>> preds(J);
    for (int j = 0; j < J; ++j)
      for (int jj = j - 1; jj >= 0; --jj) {
        bool share = false;
        for (int c = 0; c < C; ++c) share |= sg[jj].sc[c] == sg[j].sc[c];
        if (share) {
          bool already = false;
          for (int x : preds[j]) already |= x == jj;
          if (!already) preds[j].push_back(jj);
        }
      }
    // alpha-beta schedule: a step lasts its slowest flow's tau
    {
      std::vector<i64> end(J, 0);
      for (int j = 0; j < J; ++j) {
        i64 t = 0;
        for (int x : preds[j]) t = std::max(t, end[x]);
        for (int k = 0; k < seg_n[j]; ++k) {
          const FStep& st = steps[seg_first[j] + k];
          i64 m = 0;
          for (auto& pr : st.pairs) m = std::max(m, tau(cl.gpu_to_gpu(pr[0], pr[1], pr[2], pr[3]), st.bytes));
          t += m;
        }
        end[j] = t;
        sync_ab = std::max(sync_ab, t);
      }
    }
    // flow level
    std::vector<int> pending(steps.size(), 0);
    std::vector<i64> step_done(steps.size(), 0);
    std::vector<int> waiting(J, 0);  // unfinished predecessors
    for (int j = 0; j < J; ++j) waiting[j] = (int)preds[j].size();
    FlowEngine E{this};
    auto start_step = [&](int id, i64 now) {
      for (auto& pr : steps[id].pairs) {
        FFlow f = make_flow(pr[0], pr[1], pr[2], pr[3], steps[id].bytes);
        f.step = id;
        E.add(f, now);
      }
      pending[id] = (int)steps[id].pairs.size();
    };
    for (int j = 0; j < J; ++j)
      if (!waiting[j]) start_step(seg_first[j], 0);
    E.run(
        [&](const FFlow& f, i64 done) {  // a flow completed: its step ends with its last flow
          fcts.push_back(done - f.arrive);
          step_done[f.step] = std::max(step_done[f.step], done);
          if (--pending[f.step] == 0) E.timer(step_done[f.step], f.step);
        },
        [&](int id, i64 now) {  // a step completed at `now`
          const int j = steps[id].seg;
          if (steps[id].k + 1 < seg_n[j]) {
            start_step(id + 1, now);
            return;
          }
          sync_flow = std::max(sync_flow, now);
          for (int jj = j + 1; jj < J; ++jj) {
            bool dep = false;
            for (int x : preds[jj]) dep |= x == j;
            if (dep && --waiting[jj] == 0) start_step(seg_first[jj], now);
          }
        });
    return 0;
  }
};

thread_local std::string g_err;

}  // namespace

// ----------------------------------------------------------------------------
// C API for oracle/oracle.py (ctypes)
// ----------------------------------------------------------------------------
extern "C" {

const char* orc_last_error() { return g_err.c_str(); }

void* orc_create(const orc_input* in) {
  g_err.clear();
  if (!in || in->n_types < 1 || in->n_types > 8 || in->n_nodes < 1 || in->B < 1 || in->L < 1) {
    g_err = "invalid input";
    return nullptr;
  }
  if (in->interleave < 1 || in->interleave > 8) {
    g_err = "interleave must be 1..8";
    return nullptr;
  }
  if (in->mem_check && (in->interleave > 1 || in->ep_dp || in->mixtp)) {
    g_err = "mem_check is not defined with interleave / ep_dp / mixtp (DESIGN V.1-V.3)";
    return nullptr;
  }
  if (in->sync_buckets < 0 || in->sync_buckets > 2 || (in->sync_buckets == 2 && in->interleave > 1)) {
    g_err = "sync_buckets must be 0..2 and is not defined with interleave (DESIGN B.1)";
    return nullptr;
  }
  if (in->ep_dp && in->mixtp) {
    g_err = "ep_dp is not defined with mixtp (DESIGN V.1)";
    return nullptr;
  }
  Oracle* o = new Oracle();
  o->in = *in;
  o->types.assign(in->types, in->types + in->n_types);
  o->node_type.assign(in->node_type, in->node_type + in->n_nodes);
  o->init();
  return o;
}
void orc_destroy(void* h) { delete (Oracle*)h; }
i64 orc_space_size(void* h) { return ((Oracle*)h)->N; }
i64 orc_n_templates(void* h) { return (i64)((Oracle*)h)->tpls.size(); }
i64 orc_template_prefix(void* h, i64 k) {
  Oracle* o = (Oracle*)h;
  if (k < 0 || k > (i64)o->tpls.size()) return -1;
  return k == (i64)o->tpls.size() ? o->N : o->tpls[k].prefix;
}
i64 orc_eval(void* h, i64 i) { return ((Oracle*)h)->eval(i); }
// 0 = literal (default), 1 = compact (header comment)
void orc_set_compact(void* h, int compact) { ((Oracle*)h)->compact_mode = compact ? 1 : 0; }

// Evaluates idx[0..n) (or the range [first, first+n) if idx == NULL) on
// `threads` host threads.
void orc_eval_many(void* h, const i64* idx, i64 first, i64 n, i64* out, int threads) {
  Oracle* o = (Oracle*)h;
  if (threads < 1) threads = 1;
  std::atomic<i64> next{0};
  auto work = [&]() {
    for (;;) {
      i64 k = next.fetch_add(4);  // small grabs: per-candidate cost varies ~1000x
      if (k >= n) return;
      for (i64 t = k; t < std::min(n, k + 4); ++t) out[t] = o->eval(idx ? idx[t] : first + t);
    }
  };
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) pool.emplace_back(work);
  for (auto& t : pool) t.join();
}

// Human-readable plan (for tests / debugging): template, layers, micro-batches, placement.
int orc_describe(void* h, i64 i, char* buf, int cap) {
  Oracle* o = (Oracle*)h;
  if (i < 0 || i >= o->N) return -1;
  Plan p = o->decode(i);
  o->place(p);
  o->partition(p);
  o->check_memory(p);
  std::string s = "{\"b\":" + std::to_string(p.tpl->b) + ",\"status\":" + std::to_string(p.status) + ",\"classes\":[";
  for (size_t c = 0; c < p.tpl->cls.size(); ++c) {
    const ClassSpec& cs = p.tpl->cls[c];
    s += c ? ",{" : "{";
    s += "\"D\":" + std::to_string(cs.D) + ",\"stages\":[";
    for (size_t k = 0; k < cs.st.size(); ++k)
      s += (k ? ",[" : "[") + std::to_string(cs.st[k].type) + "," + std::to_string(cs.st[k].tp) +
           (cs.st[k].type2 >= 0 ? "," + std::to_string(cs.st[k].type2) : std::string()) + "]";
    s += "],\"layers\":[";
    for (size_t k = 0; k < p.layers[c].size(); ++k) s += (k ? "," : "") + std::to_string(p.layers[c][k]);
    s += "],\"mb\":[";
    if (c < p.mb.size())
      for (size_t k = 0; k < p.mb[c].size(); ++k) s += (k ? "," : "") + std::to_string(p.mb[c][k]);
    s += "],\"place\":[";
    for (size_t r = 0; r < p.place[c].size(); ++r) {
      s += r ? ",[" : "[";
      for (size_t k = 0; k < p.place[c][r].size(); ++k)
        s += (k ? ",[" : "[") + std::to_string(p.place[c][r][k].node) + "," + std::to_string(p.place[c][r][k].base) +
             (p.place[c][r][k].node2 >= 0 ? "," + std::to_string(p.place[c][r][k].node2) : std::string()) + "]";
      s += "]";
    }
    s += "]}";
  }
  s += "]}";
  if ((int)s.size() + 1 > cap) return (int)s.size() + 1;
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return 0;
}

// --- building blocks exposed for the pin tests -------------------------------
// DESIGN M.1: bytes needed on one device of stage s (of P) with l layers, m micro-batches
i64 orc_device_bytes(void* h, int type, int tp, int P, int s, i64 l, i64 m, int b) {
  return ((Oracle*)h)->device_bytes(StageSpec{type, tp}, P, s, l, m, b);
}
// per-hop delay before rounding: frame*8 / uni Gbps
double orc_hop_delay_exact(double gbps, int bidir, i64 frame) {
  orc_hop hp{gbps, bidir, 0};
  return (double)(frame * 8) / uni_gbps(hp);
}
i64 orc_ring_sim(const i64* tau_edges, int n, int steps) {
  return ring_sim(std::vector<i64>(tau_edges, tau_edges + n), steps);
}
// V.2: one interleaved pipeline (P stages, v chunks, m micro-batches): f, g
// [P][v] row-major, c[P-1] boundary costs, cw the wrap cost
i64 orc_pipeline_ilv(int P, int v, int m, const i64* f, const i64* g, const i64* c, i64 cw) {
  std::vector<Oracle::SimGroup> G(P);
  for (int s = 0; s < P; ++s) {
    G[s].P = P; G[s].s = s; G[s].m = m; G[s].v = v;
    G[s].f.assign(f + s * v, f + s * v + v);
    G[s].g.assign(g + s * v, g + s * v + v);
    G[s].c_prev = s > 0 ? c[s - 1] : 0;
    G[s].c_next = s + 1 < P ? c[s] : 0;
    G[s].c_wrap = cw;
  }
  return Oracle::run_pipelines(G);
}
// V.2 op order of stage s: out[3 x n] = (fwd, chunk, micro-batch); returns n
int orc_op_order(int P, int s, int m, int v, int* out, int cap) {
  auto o = Oracle::op_order(P, s, m, v);
  for (size_t k = 0; k < o.size() && (int)k < cap; ++k) {
    out[3 * k] = o[k].fwd;
    out[3 * k + 1] = o[k].k;
    out[3 * k + 2] = o[k].j;
  }
  return (int)o.size();
}
// V.3: all-to-all over the union of groups (node, base) x n of TP t at micro-batch b
i64 orc_ep_alltoall_groups(void* h, const int* nodes, const int* bases, int n, int t, int b) {
  std::vector<Group> gs;
  for (int k = 0; k < n; ++k) gs.push_back(Group{nodes[k], bases[k]});
  return ((Oracle*)h)->ep_alltoall_x(gs, t, b);
}

// one pipeline (P stages, m micro-batches) through the event engine
i64 orc_pipeline(int P, int m, const i64* f, const i64* g, const i64* c) {
  std::vector<Oracle::SimGroup> G(P);
  for (int s = 0; s < P; ++s) {
    G[s].P = P; G[s].s = s; G[s].m = m; G[s].f = {f[s]}; G[s].g = {g[s]};
    G[s].c_prev = s > 0 ? c[s - 1] : 0;
    G[s].c_next = s + 1 < P ? c[s] : 0;
  }
  return Oracle::run_pipelines(G);
}
void orc_hamilton(i64 n, const i64* w, int k, i64* out) {
  std::vector<i64> q = hamilton(n, std::vector<i64>(w, w + k));
  for (int i = 0; i < k; ++i) out[i] = q[i];
}
// per-device FLOPs/bytes/duration of one op on device type `type` with TP t
void orc_op(void* h, int type, int kind, int bwd, int t, int b, i64* flop, i64* bytes, i64* dur) {
  Oracle* o = (Oracle*)h;
  Cost c = op_cost(o->in, kind, t, b);
  *flop = c.flop * (bwd ? 2 : 1);
  *bytes = c.bytes * (bwd ? 2 : 1);
  *dur = op_dur(o->in, o->types[type], kind, bwd != 0, t, b);
}
// gradient bytes of a sync segment of `n_layers` layers (C.6); Table 1 pin
i64 orc_segment_bytes(void* h, i64 n_layers, int has_first, int has_last) {
  const orc_input& in = ((Oracle*)h)->in;
  const i64 hkv = in.kv_heads * in.h / in.heads;
  const i64 Wlayer = in.h * (2 * in.h + 2 * hkv) + in.nm * in.h * in.ffn * in.E + (in.E > 1 ? in.h * in.E : 0) + 2 * in.h;
  i64 S = n_layers * Wlayer * in.bpe_grad;
  if (has_first) S += in.V * in.h * in.bpe_grad;
  if (has_last) S += (in.V * in.h * (in.tied ? 0 : 1) + in.h) * in.bpe_grad;
  return S;
}
// TP all-reduce (A16) of a stage group (node, base, tp) at micro-batch size b:
// literal ring; EP all-to-all (A17) of the same group
i64 orc_tp_allreduce(void* h, int node, int base, int tp, int b) {
  return ((Oracle*)h)->tp_allreduce(Group{node, base}, tp, b);
}
i64 orc_ep_alltoall(void* h, int node, int base, int tp, int b) {
  return ((Oracle*)h)->ep_alltoall(Group{node, base}, tp, b);
}
// gradient-sync segments of candidate i (C.6): per segment a, z, S, t*, RS, AR
// (6 int64 each, literal mode); returns J, or -J - 1 if cap is too small, or
// the candidate's negative status
int orc_segments(void* h, i64 i, i64* out, int cap) {
  Oracle* o = (Oracle*)h;
  if (i < 0 || i >= o->N) return INT32_MIN;
  Plan p = o->plan_of(i);
  if (p.status) return p.status;
  const auto sg = o->segments(p, false);
  if ((int)sg.size() > cap) return -(int)sg.size() - 1;
  for (size_t j = 0; j < sg.size(); ++j) {
    i64* r = out + 6 * j;
    r[0] = sg[j].a; r[1] = sg[j].z; r[2] = sg[j].S; r[3] = sg[j].tstar; r[4] = sg[j].RS; r[5] = sg[j].AR;
  }
  return (int)sg.size();
}
// Resharding decision (§2 "Resharding"): the synchronisation
// of a source and a destination DP group needs resharding iff (1) their
// micro-batch sizes differ or (2) their TP degrees differ; communication that
// is pipeline-sequential (PP only) never does.  Cost model: condition (2) is
// the reshard term RS of C.6 / A14; condition (1) is flagged only (A15).
int orc_needs_reshard(int src_tp, int src_mb, int dst_tp, int dst_mb, int pp_only) {
  if (pp_only) return 0;
  return (src_mb != dst_mb || src_tp != dst_tp) ? 1 : 0;
}
// f3 (DESIGN F.1): out = {status, sync_ab, sync_flow, n_flows, T0, T_iter}; fct (may be
// NULL) receives up to cap FCTs in completion order
void orc_flow_resim(void* h, i64 i, i64* out, i64* fct, i64 cap) {
  i64 ab = 0, fw = 0, T0 = 0;
  std::vector<i64> f;
  const int st = ((Oracle*)h)->flow_resim(i, ab, fw, f);
  const i64 T = st ? st : ((Oracle*)h)->eval_mode(i, true, &T0);
  out[0] = st; out[1] = ab; out[2] = fw; out[3] = (i64)f.size(); out[4] = st ? 0 : T0; out[5] = T;
  if (fct)
    for (i64 k = 0; k < std::min<i64>(cap, (i64)f.size()); ++k) fct[k] = f[k];
}
// f3 building block: independent flows through the same fluid engine.  Flow f
// arrives at arrive[f] with bytes[f], fixed latency alpha[f], private cap
// cap[f] and links inc[f * maxl + q] (q < nfl[f]) of capacity linkcap[e];
// completion times (drain end + alpha) out.
void orc_flow_sim(void* h, int nf, const double* linkcap, const int* nfl, const int* inc, int maxl, const i64* arrive,
                  const i64* bytes, const i64* alpha, const double* cap, i64* done) {
  Oracle* o = (Oracle*)h;
  o->ext_linkcap.assign(linkcap, linkcap + [&] { int m = 0; for (int f = 0; f < nf; ++f) for (int q = 0; q < nfl[f]; ++q) m = std::max(m, inc[f * maxl + q] + 1); return m; }());
  Oracle::FlowEngine E{o};
  std::vector<Oracle::FFlow> fs(nf);
  for (int f = 0; f < nf; ++f) {
    Oracle::FFlow x{};
    x.bytes = bytes[f];
    x.alpha = alpha[f];
    x.cap = cap[f];
    x.nl = nfl[f];
    for (int q = 0; q < nfl[f]; ++q) x.link[q] = inc[f * maxl + q];
    x.step = f;
    fs[f] = x;
    E.timer(arrive[f], f);
  }
  E.run([&](const Oracle::FFlow& x, i64 t) { done[x.step] = t; }, [&](int f, i64 now) { E.add(fs[f], now); });
  o->ext_linkcap.clear();
}
// f3 building block for the max-min pins: nf flows over nl links; flow f
// uses the links inc[f * maxl + q] (q < nfl[f], -1 padded); per-flow cap;
// rates out (progressive filling as in Oracle::maxmin, capacities given)
void orc_maxmin(int nf, int nl, const double* linkcap, const int* nfl, const int* inc, int maxl, const double* cap,
                double* rate) {
  std::vector<std::vector<int>> I(nf);
  std::map<int, double> lc;
  for (int e = 0; e < nl; ++e) lc[e] = linkcap[e];
  for (int f = 0; f < nf; ++f) I[f].assign(inc + f * maxl, inc + f * maxl + nfl[f]);
  std::vector<double> r;
  maxmin_fill(nf, I, lc, std::vector<double>(cap, cap + nf), r);
  for (int f = 0; f < nf; ++f) rate[f] = r[f];
}
i64 orc_act_bytes(void* h, int b) { return ((Oracle*)h)->act_bytes(b); }
// link between two GPUs (node, local rank) -> alpha, beta
void orc_link(void* h, int n1, int r1, int n2, int r2, i64* alpha, double* beta) {
  Oracle* o = (Oracle*)h;
  Link l = o->cl.gpu_to_gpu(n1, r1, n2, r2);
  *alpha = l.alpha;
  *beta = l.beta;
}
}
