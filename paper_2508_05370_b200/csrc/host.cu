// host.cu — C-ABI host side of libhsim (include/hsim.h).
//
// hsim_create validates the three descriptions, derives
// link delays from Table-4-style fields, per-op roofline
// durations (DESIGN.md C.5), enumerates the candidate templates (C.2), places
// each class (C.3), derives its base layer split, p2p costs, sub-classes and
// link-class masks (C.4, C.6, A13), and uploads everything to the device.  The
// per-candidate work (decode digits, partition, stage sums, 1F1B, sync,
// top-k) runs only in the CUDA kernels (kernels.cu).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "hsim.h"
#include "hsim_core.cuh"

using namespace hsim;

namespace {
thread_local std::string g_err;

struct Fail {
  int code;
  std::string msg;
};
[[noreturn]] void fail(int code, const std::string& m) { throw Fail{code, m}; }

constexpr i64 TWO53 = (i64)1 << 53;

double uni(const hsim_hop& h) { return h.bidir ? h.gbps / 2.0 : h.gbps; }

// alpha = sum of per-hop ceil(frame*8 / uni Gbps) (A9); beta = slowest hop, B/ns
Link path_link(const hsim_path& p, i64 frame) {
  Link l{0, 1e300};
  for (int k = 0; k < p.n_hops; ++k) {
    const double u = uni(p.hops[k]);
    l.alpha += ceilq(frame * 8, u);
    l.beta = std::min(l.beta, u / 8.0);
  }
  return l;
}
Link cat(const Link& a, const Link& b) { return Link{a.alpha + b.alpha, std::min(a.beta, b.beta)}; }
i64 tau(const Link& e, i64 x) { return e.alpha + ceilq(x, e.beta); }

// A stage of a class is (type code, tp); the code carries a V.1 mixed group's
// second type: code = type | (type2 + 1) << 8 (type2 = -1: homogeneous)
int st_t(int code) { return code & 255; }
int st_t2(int code) { return (code >> 8) - 1; }
int st_code(int t, int t2) { return t | (t2 + 1) << 8; }
// a placed stage group: tp GPUs from base on node; V.1: tp/2 from base on node
// and tp/2 from base on node2
struct GPl { int node, base, node2; };
std::pair<int, int> gdev(const GPl& g, int tp, int q) {
  if (g.node2 < 0) return {g.node, g.base + q};
  return q < tp / 2 ? std::make_pair(g.node, g.base + q) : std::make_pair(g.node2, g.base + q - tp / 2);
}

i64 hamilton_floor_rem(i64 n, i64 w, i64 W, i64* rem) {
  *rem = n * w % W;
  return n * w / W;
}

}  // namespace

struct hsim_handle {
  // copies of the descriptions
  hsim_cluster_desc cd{};
  hsim_model_desc md{};
  std::vector<hsim_device_type> types;
  std::vector<int32_t> node_type;
  int nt = 0;
  // derived (host)
  Link intra[MAXT][MAXG][MAXG];
  Link rail[MAXT][MAXT];
  std::map<std::pair<i64, u64>, int> lc_id;
  std::vector<Link> lcs;
  std::vector<int> bs;                         // sorted micro-batch sizes
  // durations [type][lg tp][b index]
  struct Dur { i64 attn_f, attn_b, mlp_f, mlp_b, emb_f, emb_b, head_f, head_b, ar, a2a; bool ok; };
  std::vector<Dur> dur;
  Dur& dur_at(int t, int lg, int bi) { return dur[((size_t)t * 4 + lg) * bs.size() + bi]; }
  u64 tp_mask[MAXT][4];
  // templates
  std::vector<i64> prefix;
  std::vector<int32_t> bucket;
  std::vector<i64> cprefix;
  std::vector<int32_t> cbucket;
  std::vector<TplRec> tpl;
  std::vector<i64> pool;
  std::map<std::vector<int>, int32_t> crec_of;
  std::vector<std::vector<int>> nodes_of_type;
  i64 n_of_type[MAXT] = {0, 0, 0, 0};
  uint32_t pmask_all = 0;   // union of template depth masks (which depth kernels to launch)
  i64 layer_fb_max = 0, ext_max = 0, c_max = 0;  // bound of every 1F1B time (fp64-exact pipelines, < 2^52)
  int depth_max = 0;
  int stages_max = 0;       // max over templates of the stages of all classes (S.1 scratch rows)
  int pcnt_max[FASTP + 1] = {0};  // max #classes of depth P in one template (job-list capacity)
  int ilv = 1;              // V.2: model chunks per stage (1 = non-interleaved)
  int ilv_jobs_max = 0;     // V.2: max #classes with P >= 2 in one template (K_ilv job-list capacity)
  int ilv_depth_max = 0;    // V.2: deepest interleaved pipeline
  i64 depth_jobs_space[FASTP + 1] = {0};  // class-jobs of depth P over the whole space
  i64 N = 0;
  Tables hT{};  // host pointers (for hsim_decode)
  // device
  Tables* dT = nullptr;
  i64* d_prefix = nullptr;
  int32_t* d_bucket = nullptr;
  i64* d_cprefix = nullptr;
  int32_t* d_cbucket = nullptr;
  static constexpr int NPLAN = 4;   // ring of pinned chunk-plan staging buffers (block-cyclic lists)
  i64* h_plan[NPLAN] = {};
  size_t h_plan_cap[NPLAN] = {};
  int plan_slot = 0;
  cudaEvent_t ev_plan[NPLAN] = {};
  cudaEvent_t ev_done = nullptr;  // end of the last call's work (orders calls made on different streams)
  bool done_recorded = false;
  int grid_cache[64] = {};        // resident blocks per SM per kernel (kernels.cu), per handle
  u64* d_xmask = nullptr;
  std::vector<u64> xmask_cross, xmask_same;
  i64* d_work = nullptr;      // work counter + per-range plan (kernels.cu)
  size_t work_cap = 0;
  TplRec* d_tpl = nullptr;
  i64* d_pool = nullptr;
  std::vector<i64> wtab;      // partition weight table (host build, device copy)
  i64* d_wtab = nullptr;
  int8_t* d_node_type = nullptr;
  std::vector<int8_t> node_type8;
  std::vector<int32_t> type_nodes;   // f3: node ids grouped by type
  int32_t* d_type_nodes = nullptr;
  // top-k scratch
  i64* d_blk = nullptr;
  size_t blk_cap = 0;
  i64* d_cells = nullptr;
  i64* d_sync_units = nullptr;  // the last top-k call's synced-segment counter (pruned K_final), or nullptr
  void* d_flow = nullptr;     // f3 scratch (flow.cu)
  size_t flow_cap = 0;
  static constexpr int NSIDE = 22, NEV = 48;  // sides 20, 21: K_pipe_multi<1,8>, <9,16>
  cudaStream_t side[NSIDE] = {};     // one stream per phase-kernel type + the final stream
  cudaEvent_t ev_fork = nullptr, ev_join[NSIDE] = {}, ev_pool[NEV] = {};
  int32_t last_launches = 0;
  int prune = 1;                // hsim_set_prune: the top-k sweep's pruned sync (default on)
  int dedup = 1;                // hsim_set_dedup: one 1F1B run per distinct class pipeline (default on)
  int cmax = 1;                 // max classes of a template
  i64 m_max = 0;                // max micro-batches of a template (dedupe key width)
  u32 pw_max = 1;               // max digit radix of a class record
  int u_max = 1;                // max sub-classes of a class record
  u64* d_hkeys[2] = {};         // dedupe hash tables (per scratch buffer): keys, results
  i64* d_hres[2] = {};
  size_t hash_cap[2] = {};
  int sm_count = 148;

  Link link(int n1, int r1, int n2, int r2) const {
    const int t1 = node_type[n1], t2 = node_type[n2];
    if (n1 == n2) return intra[t1][r1][r2];
    if (r1 == r2) return rail[t1][t2];               // Fig 2 (b)
    return cat(intra[t1][r1][r2], rail[t1][t2]);     // Fig 2 (c): NVLink hop at the source first
  }
  int lc(const Link& l) {
    u64 bits;
    std::memcpy(&bits, &l.beta, 8);
    auto key = std::make_pair(l.alpha, bits);
    auto it = lc_id.find(key);
    if (it != lc_id.end()) return it->second;
    if ((int)lcs.size() >= MAXLC) fail(HSIM_ERANGE, "more than 64 distinct link classes");
    int id = (int)lcs.size();
    lc_id[key] = id;
    lcs.push_back(l);
    return id;
  }

  void validate();
  void derive_links();
  void derive_durations();
  void enumerate();
  int32_t crec(int b_idx, int M, int D, const std::vector<std::pair<int, int>>& stages, bool ep);
  i64 moe_dur(int t, int tp, i64 b, i64 g, bool bwd) const;
  i64 a2a_groups(const std::vector<std::pair<int, int>>& groups, int tp, i64 b) const;
  std::vector<std::vector<GPl>> place(int D, const std::vector<std::pair<int, int>>& stages) const;
  Link dlink(const GPl& a, int ta, int qa, const GPl& z, int tz, int qz) const {
    const auto x = gdev(a, ta, qa), y = gdev(z, tz, qz);
    return link(x.first, x.second, y.first, y.second);
  }
  void prepare();
  void upload();
  int ensure_device() {
    if (dT) return HSIM_OK;
    try {
      upload();
    } catch (const Fail& f) {
      g_err = f.msg;
      return f.code;
    }
    return HSIM_OK;
  }
};

// ------------------------------------------------------------------------------
void hsim_handle::validate() {
  const hsim_cluster_desc& c = cd;
  const hsim_model_desc& m = md;
  if (c.n_device_types < 1 || c.n_device_types > MAXT) fail(HSIM_EINVAL, "InvalidValue: n_device_types must be 1..4");
  if (c.n_nodes < 1 || c.n_nodes > 4096) fail(HSIM_EINVAL, "InvalidValue: n_nodes must be 1..4096");
  if (!c.device_types || !c.node_type_of) fail(HSIM_EINVAL, "MissingField: device_types / node_type_of");
  if (c.frame_bytes < 1 || c.rail_alpha_ns < 0) fail(HSIM_EINVAL, "InvalidValue: frame_bytes / rail_alpha_ns");
  if (!(c.rail_gbps > 0)) fail(HSIM_EINVAL, "NonPositiveBandwidth: rail_gbps");
  for (int t = 0; t < c.n_device_types; ++t) {
    const hsim_device_type& d = c.device_types[t];
    const int g = d.gpus_per_node;
    if (g != 1 && g != 2 && g != 4 && g != 8) fail(HSIM_EINVAL, "RailMismatch: gpus_per_node must be 1, 2, 4 or 8");
    if (!(d.peak_flop_per_ns > 0) || !(d.hbm_bytes_per_ns > 0)) fail(HSIM_EINVAL, "InvalidValue: non-positive peak");
    for (int k = 0; k < HSIM_NKIND; ++k)
      if (!(d.eff_flop[k] > 0 && d.eff_flop[k] <= 1) || !(d.eff_mem[k] > 0 && d.eff_mem[k] <= 1))
        fail(HSIM_EINVAL, "InvalidValue: efficiency must be in (0, 1]");
    if (d.n_link_kinds < 1 || d.n_link_kinds > HSIM_MAX_LINK_KINDS) fail(HSIM_EINVAL, "InvalidValue: n_link_kinds");
    auto check_path = [&](const hsim_path& p, bool allow_empty) {
      if (p.n_hops < (allow_empty ? 0 : 1) || p.n_hops > HSIM_MAX_HOPS) fail(HSIM_EINVAL, "InvalidValue: path hop count");
      for (int k = 0; k < p.n_hops; ++k)
        if (!(p.hops[k].gbps > 0)) fail(HSIM_EINVAL, "NonPositiveBandwidth: hop gbps");
    };
    for (int k = 0; k < d.n_link_kinds; ++k) check_path(d.link_kinds[k], false);
    check_path(d.gpu_nic, true);
    if (!(d.nic_gbps > 0)) fail(HSIM_EINVAL, "NonPositiveBandwidth: nic_gbps");
    if (d.nic_delay_ns < 0) fail(HSIM_EINVAL, "InvalidValue: nic_delay_ns");
    for (int i = 0; i < g; ++i)
      for (int j = 0; j < g; ++j)
        if (i != j && (d.intra_kind[i][j] < 0 || d.intra_kind[i][j] >= d.n_link_kinds))
          fail(HSIM_EINVAL, "InvalidValue: intra_kind out of range");
  }
  for (int t = 1; t < c.n_device_types; ++t)
    if (c.device_types[t].gpus_per_node != c.device_types[0].gpus_per_node)
      fail(HSIM_EINVAL, "RailMismatch: every node type must have the same GPUs (= NICs) per node");
  for (int n = 0; n < c.n_nodes; ++n)
    if (c.node_type_of[n] < 0 || c.node_type_of[n] >= c.n_device_types) fail(HSIM_EINVAL, "UnknownGpuType: node_type_of");
  if (m.layers < 1 || m.hidden < 1 || m.heads < 1 || m.kv_heads < 1 || m.ffn < 1 || m.seq < 1 || m.vocab < 1 ||
      m.mlp_mats < 1 || m.moe_experts < 1 || m.moe_topk < 1 || m.bpe_act < 1 || m.bpe_grad < 1 || m.global_batch < 1)
    fail(HSIM_EINVAL, "InvalidValue: model counts must be >= 1");
  if (m.hidden % m.heads) fail(HSIM_EINVAL, "DivisibilityViolation: hidden % heads");
  if (m.heads % m.kv_heads) fail(HSIM_EINVAL, "DivisibilityViolation: heads % kv_heads");
  if (m.moe_topk > m.moe_experts) fail(HSIM_EINVAL, "InvalidValue: moe_topk > moe_experts");
  if (m.global_batch > (1 << 22)) fail(HSIM_ERANGE, "global_batch > 2^22");
  if (m.n_bset < 1 || m.n_bset > 8 || m.n_pset < 1 || m.n_pset > 16) fail(HSIM_EINVAL, "InvalidValue: bset / pset sizes");
  for (int k = 0; k < m.n_bset; ++k)
    if (m.bset[k] < 1) fail(HSIM_EINVAL, "InvalidValue: bset");
  for (int k = 0; k < m.n_pset; ++k)
    if (m.pset[k] < 1 || m.pset[k] > MAXP) fail(HSIM_EINVAL, "InvalidValue: pset entries must be 1..64");
  for (int t = 0; t < c.n_device_types; ++t)
    if (m.tpset_mask[t] & ~0xF) fail(HSIM_EINVAL, "InvalidValue: tpset_mask allows TP 1, 2, 4, 8 only");
  if (m.r_layer < 0 || m.r_batch < 0 || m.r_layer > 8 || m.r_batch > 8) fail(HSIM_EINVAL, "InvalidValue: radii");
  if (m.pmax_perturb < 0 || m.pmax_perturb > MAXP) fail(HSIM_EINVAL, "InvalidValue: pmax_perturb must be 0..64");
  if (m.homo && c.n_device_types > MAXC) fail(HSIM_EINVAL, "InvalidValue: too many classes");
  if (m.interleave < 0 || m.interleave > 8) fail(HSIM_EINVAL, "InvalidValue: interleave must be 0..8");
  if (m.ep_dp != 0 && m.ep_dp != 1) fail(HSIM_EINVAL, "InvalidValue: ep_dp must be 0 or 1");
  if (m.mixtp != 0 && m.mixtp != 1) fail(HSIM_EINVAL, "InvalidValue: mixtp must be 0 or 1");
  if (m.mem_check && (m.interleave > 1 || m.ep_dp || m.mixtp))
    fail(HSIM_EINVAL, "InvalidValue: mem_check is not defined with interleave / ep_dp / mixtp (DESIGN.md V.1-V.3)");
  if (m.ep_dp && m.mixtp) fail(HSIM_EINVAL, "InvalidValue: ep_dp is not defined with mixtp (DESIGN.md V.1)");
  if (m.sync_buckets < 0 || m.sync_buckets > 2 || (m.sync_buckets == 2 && m.interleave > 1))
    fail(HSIM_EINVAL, "InvalidValue: sync_buckets must be 0..2 and 2 is not defined with interleave (DESIGN.md B.1)");
}

void hsim_handle::derive_links() {
  const i64 fr = cd.frame_bytes;
  for (int t = 0; t < nt; ++t) {
    const hsim_device_type& d = types[t];
    for (int i = 0; i < d.gpus_per_node; ++i)
      for (int j = 0; j < d.gpus_per_node; ++j)
        intra[t][i][j] = i == j ? Link{0, 1e300} : path_link(d.link_kinds[(int)d.intra_kind[i][j]], fr);
  }
  for (int a = 0; a < nt; ++a)
    for (int b = 0; b < nt; ++b) {
      Link l = path_link(types[a].gpu_nic, fr);
      l = cat(l, Link{types[a].nic_delay_ns, types[a].nic_gbps / 8.0});
      l = cat(l, Link{cd.rail_alpha_ns, cd.rail_gbps / 8.0});
      l = cat(l, Link{types[b].nic_delay_ns, types[b].nic_gbps / 8.0});
      l = cat(l, path_link(types[b].gpu_nic, fr));
      rail[a][b] = l;
    }
  // every link the kernels may meet gets a class id, ids in (beta ascending,
  // alpha descending) order: eval_mask walks a mask from its slowest class
  {
    std::vector<Link> all;
    for (int t = 0; t < nt; ++t)
      for (int i = 0; i < types[t].gpus_per_node; ++i)
        for (int j = 0; j < types[t].gpus_per_node; ++j)
          if (i != j) all.push_back(intra[t][i][j]);
    for (int a = 0; a < nt; ++a)
      for (int i = 0; i < types[a].gpus_per_node; ++i)
        for (int b = 0; b < nt; ++b)
          for (int j = 0; j < types[b].gpus_per_node; ++j)
            all.push_back(i == j ? rail[a][b] : cat(intra[a][i][j], rail[a][b]));
    std::stable_sort(all.begin(), all.end(), [](const Link& x, const Link& y) {
      return x.beta != y.beta ? x.beta < y.beta : x.alpha > y.alpha;
    });
    for (const Link& l : all) lc(l);
  }
  std::memset(hT.lc_same, 0, sizeof(hT.lc_same));
  std::memset(hT.lc_cross, 0, sizeof(hT.lc_cross));
  for (int t = 0; t < nt; ++t)
    for (int i = 0; i < types[t].gpus_per_node; ++i)
      for (int j = 0; j < types[t].gpus_per_node; ++j)
        if (i != j) hT.lc_same[t][i][j] = (int8_t)lc(intra[t][i][j]);
  for (int a = 0; a < nt; ++a)
    for (int i = 0; i < types[a].gpus_per_node; ++i)
      for (int b = 0; b < nt; ++b)
        for (int j = 0; j < types[b].gpus_per_node; ++j) {
          Link l = i == j ? rail[a][b] : cat(intra[a][i][j], rail[a][b]);
          hT.lc_cross[a][i][b][j] = (int8_t)lc(l);
        }
  // translation invariance of every allowed TP group (A13): same link between
  // (k*tp + x) and (k*tp + y) for every block k
  for (int t = 0; t < nt; ++t) {
    const int g = types[t].gpus_per_node;
    for (int lg = 0; lg < 4; ++lg) {
      const int tp = 1 << lg;
      tp_mask[t][lg] = 0;
      if (!(md.tpset_mask[t] >> lg & 1) || g % tp) continue;
      for (int k = 1; k * tp < g; ++k)
        for (int x = 0; x < tp; ++x)
          for (int y = 0; y < tp; ++y)
            if (x != y) {
              const Link& a0 = intra[t][x][y];
              const Link& ak = intra[t][k * tp + x][k * tp + y];
              if (a0.alpha != ak.alpha || a0.beta != ak.beta)
                fail(HSIM_EINVAL, "InvalidValue: intra-node links not invariant under tp-aligned translation");
            }
      for (int q = 0; q < tp && tp > 1; ++q) tp_mask[t][lg] |= (u64)1 << lc(intra[t][q][(q + 1) % tp]);
    }
  }
}

void hsim_handle::derive_durations() {
  const i64 h = md.hidden, s = md.seq, V = md.vocab, f = md.ffn, nm = md.mlp_mats;
  const i64 hkv = (i64)md.kv_heads * h / md.heads;
  const i64 bpe = md.bpe_act, E = md.moe_experts, k = md.moe_topk;
  dur.assign((size_t)nt * 4 * bs.size(), Dur{});
  for (int t = 0; t < nt; ++t)
    for (int lg = 0; lg < 4; ++lg) {
      const i64 tp = 1 << lg;
      if (!(md.tpset_mask[t] >> lg & 1)) continue;
      // (tp > GPUs per node only in V.1 mixed groups, whose collectives crec() derives)
      if (md.heads % tp || md.kv_heads % tp) continue;
      const bool in_node = types[t].gpus_per_node % tp == 0;
      for (size_t bi = 0; bi < bs.size(); ++bi) {
        const i64 b = bs[bi], T = b * s;
        const hsim_device_type& ty = types[t];
        // (FLOP, bytes) per device, forward (DESIGN.md C.5)
        i64 fl[5], by[5];
        fl[HSIM_KIND_ATTN] = ceil_div(2 * T * h * (2 * h + 2 * hkv) + 4 * b * s * s * h, tp);
        by[HSIM_KIND_ATTN] = ceil_div(bpe * h * (2 * h + 2 * hkv), tp) + 2 * T * h * bpe;
        fl[HSIM_KIND_MLP] = ceil_div(2 * T * nm * h * f, tp);
        by[HSIM_KIND_MLP] = ceil_div(bpe * nm * h * f, tp) + 2 * T * h * bpe;
        fl[HSIM_KIND_MOE] = ceil_div(2 * T * k * nm * h * f, tp);
        by[HSIM_KIND_MOE] = ceil_div(bpe * E * nm * h * f, tp) + 2 * T * h * bpe;
        fl[HSIM_KIND_EMB] = 0;
        by[HSIM_KIND_EMB] = 2 * T * h * bpe;
        fl[HSIM_KIND_HEAD] = ceil_div(2 * T * h * V, tp);
        by[HSIM_KIND_HEAD] = ceil_div(bpe * V * h, tp) + T * h * bpe + ceil_div(T * V * bpe, tp);
        i64 dfw[5], dbw[5];
        for (int q = 0; q < 5; ++q) {
          if (2 * fl[q] >= TWO53 || 2 * by[q] >= TWO53) fail(HSIM_ERANGE, "a FLOP / byte numerator reaches 2^53");
          const double rf = ty.peak_flop_per_ns * ty.eff_flop[q];
          const double rm = ty.hbm_bytes_per_ns * ty.eff_mem[q];
          dfw[q] = std::max(ceilq(fl[q], rf), ceilq(by[q], rm));
          dbw[q] = std::max(ceilq(2 * fl[q], rf), ceilq(2 * by[q], rm));  // own rounding (A6)
        }
        Dur& d = dur_at(t, lg, bi);
        d.ok = true;
        const int mk = E > 1 ? HSIM_KIND_MOE : HSIM_KIND_MLP;
        d.attn_f = dfw[HSIM_KIND_ATTN]; d.attn_b = dbw[HSIM_KIND_ATTN];
        d.mlp_f = dfw[mk]; d.mlp_b = dbw[mk];
        d.emb_f = dfw[HSIM_KIND_EMB]; d.emb_b = dbw[HSIM_KIND_EMB];
        d.head_f = dfw[HSIM_KIND_HEAD]; d.head_b = dbw[HSIM_KIND_HEAD];
        // TP all-reduce 2(t-1) * max over ring edges; EP all-to-all (t-1) * max over pairs (A16, A17)
        const i64 A = b * s * h * bpe;
        d.ar = 0; d.a2a = 0;
        if (tp > 1 && in_node) {
          i64 mx = 0;
          for (int q = 0; q < tp; ++q) mx = std::max(mx, tau(intra[t][q][(q + 1) % tp], ceil_div(A, tp)));
          d.ar = 2 * (tp - 1) * mx;
          if (E > 1) {
            i64 my = 0;
            for (int x = 0; x < tp; ++x)
              for (int y = 0; y < tp; ++y)
                if (x != y) my = std::max(my, tau(intra[t][x][y], ceil_div(A * k, tp * tp)));
            d.a2a = (tp - 1) * my;
          }
        }
      }
    }
}

// C.3: class alone on a fresh cluster (classes of one template use disjoint
// device types, so their placements do not interact): replica-major,
// stage-major; lowest-id node of the stage's type with a free tp-aligned block.
// V.1 mixed group (type a, type a2): a tp/2-aligned block on the lowest node of
// type a with one free, then the same block on the lowest node of type a2
// where it is free.
std::vector<std::vector<GPl>> hsim_handle::place(int D, const std::vector<std::pair<int, int>>& stages) const {
  std::vector<std::vector<char>> used(cd.n_nodes);
  for (int n = 0; n < cd.n_nodes; ++n) used[n].assign(types[node_type[n]].gpus_per_node, 0);
  std::vector<std::vector<GPl>> out(D);
  for (int r = 0; r < D; ++r)
    for (const auto& st : stages) {
      const int t = st_t(st.first), t2 = st_t2(st.first), tp = st.second;
      const int w = t2 >= 0 ? tp / 2 : tp;
      GPl g{-1, -1, -1};
      for (size_t ni = 0; ni < nodes_of_type[t].size() && g.node < 0; ++ni) {
        const int n = nodes_of_type[t][ni];
        const int gp = types[t].gpus_per_node;
        for (int base = 0; base + w <= gp && g.node < 0; base += w) {
          bool fr = true;
          for (int q = 0; q < w; ++q) fr = fr && !used[n][base + q];
          if (fr) g = GPl{n, base, -1};
        }
      }
      if (g.node >= 0 && t2 >= 0) {
        for (size_t ni = 0; ni < nodes_of_type[t2].size() && g.node2 < 0; ++ni) {
          const int n = nodes_of_type[t2][ni];
          bool fr = g.base + w <= types[t2].gpus_per_node;
          for (int q = 0; q < w && fr; ++q) fr = !used[n][g.base + q];
          if (fr) g.node2 = n;
        }
        if (g.node2 < 0) g.node = -1;
      }
      if (g.node < 0) fail(HSIM_EINVAL, "InsufficientDevices: placement failed");
      for (int q = 0; q < w; ++q) used[g.node][g.base + q] = 1;
      if (g.node2 >= 0)
        for (int q = 0; q < w; ++q) used[g.node2][g.base + q] = 1;
      out[r].push_back(g);
    }
  return out;
}

// V.3: MoE op duration on type t with TP tp and the expert weights sharded
// over g devices (DESIGN.md C.5 with the weight-byte divisor g; g = tp is C.5)
i64 hsim_handle::moe_dur(int t, int tp, i64 b, i64 g, bool bwd) const {
  const i64 h = md.hidden, T = b * md.seq, f = md.ffn, nm = md.mlp_mats, bpe = md.bpe_act;
  const i64 fl = ceil_div(2 * T * md.moe_topk * nm * h * f, tp);
  const i64 by = ceil_div(bpe * md.moe_experts * nm * h * f, g) + 2 * T * h * bpe;
  const hsim_device_type& ty = types[t];
  const i64 mul = bwd ? 2 : 1;
  return std::max(ceilq(mul * fl, ty.peak_flop_per_ns * ty.eff_flop[HSIM_KIND_MOE]),
                  ceilq(mul * by, ty.hbm_bytes_per_ns * ty.eff_mem[HSIM_KIND_MOE]));
}

// V.3: all-to-all over the union of the TP groups (node, base) of size tp:
// (g - 1) x the slowest ordered pair at ceil(A k / (tp g)) bytes (A17 with g =
// #groups x tp).  Pairs are visited per distinct (node type, rank set) node
// signature -- a link depends only on (same node?, types, ranks) -- so the
// cost stays O(signatures^2 x 64) for any number of replicas.
i64 hsim_handle::a2a_groups(const std::vector<std::pair<int, int>>& groups, int tp, i64 b) const {
  const i64 g = (i64)groups.size() * tp;
  if (g == 1) return 0;
  std::map<int, uint32_t> ranks;  // node -> local ranks used
  for (auto& gr : groups)
    for (int q = 0; q < tp; ++q) ranks[gr.first] |= 1u << (gr.second + q);
  // (type, ranks) -> up to two nodes with that signature
  std::map<std::pair<int, uint32_t>, std::vector<int>> sig;
  for (auto& kv : ranks) {
    auto& v = sig[std::make_pair(node_type[kv.first], kv.second)];
    if (v.size() < 2) v.push_back(kv.first);
  }
  const i64 per = ceil_div(b * md.seq * md.hidden * md.bpe_act * md.moe_topk, (i64)tp * g);
  i64 slow = 0;
  for (auto& x : sig)
    for (auto& y : sig) {
      const int n1 = x.second[0];
      // a node of y other than n1 (cross-node links depend on types and ranks only)
      const int n2 = &x == &y ? (x.second.size() > 1 ? x.second[1] : -1) : y.second[0];
      for (int r1 = 0; r1 < MAXG; ++r1) {
        if (!(x.first.second >> r1 & 1)) continue;
        for (int r2 = 0; r2 < MAXG; ++r2) {
          if (!(y.first.second >> r2 & 1)) continue;
          if (&x == &y && r1 != r2) slow = std::max(slow, tau(link(n1, r1, n1, r2), per));  // same node
          if (n2 >= 0) slow = std::max(slow, tau(link(n1, r1, n2, r2), per));
        }
      }
    }
  return (g - 1) * slow;
}

// class record: (b, D, stages, ep) -> offset of the record in the pool.
// ep (V.3): the class is a single-class MoE template whose experts span its
// replicas -- per-stage all-to-all over every replica's group, lockstep
// replicas (one sub-class: the slowest boundary of any replica, replica 0's m).
int32_t hsim_handle::crec(int bi, int M, int D, const std::vector<std::pair<int, int>>& stages, bool ep) {
  std::vector<int> key{bi, D, ep ? 1 : 0};
  for (auto& s : stages) { key.push_back(s.first); key.push_back(s.second); }
  auto it = crec_of.find(key);
  if (it != crec_of.end()) return it->second;
  (void)M;
  const int P = (int)stages.size();
  const i64 b = bs[bi];
  const i64 A = b * md.seq * md.hidden * md.bpe_act;
  const auto pl = place(D, stages);
  bool mixed = false;
  std::vector<StageRec> sr(P);
  std::vector<i64> w(P);
  for (int s = 0; s < P; ++s) {
    const int t = st_t(stages[s].first), t2 = st_t2(stages[s].first), tp = stages[s].second, lg = __builtin_ctz(tp);
    Dur d = dur_at(t, lg, bi);
    if (t2 >= 0) {
      // V.1: equal shards on both types, every op ends with a TP collective, so
      // each op lasts as long as on the slower type (PAPER.md:280 C4); the TP
      // all-reduce ring and the all-to-all run over the group's device map
      mixed = true;
      const Dur& e = dur_at(t2, lg, bi);
      d.attn_f = std::max(d.attn_f, e.attn_f); d.attn_b = std::max(d.attn_b, e.attn_b);
      d.mlp_f = std::max(d.mlp_f, e.mlp_f);    d.mlp_b = std::max(d.mlp_b, e.mlp_b);
      d.emb_f = std::max(d.emb_f, e.emb_f);    d.emb_b = std::max(d.emb_b, e.emb_b);
      d.head_f = std::max(d.head_f, e.head_f); d.head_b = std::max(d.head_b, e.head_b);
      for (int r = 0; r < D; ++r) {
        i64 ar = 0, a2a = 0;
        for (int q = 0; q < tp; ++q) ar = std::max(ar, tau(dlink(pl[r][s], tp, q, pl[r][s], tp, (q + 1) % tp), ceil_div(A, tp)));
        ar *= 2 * (tp - 1);
        if (md.moe_experts > 1)
          for (int x = 0; x < tp; ++x)
            for (int y = 0; y < tp; ++y)
              if (x != y) a2a = std::max(a2a, (i64)(tp - 1) * tau(dlink(pl[r][s], tp, x, pl[r][s], tp, y), ceil_div(A * md.moe_topk, (i64)tp * tp)));
        if (r > 0 && (ar != d.ar || a2a != d.a2a))
          fail(HSIM_EINVAL, "InvalidValue: mixed TP groups' links differ between replicas");
        d.ar = ar;
        d.a2a = a2a;
      }
    }
    StageRec& r = sr[s];
    std::memset(&r, 0, sizeof r);
    r.type = t; r.type2 = t2; r.tp = tp; r.lg_tp = lg;
    i64 mlp_f = d.mlp_f, mlp_b = d.mlp_b, a2a = d.a2a;
    if (ep) {
      std::vector<std::pair<int, int>> grp(D);
      for (int q = 0; q < D; ++q) grp[q] = {pl[q][s].node, pl[q][s].base};
      a2a = a2a_groups(grp, tp, b);
      mlp_f = moe_dur(t, tp, b, (i64)D * tp, false);
      mlp_b = moe_dur(t, tp, b, (i64)D * tp, true);
    }
    if (md.moe_experts > 1) {
      r.layer_f = d.attn_f + d.ar + a2a + mlp_f + a2a;
      r.layer_b = d.attn_b + d.ar + a2a + mlp_b + a2a;
    } else {
      r.layer_f = d.attn_f + d.ar + d.mlp_f + d.ar;
      r.layer_b = d.attn_b + d.ar + d.mlp_b + d.ar;
    }
    r.tcomp = d.attn_f + mlp_f + d.attn_b + mlp_b;
    if (s == 0) { r.fext += d.emb_f; r.gext += d.emb_b; r.wext += d.emb_f + d.emb_b; r.emb_b = d.emb_b; }
    if (s == P - 1) { r.fext += d.head_f; r.gext += d.head_b; r.wext += d.head_f + d.head_b; }
    if (t2 >= 0) {
      for (int q = 0; q < tp; ++q) r.tp_mask |= (u64)1 << lc(dlink(pl[0][s], tp, q, pl[0][s], tp, (q + 1) % tp));
    } else {
      r.tp_mask = tp_mask[t][lg];
    }
    w[s] = ((i64)1 << 40) / r.tcomp;
    layer_fb_max = std::max(layer_fb_max, r.layer_f + r.layer_b);
    ext_max = std::max(ext_max, r.fext + r.gext);
  }
  // base layer split: Hamilton of L with weights floor(2^40 / tcomp) (C.4)
  {
    i64 W = 0, given = 0;
    for (i64 x : w) W += x;
    std::vector<i64> rem(P);
    for (int s = 0; s < P; ++s) { sr[s].l0 = (int32_t)hamilton_floor_rem(md.layers, w[s], W, &rem[s]); given += sr[s].l0; }
    std::vector<int> ord(P);
    for (int s = 0; s < P; ++s) ord[s] = s;
    std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return rem[x] > rem[y]; });
    for (i64 k = 0; k < md.layers - given; ++k) sr[ord[k]].l0 += 1;
  }
  for (int s = 0; s < P; ++s) {
    sr[s].first_node = (int16_t)pl[0][s].node; sr[s].first_base = (int16_t)pl[0][s].base;
    sr[s].last_node = (int16_t)pl[D - 1][s].node; sr[s].last_base = (int16_t)pl[D - 1][s].base;
    const int tp = sr[s].tp;
    // V.1 (single-class MIXTP templates, TplRec flag 2): the ring's wrap edge
    // D-1 -> 0 is folded in here too (the kernels' cross-class term assumes
    // homogeneous groups)
    for (int lg = 0; lg <= sr[s].lg_tp; ++lg)
      for (int r = 0; r + 1 < D + (mixed && D > 1 ? 1 : 0); ++r)
        for (int q = 0; q < (1 << lg); ++q)
          sr[s].dp_mask[lg] |= (u64)1 << lc(dlink(pl[r][s], tp, q, pl[(r + 1) % D][s], tp, q));
  }
  // p2p cost per replica per boundary (A8): rank pairs q < min(tp_s, tp_s+1),
  // max of tau(A); V.2 appends the wrap boundary stage P-1 -> stage 0
  const bool wrap = ilv > 1 && P >= 2;
  auto p2p = [&](int r, int s1, int s2) {
    const int t1 = stages[s1].second, t2 = stages[s2].second;
    i64 c = 0;
    for (int q = 0; q < std::min(t1, t2); ++q) c = std::max(c, tau(dlink(pl[r][s1], t1, q, pl[r][s2], t2, q), A));
    return c;
  };
  std::vector<std::vector<i64>> cv(D, std::vector<i64>(P, 0));  // [0, P-1) boundaries, [P-1] wrap
  for (int r = 0; r < D; ++r) {
    for (int s = 0; s + 1 < P; ++s) cv[r][s] = p2p(r, s, s + 1);
    if (wrap) cv[r][P - 1] = p2p(r, P - 1, 0);
    for (i64 c : cv[r]) c_max = std::max(c_max, c);
  }
  if (ep)  // lockstep: every replica runs the slowest boundary of any replica
    for (int r = 1; r < D; ++r)
      for (int s = 0; s < P; ++s) cv[0][s] = std::max(cv[0][s], cv[r][s]);
  depth_max = std::max(depth_max, P);
  // sub-classes (A13): replicas with identical p2p vectors, ordered by lowest replica
  std::vector<int> rep;
  std::map<std::vector<i64>, int> seen;
  for (int r = 0; r < (ep ? 1 : D); ++r)
    if (seen.emplace(cv[r], r).second) rep.push_back(r);
  const int32_t off = (int32_t)pool.size();
  if ((size_t)off + HDR_WORDS + 16 * P + rep.size() * (P + 1) > (size_t)INT32_MAX)
    fail(HSIM_ERANGE, "class-record pool exceeds 2^31 entries");
  CrecHdr hd{};
  hd.P = P;
  hd.D = D;
  hd.U = (int32_t)rep.size();
  hd.nd = P <= md.pmax_perturb ? P - 1 : 0;
  hd.pw = 1;
  for (int q = 0; q < hd.nd; ++q) hd.pw *= (u32)(2 * md.r_layer + 1);
  hd.pwdiv = make_fastdiv(hd.pw);
  hd.woff = -1;
  pw_max = std::max(pw_max, hd.pw);
  u_max = std::max(u_max, hd.U);
  pool.resize(off + HDR_WORDS + 16 * P + rep.size() * (P + 1));
  std::memcpy(&pool[off], &hd, sizeof hd);
  std::memcpy(&pool[off + HDR_WORDS], sr.data(), sizeof(StageRec) * P);
  for (size_t u = 0; u < rep.size(); ++u) {
    i64* sub = &pool[off + HDR_WORDS + 16 * P + u * (P + 1)];
    sub[0] = rep[u];
    for (int s = 0; s < P; ++s) sub[1 + s] = cv[rep[u]][s];
  }
  crec_of[key] = off;
  return off;
}

// C.2: templates in order: b ascending; HOMO family (per type "unused" or
// (tp, P, D), lexicographic with type 0 most significant), then MIXED family
// (per type (tp, P), lexicographic; D ascending); keep M >= D only.
void hsim_handle::enumerate() {
  std::vector<int> ps(md.pset, md.pset + md.n_pset);
  std::sort(ps.begin(), ps.end());
  ps.erase(std::unique(ps.begin(), ps.end()), ps.end());
  auto tp_allowed = [&](int t, int tp) {
    return (md.tpset_mask[t] >> __builtin_ctz(tp) & 1) && types[t].gpus_per_node % tp == 0 && md.heads % tp == 0 &&
           md.kv_heads % tp == 0;
  };
  const i64 rl = 2 * md.r_layer + 1, rb = 2 * md.r_batch + 1;
  // mixed radix of a template; saturates at 2^31 (rejected below) so no
  // product can overflow whatever pmax_perturb / P are
  auto radix_of = [&](const std::vector<int>& Ps) {
    const i64 cap = (i64)1 << 31;
    i64 r = 1;
    for (int P : Ps)
      if (P <= md.pmax_perturb)
        for (int k = 0; k + 1 < P; ++k) r = std::min(cap, r * rl);
    for (size_t k = 0; k + 1 < Ps.size(); ++k) r = std::min(cap, r * rb);
    return r;
  };
  i64 acc = 0;
  for (size_t bi = 0; bi < bs.size(); ++bi) {
    const int b = bs[bi];
    if (md.global_batch % b) continue;
    const i64 M = md.global_batch / b;
    auto push = [&](const std::vector<std::pair<int, std::vector<std::pair<int, int>>>>& classes) {
      i64 Dt = 0;
      std::vector<int> Ps;
      for (auto& c : classes) { Dt += c.first; Ps.push_back((int)c.second.size()); }
      if (M < Dt) return;
      const i64 R = radix_of(Ps);  // before crec(): its u32 digit radix must not wrap
      if (R >= ((i64)1 << 31)) fail(HSIM_ERANGE, "template radix exceeds 2^31");
      TplRec r{};
      r.prefix = acc;
      r.rD = 1.0 / (double)Dt;
      r.b = b; r.M = (int32_t)M; r.C = (int32_t)classes.size(); r.D = (int32_t)Dt;
      const bool ep = md.ep_dp && md.moe_experts > 1 && classes.size() == 1;  // V.3
      r.flags = ep ? 1 : 0;
      for (auto& c : classes)
        for (auto& st : c.second)
          if (st_t2(st.first) >= 0) r.flags |= 2;  // V.1 mixed TP groups
      int cnt[33] = {0}, nilv = 0;
      for (size_t c = 0; c < classes.size(); ++c) {
        const int P = (int)classes[c].second.size();
        r.crec[c] = crec((int)bi, (int)M, classes[c].first, classes[c].second, ep);
        if (ilv > 1 && P >= 2) {  // V.2: every interleaved pipeline runs in K_ilv (pmask bit 0)
          r.pmask |= 1u;
          ++nilv;
          ilv_depth_max = std::max(ilv_depth_max, P);
        } else {
          r.pmask |= 1u << std::min<int>(P, 31);
          cnt[std::min<int>(P, 32)]++;
        }
      }
      ilv_jobs_max = std::max(ilv_jobs_max, nilv);
      cmax = std::max(cmax, (int)classes.size());
      m_max = std::max(m_max, M);
      for (int q = 0; q <= FASTP; ++q) pcnt_max[q] = std::max(pcnt_max[q], cnt[q]);
      for (int q = 0; q <= FASTP; ++q) depth_jobs_space[q] += R * cnt[q];
      pmask_all |= r.pmask;
      {
        int sp = 0;
        for (int P : Ps) sp += P;
        stages_max = std::max(stages_max, sp);
      }
      tpl.push_back(r);
      prefix.push_back(acc);
      acc += R;
    };
    if (md.homo) {
      struct Opt { int tp, P, D; };
      std::vector<std::vector<Opt>> opt(nt);
      for (int t = 0; t < nt; ++t) {
        opt[t].push_back({0, 0, 0});
        for (int tp = 1; tp <= 8; tp *= 2) {
          if (!tp_allowed(t, tp)) continue;
          for (int P : ps) {
            if (P > md.layers) continue;
            for (i64 D = 1; D * P * tp <= n_of_type[t]; ++D)
              if (!md.use_all || D * P * tp == n_of_type[t]) opt[t].push_back({tp, P, (int)D});
          }
        }
      }
      std::vector<size_t> k(nt, 0);
      for (;;) {
        std::vector<std::pair<int, std::vector<std::pair<int, int>>>> cls;
        for (int t = 0; t < nt; ++t)
          if (k[t]) {
            const Opt& o = opt[t][k[t]];
            cls.push_back({o.D, std::vector<std::pair<int, int>>(o.P, {t, o.tp})});
          }
        if (!cls.empty()) push(cls);
        int t = nt - 1;
        while (t >= 0) {
          if (++k[t] < opt[t].size()) break;
          k[t] = 0;
          --t;
        }
        if (t < 0) break;
      }
    }
    if (md.mixed && nt >= 2) {
      std::vector<std::vector<std::pair<int, int>>> opt(nt);  // (tp, P)
      bool empty = false;
      for (int t = 0; t < nt; ++t) {
        for (int tp = 1; tp <= 8; tp *= 2)
          if (tp_allowed(t, tp))
            for (int P : ps) opt[t].push_back({tp, P});
        empty = empty || opt[t].empty();
      }
      if (!empty) {
        std::vector<size_t> k(nt, 0);
        for (;;) {
          i64 sumP = 0, Dmax = INT64_MAX;
          for (int t = 0; t < nt; ++t) {
            sumP += opt[t][k[t]].second;
            Dmax = std::min(Dmax, n_of_type[t] / ((i64)opt[t][k[t]].first * opt[t][k[t]].second));
          }
          if (sumP <= md.layers && Dmax >= 1) {
            std::vector<std::pair<int, int>> st;
            for (int t = 0; t < nt; ++t)
              for (int s = 0; s < opt[t][k[t]].second; ++s) st.push_back({t, opt[t][k[t]].first});
            if ((int)st.size() > MAXP) fail(HSIM_ERANGE, "pipeline deeper than 64 stages");
            for (i64 D = md.use_all ? Dmax : 1; D <= Dmax; ++D) push({{(int)D, st}});
          }
          int t = nt - 1;
          while (t >= 0) {
            if (++k[t] < opt[t].size()) break;
            k[t] = 0;
            --t;
          }
          if (t < 0) break;
        }
      }
    }
    if (md.mixtp && nt >= 2) {
      // V.1 MIXTP family: one class, every stage a mixed TP group of tp devices,
      // tp/2 of type a and tp/2 of type a2 (a < a2): tp >= 2 in both TP sets,
      // tp | heads and kv heads, tp/2 | GPUs per node; D replicas of P stages
      // need D P tp/2 GPUs of each type (use_all: exactly all of both)
      for (int a = 0; a < nt; ++a)
        for (int a2 = a + 1; a2 < nt; ++a2)
          for (int tp = 2; tp <= 8; tp *= 2) {
            const int lg = __builtin_ctz(tp);
            if (!(md.tpset_mask[a] >> lg & 1) || !(md.tpset_mask[a2] >> lg & 1) || md.heads % tp || md.kv_heads % tp ||
                types[a].gpus_per_node % (tp / 2) || types[a2].gpus_per_node % (tp / 2))
              continue;
            for (int P : ps) {
              if (P > md.layers) continue;
              for (i64 D = 1; D * P * (tp / 2) <= std::min(n_of_type[a], n_of_type[a2]); ++D) {
                if (md.use_all && (D * P * (tp / 2) != n_of_type[a] || D * P * (tp / 2) != n_of_type[a2])) continue;
                push({{(int)D, std::vector<std::pair<int, int>>(P, {st_code(a, a2), tp})}});
              }
            }
          }
    }
  }
  N = acc;
  prefix.push_back(acc);
}

void hsim_handle::prepare() {
  node_type8.assign(node_type.begin(), node_type.end());
  hT.L = md.layers;
  const i64 h = md.hidden, hkv = (i64)md.kv_heads * h / md.heads, E = md.moe_experts;
  const i64 Wlayer = h * (2 * h + 2 * hkv) + (i64)md.mlp_mats * h * md.ffn * E + (E > 1 ? h * E : 0) + 2 * h;
  hT.seg_layer_bytes = Wlayer * md.bpe_grad;
  hT.seg_first_bytes = (i64)md.vocab * h * md.bpe_grad;
  hT.seg_last_bytes = ((i64)md.vocab * h * (md.tied ? 0 : 1) + h) * md.bpe_grad;
  if (md.layers * hT.seg_layer_bytes + hT.seg_first_bytes + hT.seg_last_bytes >= TWO53)
    fail(HSIM_ERANGE, "gradient bytes reach 2^53");
  // memory feasibility (DESIGN.md M.1); overlapped sync (DESIGN.md S.1)
  hT.mem_check = md.mem_check ? 1 : 0;
  hT.sync_overlap = md.sync_overlap ? 1 : 0;
  hT.interleave = ilv;
  hT.buckets = md.sync_buckets == 2 ? 2 : 1;
  hT.ep_dp = md.ep_dp;
  hT.seg_layer_dense = (h * (2 * h + 2 * hkv) + (E > 1 ? h * E : 0) + 2 * h) * md.bpe_grad;  // V.3
  if (md.sync_overlap && md.layers > 32767) fail(HSIM_ERANGE, "sync_overlap needs layers < 2^15");
  {
    const i64 bst = (i64)md.bpe_act + md.bpe_grad + 12;  // weights + gradients + Adam fp32 master / m / v
    double worst = 0, bmax = 1;
    for (int q = 0; q < md.n_bset && q < 8; ++q) bmax = std::max(bmax, (double)md.bset[q]);
    for (int lg = 0; lg < 4; ++lg) {
      const i64 t = (i64)1 << lg;
      hT.mem_layer[lg] = (Wlayer + t - 1) / t * bst;
      hT.mem_emb[lg] = ((i64)md.vocab * h + t - 1) / t * bst;
      hT.mem_head[lg] = ((i64)md.vocab * h * (md.tied ? 0 : 1) + h + t - 1) / t * bst;
      hT.mem_K[lg] = (i64)md.seq * h * (10 * t + 24);
      // largest need any candidate can have: all layers, deepest in-flight, largest b
      worst = std::max(worst, (double)md.layers * hT.mem_layer[lg] + hT.mem_emb[lg] + hT.mem_head[lg] +
                                  (double)MAXP * md.layers * (bmax * hT.mem_K[lg]));
    }
    if (md.mem_check && worst >= 9.0e18) fail(HSIM_ERANGE, "memory need may overflow int64");
    for (int k = 0; k < MAXT; ++k) hT.mem_cap[k] = k < cd.n_device_types ? cd.device_types[k].mem_bytes : 0;
    if (md.mem_check)
      for (int k = 0; k < cd.n_device_types; ++k)
        if (cd.device_types[k].mem_bytes <= 0) fail(HSIM_EINVAL, "InvalidValue: mem_bytes must be > 0 with mem_check");
  }
  hT.r_layer = md.r_layer;
  hT.r_batch = md.r_batch;
  hT.ldiv = make_fastdiv((u32)(2 * md.r_layer + 1));
  hT.bdiv = make_fastdiv((u32)(2 * md.r_batch + 1));
  hT.n_tpl = (i64)tpl.size();
  hT.N = N;
  {  // dedupe key widths
    auto bits = [](u64 v) { int b = 0; while (v) { ++b; v >>= 1; } return b; };
    hT.dd_wt = bits((u64)(tpl.empty() ? 0 : tpl.size() - 1));
    hT.dd_wd = bits((u64)pw_max - 1);
    hT.dd_wm = bits((u64)m_max);
    hT.dd_wu = bits((u64)(u_max - 1));
    hT.dd_ok = hT.dd_wt + 2 + hT.dd_wd + hT.dd_wm + 2 * hT.dd_wu <= 63 ? 1 : 0;
  }
  hT.n_lc = (int32_t)lcs.size();
  hT.n_nodes = cd.n_nodes;
  for (size_t k = 0; k < lcs.size(); ++k) hT.lc[k] = lcs[k];
  // exact integer tau: beta = G / 2^k with every x << k < 2^52 (x <= total gradient bytes)
  {
    const i64 xmax = md.layers * hT.seg_layer_bytes + hT.seg_first_bytes + hT.seg_last_bytes;
    bool exact = true;
    for (size_t b = 0; b < lcs.size() && exact; ++b) {
      bool found = false;
      for (int k = 0; k <= 20 && !found; ++k) {
        const double v = std::ldexp(lcs[b].beta, k);  // exact scaling by 2^k
        if (v >= 1 && v < 2147483648.0 && v == std::floor(v) && (xmax < ((i64)1 << (52 - k)))) {
          hT.lc_G[b] = (i64)v;
          hT.lc_k[b] = (int8_t)k;
          hT.lc_rG[b] = 1.0 / v;
          hT.lc_rb[b] = 1.0 / lcs[b].beta;
          found = true;
        }
      }
      exact = found;
    }
    hT.lc_exact = exact ? 1 : 0;
    // classes after b (beta >= beta_b) that b does not dominate: alpha_a > alpha_b
    // (tau_b(x) >= tau_a(x) for all x when alpha_b >= alpha_a and beta_b <= beta_a)
    for (size_t b = 0; b < lcs.size(); ++b) {
      if (b > 0 && !(lcs[b - 1].beta < lcs[b].beta || (lcs[b - 1].beta == lcs[b].beta && lcs[b - 1].alpha > lcs[b].alpha)))
        fail(HSIM_EINVAL, "internal: link classes not in (beta, -alpha) order");
      hT.lc_up[b] = 0;
      for (size_t a = b + 1; a < lcs.size(); ++a)
        if (lcs[a].alpha > lcs[b].alpha) hT.lc_up[b] |= (u64)1 << a;
    }
  }
  // link classes of the q < 2^lg edges between two groups' bases (cross-class ring edges)
  {
    xmask_cross.assign((size_t)MAXT * MAXG * MAXT * MAXG * 4, 0);
    xmask_same.assign((size_t)MAXT * MAXG * MAXG * 4, 0);
    const int g = types[0].gpus_per_node;
    for (int t1 = 0; t1 < nt; ++t1)
      for (int b1 = 0; b1 < g; ++b1)
        for (int b2 = 0; b2 < g; ++b2)
          for (int lg = 0; lg < 4; ++lg) {
            for (int t2 = 0; t2 < nt; ++t2) {
              u64 m = 0;
              for (int q = 0; q < (1 << lg) && b1 + q < g && b2 + q < g; ++q) m |= (u64)1 << hT.lc_cross[t1][b1 + q][t2][b2 + q];
              xmask_cross[(((t1 * MAXG + b1) * MAXT + t2) * MAXG + b2) * 4 + lg] = m;
            }
            u64 m = 0;
            for (int q = 0; q < (1 << lg) && b1 + q < g && b2 + q < g; ++q)
              if (b1 + q != b2 + q) m |= (u64)1 << hT.lc_same[t1][b1 + q][b2 + q];
            xmask_same[((t1 * MAXG + b1) * MAXG + b2) * 4 + lg] = m;
          }
    hT.xmask_cross = xmask_cross.data();
    hT.xmask_same = xmask_same.data();
  }
  int shift = 0;
  while ((N >> shift) > 65536) ++shift;
  const i64 nbk = N > 0 ? ((N - 1) >> shift) + 1 : 1;
  bucket.assign(nbk + 1, 0);
  for (i64 b = 0; b <= nbk; ++b)
    bucket[b] = (int32_t)bsearch_le(prefix.data(), (i64)tpl.size(), std::min((b << shift), N > 0 ? N - 1 : 0));
  hT.n_bucket = nbk;
  hT.bucket_shift = shift;
  hT.tpl_bucket = bucket.data();
  cprefix.assign(prefix.size(), 0);
  for (size_t k = 0; k + 1 < prefix.size(); ++k) cprefix[k + 1] = cprefix[k] + (prefix[k + 1] - prefix[k] + CHUNK - 1) / CHUNK;
  hT.tpl_cprefix = cprefix.data();
  {
    const i64 nch = cprefix.back();
    int cs = 0;
    while ((nch >> cs) > 65536) ++cs;
    const i64 ncb = nch > 0 ? ((nch - 1) >> cs) + 1 : 1;
    cbucket.assign(ncb + 1, 0);
    for (i64 b = 0; b <= ncb; ++b)
      cbucket[b] = (int32_t)bsearch_le(cprefix.data(), (i64)tpl.size(), std::min((b << cs), nch > 0 ? nch - 1 : 0));
    hT.n_cbucket = ncb;
    hT.cbucket_shift = cs;
    hT.tpl_cbucket = cbucket.data();
  }
  // f3 link graph (DESIGN.md F.1): node lists per type, port / PCIe / NIC capacities
  {
    type_nodes.clear();
    for (int t = 0; t < MAXT; ++t) {
      hT.type_node_off[t] = (int32_t)type_nodes.size();
      if (t < nt)
        for (int n : nodes_of_type[t]) type_nodes.push_back(n);
    }
    hT.type_node_off[MAXT] = (int32_t)type_nodes.size();
    hT.type_nodes = type_nodes.data();
    hT.gpn = types[0].gpus_per_node;
    std::memset(hT.port_cap, 0, sizeof(hT.port_cap));
    for (int t = 0; t < nt; ++t) {
      const int g = types[t].gpus_per_node;
      for (int r = 0; r < g; ++r)
        for (int j = 0; j < g; ++j)
          if (j != r) {  // the port's line rate: its fastest intra-node path
            hT.port_cap[t][r][0] = std::max(hT.port_cap[t][r][0], intra[t][r][j].beta);
            hT.port_cap[t][r][1] = std::max(hT.port_cap[t][r][1], intra[t][j][r].beta);
          }
      hT.pcie_cap[t] = path_link(types[t].gpu_nic, cd.frame_bytes).beta;
      hT.nic_cap[t] = std::min(types[t].nic_gbps / 8.0, cd.rail_gbps / 8.0);
    }
  }
  // partition weight table: every class record's rows for all
  // of its boundary digits, while the total stays under 2^26 entries
  wtab.clear();
  for (auto& kv : crec_of) {
    CrecHdr* hd = (CrecHdr*)&pool[kv.second];
    const StageRec* st = (const StageRec*)&pool[kv.second + HDR_WORDS];
    if (wtab.size() + hd->pw > ((size_t)1 << 26)) continue;
    hd->woff = (int32_t)wtab.size();
    const int r = md.r_layer, base = 2 * md.r_layer + 1;
    for (u32 dig = 0; dig < hd->pw; ++dig) {
      u32 dd = dig;
      int dprev = 0, lmin = 1 << 30;
      i64 worst = 0;
      for (int s = 0; s < hd->P; ++s) {
        int d = 0;
        if (s < hd->nd) {
          d = (int)(dd % (u32)base) - r;
          dd /= (u32)base;
        }
        const int l = st[s].l0 + d - dprev;
        dprev = d;
        lmin = std::min(lmin, l);
        worst = std::max(worst, (i64)l * st[s].tcomp + st[s].wext);
      }
      const i64 w = lmin >= 1 && worst > 0 ? ((i64)1 << 40) / worst : 0;
      wtab.push_back(w | (i64)std::max(0, std::min(lmin, 65535)) << 48);
    }
  }
  hT.wtab = nullptr;  // host paths walk the stages
  hT.tpl_prefix = prefix.data();
  hT.tpl = tpl.data();
  hT.pool = pool.data();
  hT.node_type = node_type8.data();
}

void hsim_handle::upload() {
  auto ck = [](cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(e == cudaErrorMemoryAllocation ? HSIM_ENOMEM : HSIM_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
  };
  Tables dt = hT;
  ck(cudaMalloc(&d_prefix, prefix.size() * 8), "cudaMalloc prefix");
  ck(cudaMalloc(&d_bucket, bucket.size() * 4), "cudaMalloc bucket");
  ck(cudaMemcpy(d_bucket, bucket.data(), bucket.size() * 4, cudaMemcpyHostToDevice), "H2D bucket");
  dt.tpl_bucket = d_bucket;
  ck(cudaMalloc(&d_cprefix, cprefix.size() * 8), "cudaMalloc cprefix");
  ck(cudaMemcpy(d_cprefix, cprefix.data(), cprefix.size() * 8, cudaMemcpyHostToDevice), "H2D cprefix");
  dt.tpl_cprefix = d_cprefix;
  ck(cudaMalloc(&d_cbucket, cbucket.size() * 4), "cudaMalloc cbucket");
  ck(cudaMemcpy(d_cbucket, cbucket.data(), cbucket.size() * 4, cudaMemcpyHostToDevice), "H2D cbucket");
  dt.tpl_cbucket = d_cbucket;
  ck(cudaMalloc(&d_xmask, (xmask_cross.size() + xmask_same.size()) * 8), "cudaMalloc xmask");
  ck(cudaMemcpy(d_xmask, xmask_cross.data(), xmask_cross.size() * 8, cudaMemcpyHostToDevice), "H2D xmask");
  ck(cudaMemcpy(d_xmask + xmask_cross.size(), xmask_same.data(), xmask_same.size() * 8, cudaMemcpyHostToDevice), "H2D xmask");
  dt.xmask_cross = d_xmask;
  dt.xmask_same = d_xmask + xmask_cross.size();
  ck(cudaMalloc(&d_tpl, std::max<size_t>(1, tpl.size()) * sizeof(TplRec)), "cudaMalloc tpl");
  ck(cudaMalloc(&d_pool, std::max<size_t>(1, pool.size()) * 8), "cudaMalloc pool");
  ck(cudaMalloc(&d_node_type, node_type8.size()), "cudaMalloc nodes");
  ck(cudaMalloc(&dT, sizeof(Tables)), "cudaMalloc tables");
  ck(cudaMalloc(&d_cells, 8), "cudaMalloc cells");
  ck(cudaMemcpy(d_prefix, prefix.data(), prefix.size() * 8, cudaMemcpyHostToDevice), "H2D prefix");
  if (!tpl.empty()) ck(cudaMemcpy(d_tpl, tpl.data(), tpl.size() * sizeof(TplRec), cudaMemcpyHostToDevice), "H2D tpl");
  if (!pool.empty()) ck(cudaMemcpy(d_pool, pool.data(), pool.size() * 8, cudaMemcpyHostToDevice), "H2D pool");
  ck(cudaMemcpy(d_node_type, node_type8.data(), node_type8.size(), cudaMemcpyHostToDevice), "H2D nodes");
  dt.tpl_prefix = d_prefix;
  dt.tpl = d_tpl;
  dt.pool = d_pool;
  dt.node_type = d_node_type;
  ck(cudaMalloc(&d_type_nodes, std::max<size_t>(1, type_nodes.size()) * 4), "cudaMalloc type nodes");
  ck(cudaMemcpy(d_type_nodes, type_nodes.data(), type_nodes.size() * 4, cudaMemcpyHostToDevice), "H2D type nodes");
  dt.type_nodes = d_type_nodes;
  ck(cudaMalloc(&d_wtab, std::max<size_t>(1, wtab.size()) * 8), "cudaMalloc wtab");
  if (!wtab.empty()) ck(cudaMemcpy(d_wtab, wtab.data(), wtab.size() * 8, cudaMemcpyHostToDevice), "H2D wtab");
  dt.wtab = d_wtab;
  ck(cudaMemcpy(dT, &dt, sizeof(Tables), cudaMemcpyHostToDevice), "H2D tables");
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sm_count, cudaDevAttrMultiProcessorCount, dev);
  ck(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming), "cudaEventCreate");
  for (int q = 0; q < NPLAN; ++q) ck(cudaEventCreateWithFlags(&ev_plan[q], cudaEventDisableTiming), "cudaEventCreate");
  ck(cudaEventCreateWithFlags(&ev_done, cudaEventDisableTiming), "cudaEventCreate");
  for (int q = 0; q < NEV; ++q) ck(cudaEventCreateWithFlags(&ev_pool[q], cudaEventDisableTiming), "cudaEventCreate");
  // latency-bound phase kernels (deep 1F1B chains: K_pipe<P >= 9> on streams
  // 9..16, K_deep on 17) get the highest stream priority so their few
  // long-running blocks are resident before the throughput kernels fill the SMs
  int prio_lo = 0, prio_hi = 0;
  cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
  for (int q = 0; q < NSIDE; ++q) {
#ifndef HSIM_NOPRIO
#ifdef HSIM_PRIO4
    const int prio = (q >= 9 && q <= 17) || q >= 20 || q == 4 ? prio_hi : prio_lo;
#else
    const int prio = (q >= 9 && q <= 17) || q >= 20 ? prio_hi : prio_lo;
#endif
#else
    const int prio = prio_lo;
#endif
    ck(cudaStreamCreateWithPriority(&side[q], cudaStreamNonBlocking, prio), "cudaStreamCreate");
    ck(cudaEventCreateWithFlags(&ev_join[q], cudaEventDisableTiming), "cudaEventCreate");
  }
}

// =============================================================================
// C ABI
// =============================================================================
namespace hsim {
int launch_eval(hsim_handle* h, const Tables* dT, const hsim_cands* c, int64_t n, int64_t* out_ns, int32_t k,
                int64_t* out_t, int64_t* out_i, cudaStream_t st);
int launch_count(hsim_handle* h, const Tables* dT, int64_t first, int64_t n, int64_t* d_acc, cudaStream_t st);
int launch_merge(const int64_t* lists, int32_t nlists, int32_t k, int64_t* out_t, int64_t* out_i, cudaStream_t st);
int launch_flow(hsim_handle* h, const Tables* dT, const Tables& hT, const int64_t* idx, int32_t k, int64_t* out,
                int64_t* fct, int64_t fct_cap, cudaStream_t st);
}

extern "C" {

const char* hsim_last_error(void) { return g_err.c_str(); }

int hsim_create(const hsim_cluster_desc* cluster, const hsim_model_desc* model, hsim_handle** out) {
  g_err.clear();
  if (!out) { g_err = "MissingField: out"; return HSIM_EINVAL; }
  *out = nullptr;
  if (!cluster || !model) { g_err = "MissingField: cluster / model"; return HSIM_EINVAL; }
  hsim_handle* h = new (std::nothrow) hsim_handle();
  if (!h) { g_err = "out of host memory"; return HSIM_ENOMEM; }
  try {
    h->cd = *cluster;
    h->md = *model;
    h->validate();
    h->nt = cluster->n_device_types;
    h->types.assign(cluster->device_types, cluster->device_types + h->nt);
    h->node_type.assign(cluster->node_type_of, cluster->node_type_of + cluster->n_nodes);
    h->cd.device_types = h->types.data();
    h->cd.node_type_of = h->node_type.data();
    h->nodes_of_type.assign(h->nt, {});
    for (int n = 0; n < cluster->n_nodes; ++n) {
      h->nodes_of_type[h->node_type[n]].push_back(n);
      h->n_of_type[h->node_type[n]] += h->types[h->node_type[n]].gpus_per_node;
    }
    h->bs.assign(model->bset, model->bset + model->n_bset);
    std::sort(h->bs.begin(), h->bs.end());
    h->bs.erase(std::unique(h->bs.begin(), h->bs.end()), h->bs.end());
    h->derive_links();
    h->derive_durations();
    // stage-time bound keeps the partition weights floor(2^40 / t) positive
    for (const auto& d : h->dur)
      if (d.ok && (i64)model->layers * (d.attn_f + d.mlp_f + d.attn_b + d.mlp_b) + d.emb_f + d.emb_b + d.head_f + d.head_b >= ((i64)1 << 40))
        fail(HSIM_ERANGE, "a stage's compute time reaches 2^40 ns");
    h->ilv = model->interleave > 1 ? model->interleave : 1;
    h->enumerate();
    if (h->N <= 0) fail(HSIM_EINVAL, "InsufficientDevices: the candidate space is empty");
    {  // every 1F1B time <= sum of all op and message weights <= m (L max layer f+g + 2 max emb/head f+g
       // + 2 P max p2p), m <= global batch
      // (V.2: every micro-batch crosses v P boundaries each way, the wraps included)
      const double bound = (double)model->global_batch *
                           ((double)model->layers * h->layer_fb_max + 2.0 * h->ext_max +
                            2.0 * h->ilv * (h->depth_max + 1) * (double)h->c_max);
      if (bound >= 4503599627370496.0) fail(HSIM_ERANGE, "1F1B times may reach 2^52 ns");
    }
    h->prepare();
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) == cudaSuccess && ndev > 0) h->upload();  // else: host-only handle
    else cudaGetLastError();
  } catch (const Fail& f) {
    g_err = f.msg;
    hsim_destroy(h);
    return f.code;
  } catch (const std::bad_alloc&) {
    g_err = "out of host memory";
    hsim_destroy(h);
    return HSIM_ENOMEM;
  }
  *out = h;
  return HSIM_OK;
}

void hsim_destroy(hsim_handle* h) {
  if (!h) return;
  cudaFree(h->d_prefix);
  cudaFree(h->d_bucket);
  cudaFree(h->d_cprefix);
  cudaFree(h->d_cbucket);
  for (int q = 0; q < hsim_handle::NPLAN; ++q)
    if (h->h_plan[q]) cudaFreeHost(h->h_plan[q]);
  cudaFree(h->d_xmask);
  cudaFree(h->d_work);
  cudaFree(h->d_tpl);
  cudaFree(h->d_pool);
  cudaFree(h->d_wtab);
  cudaFree(h->d_node_type);
  cudaFree(h->d_type_nodes);
  cudaFree(h->dT);
  cudaFree(h->d_blk);
  cudaFree(h->d_cells);
  cudaFree(h->d_flow);
  for (int q = 0; q < 2; ++q) {
    cudaFree(h->d_hkeys[q]);
    cudaFree(h->d_hres[q]);
  }
  for (int q = 0; q < hsim_handle::NSIDE; ++q) {
    if (h->side[q]) cudaStreamDestroy(h->side[q]);
    if (h->ev_join[q]) cudaEventDestroy(h->ev_join[q]);
  }
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  for (int q = 0; q < hsim_handle::NPLAN; ++q)
    if (h->ev_plan[q]) cudaEventDestroy(h->ev_plan[q]);
  if (h->ev_done) cudaEventDestroy(h->ev_done);
  for (int q = 0; q < hsim_handle::NEV; ++q)
    if (h->ev_pool[q]) cudaEventDestroy(h->ev_pool[q]);
  delete h;
}

int64_t hsim_space_size(const hsim_handle* h) { return h ? h->N : -1; }
int64_t hsim_n_templates(const hsim_handle* h) { return h ? (int64_t)h->tpl.size() : -1; }
int64_t hsim_template_first(const hsim_handle* h, int64_t k) {
  if (!h || k < 0 || k > (int64_t)h->tpl.size()) return -1;
  return h->prefix[k];
}
int32_t hsim_last_launch_count(const hsim_handle* h) { return h ? h->last_launches : -1; }

int hsim_decode(const hsim_handle* h, int64_t i, char* json, size_t cap) {
  g_err.clear();
  if (!h) { g_err = "NULL handle"; return HSIM_ESTATE; }
  if (i < 0 || i >= h->N) { g_err = "index out of range"; return HSIM_ERANGE; }
  const TplRec& tp = h->tpl[find_template(h->hT, i)];
  ClassSplit cs[MAXC];
  const int st = partition_any(h->hT, tp, i - tp.prefix, cs);
  std::string s = "{\"index\":" + std::to_string(i) + ",\"b\":" + std::to_string(tp.b) + ",\"M\":" + std::to_string(tp.M) +
                  ",\"status\":" + std::to_string(st) + ",\"classes\":[";
  for (int c = 0; c < tp.C; ++c) {
    const CrecHdr* hd = crec_hdr(h->hT, tp.crec[c]);
    const StageRec* sr = crec_stages(h->hT, tp.crec[c]);
    std::vector<std::pair<int, int>> stages;
    for (int q = 0; q < hd->P; ++q) stages.push_back({st_code(sr[q].type, sr[q].type2), sr[q].tp});
    s += c ? ",{" : "{";
    s += "\"D\":" + std::to_string(hd->D) + ",\"subclasses\":" + std::to_string(hd->U) + ",\"stages\":[";
    for (int q = 0; q < hd->P; ++q)
      s += (q ? ",[" : "[") + std::to_string(sr[q].type) + "," + std::to_string(sr[q].tp) +
           (sr[q].type2 >= 0 ? "," + std::to_string(sr[q].type2) : std::string()) + "]";
    s += "],\"layers\":[";
    {
      u32 dig = (u32)(i - tp.prefix);
      for (int c2 = 0; c2 < c; ++c2) dig /= crec_hdr(h->hT, tp.crec[c2])->pw;
      LayerWalk lw = walk(h->hT, hd, dig % hd->pw);
      for (int q = 0; q < hd->P; ++q) s += (q ? "," : "") + std::to_string(lw.next(sr));
    }
    s += "],\"mb\":[";
    if (st == 0)
      for (int r = 0; r < hd->D; ++r) s += (r ? "," : "") + std::to_string(mb_of(cs[c], r));
    s += "],\"place\":[";
    try {
      const auto pl = h->place(hd->D, stages);
      for (int r = 0; r < hd->D; ++r) {
        s += r ? ",[" : "[";
        for (int q = 0; q < hd->P; ++q)
          s += (q ? ",[" : "[") + std::to_string(pl[r][q].node) + "," + std::to_string(pl[r][q].base) +
               (pl[r][q].node2 >= 0 ? "," + std::to_string(pl[r][q].node2) : std::string()) + "]";
        s += "]";
      }
    } catch (const Fail& f) {
      g_err = f.msg;
      return f.code;
    }
    s += "]}";
  }
  s += "]}";
  if (!json || s.size() + 1 > cap) { g_err = "buffer too small"; return HSIM_ERANGE; }
  std::memcpy(json, s.c_str(), s.size() + 1);
  return HSIM_OK;
}

static int check_cands(const hsim_handle* h, const hsim_cands* c, int64_t n) {
  if (!c || n < 0) { g_err = "InvalidValue: cands / n"; return HSIM_EINVAL; }
  if (n == 0 || c->idx) return HSIM_OK;
  if (c->first < 0) { g_err = "index out of range"; return HSIM_ERANGE; }
  int64_t last;
  if (c->block == 0) last = c->first + n - 1;
  else {
    if (c->block < 0 || c->stride < c->block) { g_err = "InvalidValue: block / stride"; return HSIM_EINVAL; }
    last = c->first + ((n - 1) / c->block) * c->stride + (n - 1) % c->block;
  }
  if (last >= h->N) { g_err = "index out of range"; return HSIM_ERANGE; }
  return HSIM_OK;
}

int hsim_eval_batch(hsim_handle* h, const hsim_cands* cands, int64_t n, int64_t* out_ns, void* stream) {
  g_err.clear();
  if (!h) { g_err = "NULL handle"; return HSIM_ESTATE; }
  int rc = check_cands(h, cands, n);
  if (rc) return rc;
  h->last_launches = 0;
  if (n == 0) return HSIM_OK;
  if ((rc = h->ensure_device())) return rc;
  return launch_eval(h, h->dT, cands, n, out_ns, 0, nullptr, nullptr, (cudaStream_t)stream);
}

int hsim_topk(hsim_handle* h, const hsim_cands* cands, int64_t n, int32_t k, int64_t* out_t_ns, int64_t* out_idx,
              int64_t* out_ns, void* stream) {
  g_err.clear();
  if (!h) { g_err = "NULL handle"; return HSIM_ESTATE; }
  if (k < 1 || k > 1024 || !out_t_ns || !out_idx) { g_err = "InvalidValue: k must be 1..1024 with output buffers"; return HSIM_EINVAL; }
  int rc = check_cands(h, cands, n);
  if (rc) return rc;
  h->last_launches = 0;
  if ((rc = h->ensure_device())) return rc;
  return launch_eval(h, h->dT, cands, n, out_ns, k, out_t_ns, out_idx, (cudaStream_t)stream);
}

int hsim_merge_topk(const int64_t* lists, int32_t nlists, int32_t k, int64_t* out_t_ns, int64_t* out_idx, void* stream) {
  g_err.clear();
  if (k < 1 || k > 1024 || nlists < 0 || !out_t_ns || !out_idx || (nlists > 0 && !lists)) {
    g_err = "InvalidValue: merge arguments";
    return HSIM_EINVAL;
  }
  return launch_merge(lists, nlists, k, out_t_ns, out_idx, (cudaStream_t)stream);
}

int hsim_flow_resim(hsim_handle* h, const int64_t* idx, int32_t k, int64_t* out, int64_t* fct, int64_t fct_cap,
                    void* stream) {
  g_err.clear();
  if (!h) { g_err = "NULL handle"; return HSIM_ESTATE; }
  if (k < 0 || k > 1024 || (k > 0 && (!idx || !out)) || fct_cap < 0) {
    g_err = "InvalidValue: k must be 0..1024 with idx and out";
    return HSIM_EINVAL;
  }
  if ((i64)h->md.layers > 256) { g_err = "InvalidValue: flow re-simulation supports up to 256 layers"; return HSIM_EINVAL; }
  if (h->ilv > 1 || h->md.ep_dp || h->md.mixtp || h->md.sync_buckets == 2) { g_err = "InvalidValue: flow re-simulation is defined for the default schedule only (no interleave / ep_dp / mixtp)"; return HSIM_EINVAL; }
  if (k == 0) return HSIM_OK;
  int rc = h->ensure_device();
  if (rc) return rc;
  return launch_flow(h, h->dT, h->hT, idx, k, out, fct, fct_cap, (cudaStream_t)stream);
}

int hsim_set_prune(hsim_handle* h, int on) {
  g_err.clear();
  if (!h) { g_err = "NULL handle"; return HSIM_ESTATE; }
  h->prune = on ? 1 : 0;
  return HSIM_OK;
}

int hsim_set_dedup(hsim_handle* h, int on) {
  g_err.clear();
  if (!h) { g_err = "NULL handle"; return HSIM_ESTATE; }
  h->dedup = on ? 1 : 0;
  return HSIM_OK;
}

int hsim_dedup_active(const hsim_handle* h) {
  g_err.clear();
  if (!h) { g_err = "NULL handle"; return -1; }
  return h->dedup && h->hT.dd_ok && h->ilv <= 1 && !h->md.sync_overlap ? 1 : 0;
}

int64_t hsim_last_sync_units(const hsim_handle* h) {
  g_err.clear();
  if (!h) { g_err = "NULL handle"; return -1; }
  if (!h->d_sync_units || h->ilv > 1) return -1;
  int64_t v = 0;
  if (cudaDeviceSynchronize() != cudaSuccess || cudaMemcpy(&v, h->d_sync_units, 8, cudaMemcpyDeviceToHost) != cudaSuccess) {
    g_err = "cudaMemcpy";
    return -1;
  }
  return v;
}

int64_t hsim_count_cells(const hsim_handle* h, int64_t first, int64_t n) {
  g_err.clear();
  if (!h || first < 0 || n < 0 || first + n > h->N) { g_err = "index out of range"; return -1; }
  if (const_cast<hsim_handle*>(h)->ensure_device()) return -1;
  if (launch_count(const_cast<hsim_handle*>(h), h->dT, first, n, h->d_cells, 0)) return -1;
  int64_t v = 0;
  if (cudaMemcpy(&v, h->d_cells, 8, cudaMemcpyDeviceToHost) != cudaSuccess) { g_err = "cudaMemcpy"; return -1; }
  return v;
}

}  // extern "C"

// scratch accessor for kernels.cu
namespace hsim {
int ensure_work_scratch(hsim_handle* h, size_t entries, int64_t** out) {
  if (entries > h->work_cap) {
    cudaFree(h->d_work);
    h->d_work = nullptr;
    h->work_cap = 0;
    if (cudaMalloc(&h->d_work, entries * 8) != cudaSuccess) { g_err = "cudaMalloc work scratch"; return HSIM_ENOMEM; }
    h->work_cap = entries;
  }
  *out = h->d_work;
  return 0;
}
const Tables& host_tables(const hsim_handle* h) { return h->hT; }
// chunk of candidate i (host copy of the template tables)
static i64 host_chunk_of(const hsim_handle* h, i64 i) {
  const i64 tau = find_template(h->hT, i);
  return h->cprefix[tau] + (i - h->prefix[tau]) / CHUNK;
}
// Per-call chunk plan of a range / block-cyclic candidate list: for range r,
// c0[r] = chunk of its first candidate and pre[r] = #chunks of ranges < r.
// Written to one of NPLAN pinned host buffers [c0 (nr) | pre (nr + 1)] (a
// ring: the host waits only if the buffer's copy from NPLAN calls ago has not
// run yet); *ev = the event to record after the copy.  Returns the total.
i64 host_plan(hsim_handle* h, i64 first, i64 block, i64 stride, i64 n, i64 nr, i64** buf, cudaEvent_t* ev) {
  const int q = h->plan_slot;
  h->plan_slot = (q + 1) % hsim_handle::NPLAN;
  cudaEventSynchronize(h->ev_plan[q]);  // that buffer's previous H2D copy has been consumed
  const size_t need = (size_t)(2 * nr + 1);
  if (need > h->h_plan_cap[q]) {
    if (h->h_plan[q]) cudaFreeHost(h->h_plan[q]);
    h->h_plan[q] = nullptr;
    h->h_plan_cap[q] = 0;
    if (cudaMallocHost(&h->h_plan[q], need * 8) != cudaSuccess) return -1;
    h->h_plan_cap[q] = need;
  }
  i64* c0 = h->h_plan[q];
  i64* pre = h->h_plan[q] + nr;
  i64 acc = 0;
  for (i64 r = 0; r < nr; ++r) {
    const i64 start = block ? first + r * stride : first;
    const i64 len = block ? std::min(block, n - r * block) : n;
    c0[r] = host_chunk_of(h, start);
    pre[r] = acc;
    acc += host_chunk_of(h, start + len - 1) - c0[r] + 1;
  }
  pre[nr] = acc;
  *buf = h->h_plan[q];
  *ev = h->ev_plan[q];
  return acc;
}
// chunk range [c0, c0 + count) of one contiguous candidate range (no staging)
i64 range_chunks(const hsim_handle* h, i64 first, i64 n, i64* c0) {
  *c0 = host_chunk_of(h, first);
  return host_chunk_of(h, first + n - 1) - *c0 + 1;
}
// per-handle cross-call ordering: a call waits for the previous call's work
// (whatever stream it ran on) and records its own end
void call_begin(hsim_handle* h, cudaStream_t st) {
  if (h->done_recorded) cudaStreamWaitEvent(st, h->ev_done, 0);
}
void call_end(hsim_handle* h, cudaStream_t st) {
  cudaEventRecord(h->ev_done, st);
  h->done_recorded = true;
}
int* grid_cache(hsim_handle* h) { return h->grid_cache; }
uint32_t depth_mask(const hsim_handle* h) { return h->pmask_all; }
cudaStream_t side_stream(const hsim_handle* h, int q) { return h->side[q % hsim_handle::NSIDE]; }
cudaEvent_t fork_event(const hsim_handle* h) { return h->ev_fork; }
cudaEvent_t pool_event(const hsim_handle* h, int q) { return h->ev_pool[q % hsim_handle::NEV]; }
cudaEvent_t join_event(const hsim_handle* h, int q) { return h->ev_join[q % hsim_handle::NSIDE]; }
int depth_jobs_max(const hsim_handle* h, int P) { return P >= 0 && P <= FASTP ? h->pcnt_max[P] : 0; }
int64_t depth_jobs_space(const hsim_handle* h, int P) { return P >= 0 && P <= FASTP ? h->depth_jobs_space[P] : 0; }
int stages_max(const hsim_handle* h) { return h->stages_max; }
int sync_overlap(const hsim_handle* h) { return h->md.sync_overlap; }
int interleave_v(const hsim_handle* h) { return h->ilv; }
int ilv_jobs_max(const hsim_handle* h) { return h->ilv_jobs_max; }
int ilv_depth_max(const hsim_handle* h) { return h->ilv_depth_max; }
int sync_buckets(const hsim_handle* h) { return h->md.sync_buckets == 2 ? 2 : 1; }
int prune_enabled(const hsim_handle* h) { return h->prune; }
int dedup_enabled(const hsim_handle* h) { return h->dedup && h->hT.dd_ok; }
int class_max(const hsim_handle* h) { return h->cmax; }
// dedupe hash table of scratch buffer q with at least cap entries (a power of
// two); zeroed when (re)allocated, and K_final clears every key it owns, so
// the table is all-empty between calls
int ensure_hash_scratch(hsim_handle* h, int q, size_t cap, u64** keys, int64_t** res) {
  if (cap > h->hash_cap[q]) {
    cudaFree(h->d_hkeys[q]);
    cudaFree(h->d_hres[q]);
    h->d_hkeys[q] = nullptr;
    h->d_hres[q] = nullptr;
    h->hash_cap[q] = 0;
    if (cudaMalloc(&h->d_hkeys[q], cap * 8) != cudaSuccess || cudaMalloc(&h->d_hres[q], cap * 8) != cudaSuccess ||
        cudaMemset(h->d_hkeys[q], 0, cap * 8) != cudaSuccess) {
      g_err = "cudaMalloc dedupe table";
      return HSIM_ENOMEM;
    }
    h->hash_cap[q] = cap;
  }
  *keys = h->d_hkeys[q];
  *res = h->d_hres[q];
  return 0;
}
void set_sync_counter(hsim_handle* h, i64* p) { h->d_sync_units = p; }
int ensure_block_scratch(hsim_handle* h, size_t entries, int64_t** out) {
  if (entries > h->blk_cap) {
    cudaFree(h->d_blk);
    h->d_blk = nullptr;
    h->blk_cap = 0;
    if (cudaMalloc(&h->d_blk, entries * 8) != cudaSuccess) { g_err = "cudaMalloc block scratch"; return HSIM_ENOMEM; }
    h->blk_cap = entries;
  }
  *out = h->d_blk;
  return 0;
}
int sm_count(const hsim_handle* h) { return h->sm_count; }
int ensure_flow_scratch(hsim_handle* h, size_t bytes, void** out) {
  if (bytes > h->flow_cap) {
    cudaFree(h->d_flow);
    h->d_flow = nullptr;
    h->flow_cap = 0;
    if (cudaMalloc(&h->d_flow, bytes) != cudaSuccess) { g_err = "cudaMalloc flow scratch"; return HSIM_ENOMEM; }
    h->flow_cap = bytes;
  }
  *out = h->d_flow;
  return 0;
}
void set_launches(hsim_handle* h, int n) { h->last_launches = n; }
void set_error(const char* m) { g_err = m; }
}  // namespace hsim
