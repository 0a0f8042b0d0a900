// kernels.cu — the hot path on the B200 (sm_100a).
//
// K0 k_plan   (1 block): maps the candidate list (a range, or a block-cyclic
//             set of ranges) onto template-aligned chunks of <= 32 candidates
//             and resets the work counter.
// K1 k_eval   (persistent, grid = SMs x resident blocks): each warp pulls a
//             chunk with one atomicAdd, so its 32 lanes share one template
//             (same classes, depths, sub-classes: no divergence); lane = one
//             candidate: decode -> partition -> stage durations -> 1F1B
//             max-plus (register-resident for depth <= 8) -> gradient sync.
//             Results are stored coalesced; in top-k mode each warp keeps a
//             sorted top-k list (threshold-filtered insertion).
//             Explicit index lists (idx != NULL) use 32 list entries per warp.
// K3 k_merge  (1 block): merges the per-warp sorted lists (each abandoned at
//             its first element above the running threshold).
// K_count     evaluation that reduces the number of 1F1B cells (algorithmic
//             work for the ALU-roofline fraction).
#include <cuda_runtime.h>

#include "hsim.h"
#include "hsim_core.cuh"

namespace hsim {

int ensure_block_scratch(hsim_handle* h, size_t entries, int64_t** out);
int ensure_work_scratch(hsim_handle* h, size_t entries, int64_t** out);
const Tables& host_tables(const hsim_handle* h);
int sm_count(const hsim_handle* h);
void set_launches(hsim_handle* h, int n);
void set_error(const char* m);

#ifndef HSIM_MINB
#define HSIM_MINB 1
#endif
constexpr int NT = 128;         // threads per block of K1
constexpr int WPB = NT / 32;    // warps per block
constexpr int MT = 256;         // threads of K3
constexpr int KMAX = 1024;      // max k
constexpr i64 KEY_INF = INT64_MAX;
constexpr unsigned FULL = 0xffffffffu;

struct Cands {
  const i64* idx;
  i64 first, block, stride, n;
};

__device__ __forceinline__ bool key_less(i64 t1, i64 i1, i64 t2, i64 i2) {
  return t1 < t2 || (t1 == t2 && i1 < i2);
}

__device__ void load_tables(Tables& sT, const Tables* __restrict__ gT) {
  const int words = sizeof(Tables) / 8;
  const i64* src = (const i64*)gT;
  i64* dst = (i64*)&sT;
  for (int w = threadIdx.x; w < words; w += blockDim.x) dst[w] = src[w];
  __syncthreads();
}

__device__ __forceinline__ i64 chunk_of(const Tables& T, i64 i) {
  const i64 tau = find_template(T, i);
  return T.tpl_cprefix[tau] + (i - T.tpl_prefix[tau]) / CHUNK;
}

// work scratch layout: [0] counter, [1] total items, [2 .. 2+nr) c0, [2+nr .. 3+2nr) prefix
__global__ void __launch_bounds__(1024) k_plan(const Tables* __restrict__ gT, Cands c, i64 nr, i64* __restrict__ work) {
  __shared__ Tables sT;
  __shared__ i64 carry_s;
  __shared__ i64 part[1024];
  load_tables(sT, gT);
  i64* c0 = work + 2;
  i64* pre = work + 2 + nr;
  if (threadIdx.x == 0) carry_s = 0;
  __syncthreads();
  for (i64 base = 0; base < nr; base += 1024) {
    const i64 r = base + threadIdx.x;
    i64 cnt = 0;
    if (r < nr) {
      const i64 start = c.block ? c.first + r * c.stride : c.first;
      const i64 len = c.block ? imin(c.block, c.n - r * c.block) : c.n;
      const i64 a = chunk_of(sT, start), b = chunk_of(sT, start + len - 1);
      c0[r] = a;
      cnt = b - a + 1;
    }
    part[threadIdx.x] = cnt;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {  // inclusive scan
      const i64 v = threadIdx.x >= off ? part[threadIdx.x - off] : 0;
      __syncthreads();
      part[threadIdx.x] += v;
      __syncthreads();
    }
    if (r < nr) pre[r] = carry_s + part[threadIdx.x] - cnt;
    __syncthreads();
    if (threadIdx.x == 1023) carry_s += part[1023];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    pre[nr] = carry_s;
    work[0] = 0;
    work[1] = carry_s;
  }
}

// --- per-warp top-k list in global memory: [k times | k indices], sorted ----------
struct WarpTopK {
  i64* wl;
  int k, cnt;
  i64 thrT, thrI;
};

__device__ void warp_offer(WarpTopK& w, i64 t, i64 i, bool valid) {
  const int lane = threadIdx.x & 31;
  const bool cand = valid && (w.cnt < w.k || key_less(t, i, w.thrT, w.thrI));
  unsigned mask = __ballot_sync(FULL, cand);
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
}

__global__ void __launch_bounds__(NT, HSIM_MINB) k_eval(const Tables* __restrict__ gT, Cands c, i64 nr, i64* __restrict__ work,
                                             i64* __restrict__ out, int k, i64* __restrict__ lists) {
  __shared__ Tables sT;
  load_tables(sT, gT);
  const int lane = threadIdx.x & 31;
  const i64 wid = (i64)blockIdx.x * WPB + (threadIdx.x >> 5);
  WarpTopK tk{lists ? lists + wid * 2 * k : nullptr, k, 0, KEY_INF, KEY_INF};
  const i64* c0 = work + 2;
  const i64* pre = work + 2 + nr;
  const i64 total = c.idx ? (c.n + 31) / 32 : work[1];
  for (;;) {
    i64 item = 0;
    if (lane == 0) item = atomicAdd((unsigned long long*)work, 1ull);
    item = __shfl_sync(FULL, item, 0);
    if (item >= total) break;
    i64 t = -1, i = -1, T = INT64_MIN, tau = -1;
    bool valid;
    if (c.idx) {
      t = item * 32 + lane;
      valid = t < c.n;
      if (valid) {
        i = c.idx[t];
        if (i >= 0 && i < sT.N) tau = find_template(sT, i);
      }
    } else {
      const i64 r = bsearch_le(pre, nr, item);
      const i64 g = c0[r] + (item - pre[r]);
      tau = bsearch_le(sT.tpl_cprefix, sT.n_tpl, g);
      const i64 lo = sT.tpl_prefix[tau] + (g - sT.tpl_cprefix[tau]) * CHUNK;
      const i64 start = c.block ? c.first + r * c.stride : c.first;
      const i64 len = c.block ? imin(c.block, c.n - r * c.block) : c.n;
      const i64 end = imin(start + len, sT.tpl_prefix[tau + 1]);
      i = lo + lane;
      valid = i >= start && i < end;
      if (valid) t = (c.block ? r * c.block : 0) + (i - start);
    }
    // evaluate each template present in the warp with warp-uniform code
    // (chunk mode: exactly one; explicit lists: lanes grouped by template)
    unsigned todo = __ballot_sync(FULL, tau >= 0);
    while (todo) {
      const i64 tg = __shfl_sync(FULL, tau, __ffs(todo) - 1);
      const bool in_g = tau == tg;
      todo &= ~__ballot_sync(FULL, in_g);
      const TplRec tp = sT.tpl[tg];
      const i64 Tg = eval_group(sT, tp, i - tp.prefix, in_g);
      if (in_g) T = Tg;
    }
    if (valid && out) out[t] = T;
    if (k) warp_offer(tk, T, i, valid && T >= 0);
  }
  if (k) {  // pad the list
    for (int a = tk.cnt + lane; a < k; a += 32) { tk.wl[a] = KEY_INF; tk.wl[k + a] = -1; }
  }
}

// --- K3: shared-memory running top-k over sorted lists ----------------------------
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

__global__ void __launch_bounds__(MT) k_merge(const i64* __restrict__ blk, int nblk, int k, i64* __restrict__ out_t,
                                              i64* __restrict__ out_i) {
  extern __shared__ __align__(16) unsigned char dyn[];
  TopK& tk = *reinterpret_cast<TopK*>(dyn);
  if (threadIdx.x == 0) tk.count = 0;
  __syncthreads();
  for (int b = 0; b < nblk; ++b) {
    const i64* bt = blk + (i64)b * 2 * k;
    for (int a0 = 0; a0 < k; a0 += MT) {
      // each list is sorted: stop at its first element that cannot enter
      const i64 t0 = bt[a0], i0 = bt[k + a0];
      if (t0 == KEY_INF) break;
      if (tk.count >= k && !key_less(t0, i0, tk.lt[k - 1], tk.li[k - 1])) break;
      const int a = a0 + threadIdx.x;
      const bool v = a < k && bt[a] != KEY_INF;
      topk_offer(tk, k, v ? bt[a] : 0, v ? bt[k + a] : 0, v);
    }
  }
  __syncthreads();
  for (int a = threadIdx.x; a < k; a += MT) {
    out_t[a] = a < tk.count ? tk.lt[a] : KEY_INF;
    out_i[a] = a < tk.count ? tk.li[a] : -1;
  }
}

__global__ void __launch_bounds__(256) k_count(const Tables* __restrict__ gT, i64 first, i64 n, unsigned long long* acc) {
  __shared__ Tables sT;
  load_tables(sT, gT);
  unsigned long long local = 0;
  const i64 step = (i64)gridDim.x * 256;
  for (i64 t = (i64)blockIdx.x * 256 + threadIdx.x; t < n; t += step) {
    i64 cells = 0;
    if (eval_candidate(sT, first + t, &cells) >= 0) local += (unsigned long long)cells;
  }
  atomicAdd(acc, local);
}

static int eval_grid(const hsim_handle* h) {
  static int per_sm = 0;
  if (!per_sm) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_eval, NT, 0) != cudaSuccess || per_sm < 1) per_sm = 1;
  }
  return sm_count(h) * per_sm;
}

static void merge_attr() {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_merge, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(TopK));
    attr = true;
  }
}

int launch_eval(hsim_handle* h, const Tables* dT, const hsim_cands* cc, int64_t n, int64_t* out_ns, int32_t k,
                int64_t* out_t, int64_t* out_i, cudaStream_t st) {
  Cands c{cc->idx, cc->first, cc->block, cc->stride, n};
  const int grid = eval_grid(h);
  const i64 nr = c.idx ? 0 : (c.block ? (n + c.block - 1) / c.block : 1);
  i64* work = nullptr;
  if (ensure_work_scratch(h, (size_t)(3 + 2 * nr), &work)) return HSIM_ENOMEM;
  i64* lists = nullptr;
  if (k && ensure_block_scratch(h, (size_t)grid * WPB * 2 * k, &lists)) return HSIM_ENOMEM;
  int launches = 0;
  if (n > 0) {
    if (c.idx) {
      cudaMemsetAsync(work, 0, 8, st);
    } else {
      k_plan<<<1, 1024, 0, st>>>(dT, c, nr, work);
      ++launches;
    }
    k_eval<<<grid, NT, 0, st>>>(dT, c, nr, work, out_ns, k, lists);
    ++launches;
  }
  if (k) {
    merge_attr();
    // n == 0 merges no list and only writes the (INT64_MAX, -1) padding
    k_merge<<<1, MT, sizeof(TopK), st>>>(lists, n > 0 ? grid * WPB : 0, k, out_t, out_i);
    ++launches;
  }
  set_launches(h, launches);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(cudaGetErrorString(e));
    return HSIM_ECUDA;
  }
  return HSIM_OK;
}

int launch_merge(const int64_t* lists, int32_t nlists, int32_t k, int64_t* out_t, int64_t* out_i, cudaStream_t st) {
  merge_attr();
  k_merge<<<1, MT, sizeof(TopK), st>>>(lists, nlists, k, out_t, out_i);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(cudaGetErrorString(e));
    return HSIM_ECUDA;
  }
  return HSIM_OK;
}

int launch_count(const Tables* dT, int64_t first, int64_t n, int64_t* d_acc, cudaStream_t st) {
  cudaMemsetAsync(d_acc, 0, 8, st);
  if (n > 0) k_count<<<148 * 4, 256, 0, st>>>(dT, first, n, (unsigned long long*)d_acc);
  cudaError_t e = cudaStreamSynchronize(st);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(cudaGetErrorString(e));
    return HSIM_ECUDA;
  }
  return 0;
}

}  // namespace hsim
