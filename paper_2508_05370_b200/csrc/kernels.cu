// kernels.cu — the hot path on the B200 (sm_100a).
//
// K1 k_eval: persistent grid (a multiple of the 148 SMs); each thread
//    evaluates one candidate per iteration (hsim_core.cuh: decode ->
//    partition -> stage durations -> 1F1B max-plus -> sync), writes its int64
//    result with coalesced stores and, in top-k mode, feeds a block-level
//    top-k (threshold filter + bitonic sort + rank merge in shared memory).
// K3 k_merge: one block merges the per-block top-k lists (sorted, so each
//    list is abandoned at its first element above the running threshold).
// K_count: same evaluation, reduces the number of simulated 1F1B cells (the
//    algorithmic work behind the ALU-roofline fraction).
#include <cuda_runtime.h>

#include "hsim.h"
#include "hsim_core.cuh"

namespace hsim {

int ensure_block_scratch(hsim_handle* h, size_t entries, int64_t** out);
int sm_count(const hsim_handle* h);
void set_launches(hsim_handle* h, int n);
void set_error(const char* m);

constexpr int NT = 256;         // threads per block
constexpr int KMAX = 1024;      // max k
constexpr i64 KEY_INF = INT64_MAX;

struct Cands {
  const i64* idx;
  i64 first, block, stride;
};

__device__ __forceinline__ i64 cand_index(const Cands& c, i64 t) {
  if (c.idx) return c.idx[t];
  if (c.block == 0) return c.first + t;
  return c.first + (t / c.block) * c.stride + (t % c.block);
}

__device__ __forceinline__ bool key_less(i64 t1, i64 i1, i64 t2, i64 i2) {
  return t1 < t2 || (t1 == t2 && i1 < i2);
}

// Shared-memory running top-k of one block.
struct TopK {
  i64 lt[KMAX], li[KMAX];   // sorted ascending, `count` valid
  i64 nt[KMAX], ni[KMAX];   // merge target
  i64 bt[NT], bi[NT];       // incoming batch
  int count, nbuf;
};

// Offer one (t, i) per thread (valid == false: nothing).  All threads of the
// block must call it.
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
  // bitonic sort of the batch (NT elements)
  for (int size = 2; size <= NT; size <<= 1)
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
  for (int a = tid; a < cnt; a += NT) {
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
  for (int a = tid; a < ncnt; a += NT) { s.lt[a] = s.nt[a]; s.li[a] = s.ni[a]; }
  if (tid == 0) s.count = ncnt;
  __syncthreads();
}

__device__ void load_tables(Tables& sT, const Tables* __restrict__ gT) {
  const int words = sizeof(Tables) / 8;
  const i64* src = (const i64*)gT;
  i64* dst = (i64*)&sT;
  for (int w = threadIdx.x; w < words; w += blockDim.x) dst[w] = src[w];
  __syncthreads();
}

__global__ void __launch_bounds__(NT) k_eval(const Tables* __restrict__ gT, Cands c, i64 n, i64* __restrict__ out,
                                             int k, i64* __restrict__ blk) {
  __shared__ Tables sT;
  extern __shared__ __align__(16) unsigned char dyn[];
  TopK& tk = *reinterpret_cast<TopK*>(dyn);
  load_tables(sT, gT);
  if (k) {
    if (threadIdx.x == 0) tk.count = 0;
    __syncthreads();
  }
  const i64 step = (i64)gridDim.x * NT;
  for (i64 base = (i64)blockIdx.x * NT; base < n; base += step) {
    const i64 t = base + threadIdx.x;
    i64 i = -1, T = INT64_MIN;
    if (t < n) {
      i = cand_index(c, t);
      T = eval_candidate(sT, i, nullptr);
      if (out) out[t] = T;
    }
    if (k) topk_offer(tk, k, T, i, t < n && T >= 0);
  }
  if (k) {
    __syncthreads();
    i64* bt = blk + (i64)blockIdx.x * 2 * k;
    for (int a = threadIdx.x; a < k; a += NT) {
      bt[a] = a < tk.count ? tk.lt[a] : KEY_INF;
      bt[k + a] = a < tk.count ? tk.li[a] : -1;
    }
  }
}

__global__ void __launch_bounds__(NT) k_merge(const i64* __restrict__ blk, int nblk, int k, i64* __restrict__ out_t,
                                              i64* __restrict__ out_i) {
  extern __shared__ __align__(16) unsigned char dyn[];
  TopK& tk = *reinterpret_cast<TopK*>(dyn);
  if (threadIdx.x == 0) tk.count = 0;
  __syncthreads();
  for (int b = 0; b < nblk; ++b) {
    const i64* bt = blk + (i64)b * 2 * k;
    for (int a0 = 0; a0 < k; a0 += NT) {
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
  for (int a = threadIdx.x; a < k; a += NT) {
    out_t[a] = a < tk.count ? tk.lt[a] : KEY_INF;
    out_i[a] = a < tk.count ? tk.li[a] : -1;
  }
}

__global__ void __launch_bounds__(NT) k_count(const Tables* __restrict__ gT, i64 first, i64 n, unsigned long long* acc) {
  __shared__ Tables sT;
  load_tables(sT, gT);
  unsigned long long local = 0;
  const i64 step = (i64)gridDim.x * NT;
  for (i64 t = (i64)blockIdx.x * NT + threadIdx.x; t < n; t += step) {
    i64 cells = 0;
    if (eval_candidate(sT, first + t, &cells) >= 0) local += (unsigned long long)cells;
  }
  atomicAdd(acc, local);
}

static int grid_for(const hsim_handle* h, i64 n) {
  const i64 want = (n + NT - 1) / NT;
  const i64 cap = (i64)sm_count(h) * 4;  // 4 resident blocks of 256 per SM
  return (int)(want < cap ? (want > 0 ? want : 1) : cap);
}

int launch_eval(hsim_handle* h, const Tables* dT, const hsim_cands* cc, int64_t n, int64_t* out_ns, int32_t k,
                int64_t* out_t, int64_t* out_i, cudaStream_t st) {
  Cands c{cc->idx, cc->first, cc->block, cc->stride};
  const int grid = grid_for(h, n);
  i64* blk = nullptr;
  size_t smem = 0;
  if (k) {
    if (ensure_block_scratch(h, (size_t)grid * 2 * k, &blk)) return HSIM_ENOMEM;
    smem = sizeof(TopK);
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_eval, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(TopK));
      cudaFuncSetAttribute(k_merge, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(TopK));
      attr = true;
    }
  }
  if (n > 0) k_eval<<<grid, NT, smem, st>>>(dT, c, n, out_ns, k, blk);
  int launches = n > 0 ? 1 : 0;
  if (k) {
    // n == 0 merges no list and only writes the (INT64_MAX, -1) padding
    k_merge<<<1, NT, smem, st>>>(blk, n > 0 ? grid : 0, k, out_t, out_i);
    launches += 1;
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
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_merge, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(TopK));
    attr = true;
  }
  k_merge<<<1, NT, sizeof(TopK), st>>>(lists, nlists, k, out_t, out_i);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(cudaGetErrorString(e));
    return HSIM_ECUDA;
  }
  return HSIM_OK;
}

int launch_count(const Tables* dT, int64_t first, int64_t n, int64_t* d_acc, cudaStream_t st) {
  cudaMemsetAsync(d_acc, 0, 8, st);
  if (n > 0) k_count<<<148 * 4, NT, 0, st>>>(dT, first, n, (unsigned long long*)d_acc);
  cudaError_t e = cudaStreamSynchronize(st);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(cudaGetErrorString(e));
    return HSIM_ECUDA;
  }
  return 0;
}

}  // namespace hsim
