// Budgeted split-candidate selection on sm_100a.
//
// Replaces splitkit.densify_controller.select_candidates and the helpers it
// calls (/root/reference/pkg/src/splitkit/densify_controller.py:66-106):
// eligibility, the combined score and np.argsort(-score, kind="stable")[:take].
//
// One cooperative (co-resident) launch; every block owns a contiguous index
// range, so block order == index order:
//   pass 0     grad_norm = grad_sum / accum_count (numpy's IEEE division),
//              eligibility, score, and an order-preserving 64-bit key
//              (ascending key == descending score, -0 == +0, NaN last); keys
//              are kept in the workspace (L2-resident) and histogrammed on
//              their top 11 bits.
//   passes 1-5 radix select of the take-th smallest key, 11/11/11/11/9 bits
//              (grid barrier after each histogram; every block resolves the
//              digit redundantly from the merged histogram), stopping early once
//              the take-th key is the last of its bucket (whole bucket taken).
//   final      key < T selected; ties key == T selected in ascending index
//              order up to the remaining budget, using an exclusive scan of
//              per-block tie counts (bit-exact with the stable argsort).
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "igs_common.cuh"

namespace cg = cooperative_groups;

namespace igs {
namespace sel {

constexpr int NT = 512;
constexpr int NBK = 2048;
constexpr int PASSES = 6;
constexpr int U = 4;                     // elements per thread per streaming step
constexpr unsigned long long kIneligible = ~0ull;
constexpr int MAX_GRID = 4096;

struct State {
  unsigned long long n_elig;
  unsigned long long pad[15];
};

struct Params {
  const double* grad_sum;
  long long accum;
  const double* edge;
  long long n;
  double thr;
  int warmup, policy;
  long long take_cap;
  uint8_t* mask;
  long long* counts;
  unsigned long long* keys;
  unsigned* hist;        // PASSES x NBK
  unsigned* blk_ties;    // gridDim
  State* state;
};

__device__ __forceinline__ unsigned long long score_key(double s) {
  if (s != s) return 0xFFF8000000000000ull;   // NaN: after every number
  if (s == 0.0) s = 0.0;                       // -0 ties with +0
  unsigned long long b = (unsigned long long)__double_as_longlong(s);
  unsigned long long u = (b >> 63) ? ~b : (b | 0x8000000000000000ull);  // ascending score
  return ~u;                                                            // ascending key
}

__device__ __forceinline__ int pass_shift(int p) { return p < 5 ? 53 - 11 * p : 0; }
__device__ __forceinline__ unsigned pass_mask(int p) { return p < 5 ? 2047u : 511u; }

struct Smem {
  unsigned h[NBK];
  unsigned warp_sums[32];
  unsigned long long u64[4];
  unsigned u32[4];  // [0] digit, [1] tie scratch, [2] bucket count
};

// Every block: find the digit of rank `rank` in the merged histogram of pass p.
// count: how many keys fall in the chosen digit's bucket.
__device__ void resolve_digit(const Params& P, Smem& s, int p, unsigned long long& prefix,
                              unsigned long long& pmask, unsigned long long& rank,
                              unsigned& count) {
  const unsigned* gh = P.hist + p * NBK;
  constexpr int PER = NBK / NT;
  unsigned loc[PER], sum = 0;
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    loc[k] = __ldcg(&gh[threadIdx.x * PER + k]);
    sum += loc[k];
  }
  unsigned total;
  unsigned before = block_exclusive_scan(sum, s.warp_sums, &total);
  unsigned long long cum = before;
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    if (loc[k] && rank >= cum && rank < cum + loc[k]) {
      s.u32[0] = threadIdx.x * PER + k;
      s.u32[2] = loc[k];
      s.u64[0] = rank - cum;
    }
    cum += loc[k];
  }
  __syncthreads();
  const int sh = pass_shift(p);
  prefix |= (unsigned long long)s.u32[0] << sh;
  pmask |= (unsigned long long)pass_mask(p) << sh;
  rank = s.u64[0];
  count = s.u32[2];
  __syncthreads();
}

__global__ void __launch_bounds__(NT) select_kernel(Params P) {
  cg::grid_group grid = cg::this_grid();
  __shared__ Smem s;
  const long long per_blk = (P.n + gridDim.x - 1) / gridDim.x;
  const long long lo = min((long long)blockIdx.x * per_blk, P.n);
  const long long hi = min(lo + per_blk, P.n);
  const double inv_none = 0.0;

  // pass 0: keys + top-digit histogram + eligible count
  for (int i = threadIdx.x; i < NBK; i += NT) s.h[i] = 0;
  __syncthreads();
  unsigned elig = 0;
  const bool need_edge = P.warmup || P.policy != IGS_POLICY_GRAD;
  for (long long i0 = lo + threadIdx.x; i0 < hi; i0 += U * NT) {  // U per thread, loads first
    double gs[U], ed[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long i = i0 + u * NT;
      gs[u] = i < hi ? __ldcs(P.grad_sum + i) : 0.0;
      ed[u] = (i < hi && need_edge) ? __ldcs(P.edge + i) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long i = i0 + u * NT;
      if (i >= hi) break;
      double g = P.accum ? gs[u] / (double)P.accum : inv_none;
      bool e = P.warmup || g > P.thr;
      double sc;
      if (P.warmup || P.policy == IGS_POLICY_EDGE) sc = ed[u];
      else if (P.policy == IGS_POLICY_GRAD) sc = g;
      else sc = ed[u] * g;
      unsigned long long k = e ? score_key(sc) : kIneligible;
      P.keys[i] = k;
      if (e) {
        ++elig;
        atomicAdd(&s.h[k >> 53], 1u);
      }
    }
  }
  elig = __reduce_add_sync(0xffffffffu, elig);
  if (lane_id() == 0 && elig) atomicAdd(&P.state->n_elig, (unsigned long long)elig);
  __syncthreads();
  for (int i = threadIdx.x; i < NBK; i += NT)
    if (s.h[i]) atomicAdd(&P.hist[i], s.h[i]);
  grid.sync();

  const unsigned long long n_elig = __ldcg(&P.state->n_elig);
  const unsigned long long take =
      n_elig < (unsigned long long)P.take_cap ? n_elig : (unsigned long long)P.take_cap;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    P.counts[0] = (long long)n_elig;
    P.counts[1] = (long long)take;
  }
  if (take == 0) {  // uniform across the grid
    for (long long i = lo + threadIdx.x; i < hi; i += NT) P.mask[i] = 0;
    return;
  }
  unsigned long long prefix = 0, pmask = 0, rank = take - 1;
  unsigned count = 0;
  resolve_digit(P, s, 0, prefix, pmask, rank, count);
  // Early exit (uniform over the grid): once the take-th key is the LAST of its bucket, the
  // whole bucket is selected and no tie needs ranking -- the mask is (key & pmask) <= prefix.
  bool whole = rank + 1 == count;
  for (int p = 1; p < PASSES && !whole; ++p) {
    for (int i = threadIdx.x; i < NBK; i += NT) s.h[i] = 0;
    __syncthreads();
    const int sh = pass_shift(p);
    const unsigned dm = pass_mask(p);
    for (long long i0 = lo + threadIdx.x; i0 < hi; i0 += U * NT) {
      unsigned long long kv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) kv[u] = i0 + u * NT < hi ? __ldcg(&P.keys[i0 + u * NT]) : kIneligible;
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (kv[u] != kIneligible && (kv[u] & pmask) == prefix) atomicAdd(&s.h[(kv[u] >> sh) & dm], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < NBK; i += NT)
      if (s.h[i]) atomicAdd(&P.hist[p * NBK + i], s.h[i]);
    grid.sync();
    resolve_digit(P, s, p, prefix, pmask, rank, count);
    whole = rank + 1 == count;
  }
  if (whole) {
    for (long long i = lo + threadIdx.x; i < hi; i += NT) {
      const unsigned long long k = __ldcg(&P.keys[i]);
      P.mask[i] = k != kIneligible && (k & pmask) <= prefix;
    }
    return;
  }
  const unsigned long long T = prefix;
  const unsigned long long need_ties = rank + 1;  // ties of T inside the top `take`

  // per-block tie counts
  unsigned ties = 0;
  for (long long i0 = lo + threadIdx.x; i0 < hi; i0 += U * NT) {
    unsigned long long kv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) kv[u] = i0 + u * NT < hi ? __ldcg(&P.keys[i0 + u * NT]) : ~T;
#pragma unroll
    for (int u = 0; u < U; ++u) ties += (kv[u] == T);
  }
  ties = __reduce_add_sync(0xffffffffu, ties);
  if (threadIdx.x == 0) s.u32[1] = 0;
  __syncthreads();
  if (lane_id() == 0 && ties) atomicAdd(&s.u32[1], ties);
  __syncthreads();
  if (threadIdx.x == 0) P.blk_ties[blockIdx.x] = s.u32[1];
  grid.sync();
  // exclusive prefix of the tie counts of the blocks before this one
  unsigned long long before = 0;
  for (unsigned b = threadIdx.x; b < blockIdx.x; b += NT) before += __ldcg(&P.blk_ties[b]);
  before = __reduce_add_sync(0xffffffffu, (unsigned)before);
  if (threadIdx.x == 0) s.u64[1] = 0;
  __syncthreads();
  if (lane_id() == 0 && before) atomicAdd(&s.u64[1], before);
  __syncthreads();
  unsigned long long run = s.u64[1];
  // U-element steps; the tie scan (in index order) only runs for steps that hold a tie
  for (long long c0 = lo; c0 < hi; c0 += U * NT) {
    unsigned long long kv[U];
    int any = 0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long i = c0 + u * NT + threadIdx.x;
      kv[u] = i < hi ? __ldcg(&P.keys[i]) : kIneligible;
      any |= kv[u] == T;
    }
    if (!__syncthreads_or(any)) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long long i = c0 + u * NT + threadIdx.x;
        if (i < hi) P.mask[i] = kv[u] < T;
      }
      continue;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long i = c0 + u * NT + threadIdx.x;
      const unsigned is_tie = (kv[u] == T) ? 1u : 0u;
      unsigned tot;
      const unsigned ex = block_exclusive_scan(is_tie, s.warp_sums, &tot);
      if (i < hi) P.mask[i] = (kv[u] < T) || (is_tie && run + ex < need_ties);
      run += tot;
    }
  }
}

struct Layout {
  size_t keys, hist, blk, state, total;
};

Layout layout(long long n, int grid) {
  Layout L;
  size_t off = 0;
  L.state = off;
  off += 256;
  L.hist = off;
  off = align_up(off + sizeof(unsigned) * NBK * PASSES, 256);
  L.blk = off;
  off = align_up(off + sizeof(unsigned) * (size_t)grid, 256);
  L.keys = off;
  off = align_up(off + sizeof(unsigned long long) * (size_t)n, 256);
  L.total = off;
  return L;
}

int max_grid() {
  static int cached = -1;
  if (cached < 0) {
    int bps = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, select_kernel, NT, 0) != cudaSuccess)
      return 0;
    cached = bps * sm_count();
  }
  return cached;
}

}  // namespace sel
}  // namespace igs

using namespace igs;

extern "C" {

int igs_select_workspace_bytes(int64_t n, size_t* bytes) {
  if (!bytes || n < 0) return IGS_ERR_ARGUMENT;
  *bytes = sel::layout(n, sel::MAX_GRID).total;
  return IGS_OK;
}

int igs_select_candidates(const double* grad_sum, int64_t accum_count, const double* edge_score,
                          int64_t n, double grad_threshold, int warmup, int policy,
                          int64_t take_cap, uint8_t* mask, int64_t* counts, void* workspace,
                          size_t workspace_bytes, void* stream) {
  if (n < 0 || !counts || take_cap < 0 || accum_count < 0) return IGS_ERR_ARGUMENT;
  if (policy < 0 || policy > 2) return IGS_ERR_ARGUMENT;
  cudaStream_t st = (cudaStream_t)stream;
  if (n == 0) {
    IGS_CUDA_TRY(cudaMemsetAsync(counts, 0, 2 * sizeof(int64_t), st));
    return IGS_OK;
  }
  if (!grad_sum || !edge_score || !mask) return IGS_ERR_ARGUMENT;
  int gmax = sel::max_grid();
  if (gmax <= 0) return IGS_ERR_CUDA;
  long long want = (n + sel::NT * 4 - 1) / (sel::NT * 4);  // >= 4 elements per thread
  int grid = (int)(want < gmax ? want : gmax);
  if (grid > sel::MAX_GRID) grid = sel::MAX_GRID;
  if (grid < 1) grid = 1;
  sel::Layout L = sel::layout(n, sel::MAX_GRID);
  if (!workspace || workspace_bytes < L.total) return IGS_ERR_WORKSPACE;
  char* w = (char*)workspace;
  IGS_CUDA_TRY(cudaMemsetAsync(w, 0, L.blk, st));  // state + histograms
  sel::Params P;
  P.grad_sum = grad_sum;
  P.accum = accum_count;
  P.edge = edge_score;
  P.n = n;
  P.thr = grad_threshold;
  P.warmup = warmup;
  P.policy = policy;
  P.take_cap = take_cap;
  P.mask = mask;
  P.counts = (long long*)counts;
  P.keys = (unsigned long long*)(w + L.keys);
  P.hist = (unsigned*)(w + L.hist);
  P.blk_ties = (unsigned*)(w + L.blk);
  P.state = (sel::State*)(w + L.state);
  void* args[] = {&P};
  IGS_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)sel::select_kernel, dim3(grid),
                                           dim3(sel::NT), args, 0, st));
  return IGS_OK;
}

}  // extern "C"
