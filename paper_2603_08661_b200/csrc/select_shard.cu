// Sharded budgeted selection: the per-rank kernels of the multi-GPU protocol of SURVEY.md 8(e).
//
// Every rank owns a contiguous index range [lo_r, hi_r) of the global Gaussian array, so
// global index order == (rank, local index) order.  The result is bit-identical to a
// single-device select_candidates over the concatenated arrays
// (/root/reference/pkg/src/splitkit/densify_controller.py:80-106, stable argsort :104).
//
// Per densify step, all stream-ordered on the device (no host round trip until the caller
// reads the event counts):
//   keys      key = order-preserving 64-bit image of the score (ascending key ==
//             descending score, -0 == +0, NaN last; ineligible = ~0); local histogram of the
//             top 16 key bits plus the local eligible count          -> all-reduce (sum)
//   resolve   (1 thread block) round 0: take = min(#eligible, take_cap); every round: the
//             16-bit digit holding rank take-1 of the merged histogram, narrowing the
//             prefix; after round 3 the prefix is the threshold key T
//   hist      rounds 1..3: local histogram of the next 16 bits among keys matching the
//             prefix                                                  -> all-reduce (sum)
//   ties      per-block counts of key == T and the local total        -> all-gather
//   finalize  mask = key < T, or key == T and (ties on lower ranks + ties before it on this
//             rank) < need_ties (ties broken by ascending global index)
// Four 256 KB all-reduces and one 8-byte all-gather per step; the caller issues them
// (torch.distributed / NCCL) between the launches, on the same stream.
#include <cuda_runtime.h>
#include <stdint.h>

#include "igs_common.cuh"

namespace igs {
namespace shard {

constexpr int NT = 1024;
constexpr int NBINS = 1 << 16;
constexpr int ROUNDS = 4;
constexpr int U = 4;                          // elements per thread per streaming step
constexpr unsigned long long kIneligible = ~0ull;
constexpr long long MAX_PER_BLOCK = 65535;   // 16-bit packed shared-memory counters
constexpr int SMEM_BYTES = NBINS * 2;        // two 16-bit bins per 32-bit word

struct State {
  unsigned long long prefix, pmask, rank, take, n_elig, T, need_ties, local_ties;
  int status;                                 // 0 running, 1 nothing to select
  int grid;
  int pad[14];
};

struct Layout {
  size_t state, blk, keys, total;
};

inline int grid_for(long long n) {
  long long g = (n + MAX_PER_BLOCK - 1) / MAX_PER_BLOCK;
  long long want = (n + 4 * NT - 1) / (4 * NT);
  long long sms = sm_count() > 0 ? sm_count() : 148;
  if (want > sms) want = sms;
  if (g < want) g = want;
  if (g < 1) g = 1;
  return (int)g;
}

inline Layout layout(long long n) {
  Layout L;
  size_t off = 0;
  L.state = off;
  off += 256;
  L.blk = off;
  const long long gmax = (n + MAX_PER_BLOCK - 1) / MAX_PER_BLOCK + 4096;
  off = align_up(off + sizeof(unsigned) * (size_t)gmax, 256);
  L.keys = off;
  off = align_up(off + sizeof(unsigned long long) * (size_t)n, 256);
  L.total = off;
  return L;
}

__device__ __forceinline__ unsigned long long score_key(double s) {
  if (s != s) return 0xFFF8000000000000ull;
  if (s == 0.0) s = 0.0;
  unsigned long long b = (unsigned long long)__double_as_longlong(s);
  unsigned long long u = (b >> 63) ? ~b : (b | 0x8000000000000000ull);
  return ~u;
}

__device__ __forceinline__ int round_shift(int r) { return 48 - 16 * r; }

__device__ __forceinline__ void block_range(long long n, long long& lo, long long& hi) {
  const long long per = (n + gridDim.x - 1) / gridDim.x;
  lo = min((long long)blockIdx.x * per, n);
  hi = min(lo + per, n);
}

__device__ __forceinline__ void smem_hist_add(unsigned* h, unsigned d) {
  atomicAdd(&h[d >> 1], 1u << ((d & 1u) << 4));
}

__device__ void smem_hist_flush(unsigned* h, int* out) {
  __syncthreads();
  for (int i = threadIdx.x; i < NBINS / 2; i += NT) {
    const unsigned v = h[i];
    if (v & 0xffffu) atomicAdd(&out[2 * i], (int)(v & 0xffffu));
    if (v >> 16) atomicAdd(&out[2 * i + 1], (int)(v >> 16));
  }
}

struct KeyParams {
  const double* grad_sum;
  long long accum;
  const double* edge;
  long long n;
  double thr;
  int warmup, policy;
  unsigned long long* keys;
  int* hist;      // NBINS + 1 (last: eligible count)
};

__global__ void __launch_bounds__(NT) keys_kernel(KeyParams P) {
  extern __shared__ unsigned h[];
  for (int i = threadIdx.x; i < NBINS / 2; i += NT) h[i] = 0;
  __syncthreads();
  long long lo, hi;
  block_range(P.n, lo, hi);
  unsigned elig = 0;
  const bool need_edge = P.warmup || P.policy != IGS_POLICY_GRAD;
  // U elements per thread per step, every load issued before the arithmetic
  for (long long i0 = lo + threadIdx.x; i0 < hi; i0 += U * NT) {
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
      const double g = P.accum ? gs[u] / (double)P.accum : 0.0;
      const bool e = P.warmup || g > P.thr;
      double sc;
      if (P.warmup || P.policy == IGS_POLICY_EDGE) sc = ed[u];
      else if (P.policy == IGS_POLICY_GRAD) sc = g;
      else sc = ed[u] * g;
      const unsigned long long k = e ? score_key(sc) : kIneligible;
      P.keys[i] = k;
      if (e) {
        ++elig;
        smem_hist_add(h, (unsigned)(k >> 48));
      }
    }
  }
  elig = __reduce_add_sync(0xffffffffu, elig);
  if (lane_id() == 0 && elig) atomicAdd(&P.hist[NBINS], (int)elig);
  smem_hist_flush(h, P.hist);
}

__global__ void __launch_bounds__(NT) hist_kernel(const unsigned long long* __restrict__ keys,
                                                  long long n, int round, const State* st,
                                                  int* hist) {
  if (st->status) return;
  extern __shared__ unsigned h[];
  for (int i = threadIdx.x; i < NBINS / 2; i += NT) h[i] = 0;
  __syncthreads();
  const unsigned long long prefix = st->prefix, pmask = st->pmask;
  const int sh = round_shift(round);
  long long lo, hi;
  block_range(n, lo, hi);
  for (long long i0 = lo + threadIdx.x; i0 < hi; i0 += U * NT) {
    unsigned long long kv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) kv[u] = i0 + u * NT < hi ? keys[i0 + u * NT] : kIneligible;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const unsigned long long k = kv[u];
      if (k != kIneligible && (k & pmask) == prefix)
        smem_hist_add(h, (unsigned)((k >> sh) & 0xffffu));
    }
  }
  smem_hist_flush(h, hist);
}

// One block: digit of rank st->rank in the merged histogram of `round`.  Warp w owns the
// contiguous bins [w * 2048, (w + 1) * 2048): coalesced loads, warp sums, a scan of the 32
// warp totals, then the owning warp resolves the bin with ballots (no per-thread arrays).
__global__ void __launch_bounds__(NT) resolve_kernel(const int* __restrict__ hist, int round,
                                                     long long take_cap, State* st,
                                                     long long* counts) {
  __shared__ unsigned warp_tot[32];
  __shared__ unsigned long long s_rank;
  __shared__ int s_warp;
  if (round == 0) {
    if (threadIdx.x == 0) {
      const unsigned long long ne = (unsigned long long)(unsigned)hist[NBINS];
      const unsigned long long take = ne < (unsigned long long)take_cap ? ne : (unsigned long long)take_cap;
      st->n_elig = ne;
      st->take = take;
      st->prefix = 0;
      st->pmask = 0;
      st->rank = take ? take - 1 : 0;
      st->status = take ? 0 : 1;
      st->T = 0;
      st->need_ties = 0;
      st->local_ties = 0;
      if (counts) {
        counts[0] = (long long)ne;
        counts[1] = (long long)take;
      }
    }
    __syncthreads();
  }
  if (st->status) return;
  constexpr int PERW = NBINS / (NT / 32);  // 2048 bins per warp
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int* h = hist + warp * PERW;
  unsigned sum = 0;
#pragma unroll 8
  for (int i = lane; i < PERW; i += 32) sum += (unsigned)h[i];
  sum = __reduce_add_sync(0xffffffffu, sum);
  if (lane == 0) warp_tot[warp] = sum;
  __syncthreads();
  const unsigned long long rank = st->rank;
  if (warp == 0) {
    unsigned x = warp_tot[lane], inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    const unsigned long long ex = inc - x;
    const bool mine = x && rank >= ex && rank < ex + x;
    const unsigned b = __ballot_sync(0xffffffffu, mine);
    const int w = __ffs(b) - 1;
    if (lane == w) {
      s_warp = w;
      s_rank = rank - ex;
    }
  }
  __syncthreads();
  if (warp != s_warp) return;
  // the owning warp walks its 2048 bins 32 at a time
  unsigned long long r = s_rank;
  const int* hw = hist + warp * PERW;
  for (int base = 0; base < PERW; base += 32) {
    const unsigned c = (unsigned)hw[base + lane];
    unsigned inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    const unsigned tot = __shfl_sync(0xffffffffu, inc, 31);
    if (r < tot) {
      const unsigned long long ex = inc - c;
      const bool mine = c && r >= ex && r < ex + c;
      const unsigned b = __ballot_sync(0xffffffffu, mine);
      const int l = __ffs(b) - 1;
      if (lane == l) {
        const int digit = warp * PERW + base + l;
        const int sh = round_shift(round);
        st->prefix |= (unsigned long long)digit << sh;
        st->pmask |= 0xffffull << sh;
        st->rank = r - ex;
        if (round == ROUNDS - 1) {
          st->T = st->prefix;
          st->need_ties = r - ex + 1;
        }
      }
      return;
    }
    r -= tot;
  }
}

// Per-block counts of key == T; the local total goes to *local_ties (all-gather send buffer).
__global__ void __launch_bounds__(NT) ties_kernel(const unsigned long long* __restrict__ keys,
                                                  long long n, State* st, unsigned* blk,
                                                  long long* local_ties) {
  __shared__ unsigned s_cnt;
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  const int status = st->status;
  const unsigned long long T = st->T;
  long long lo, hi;
  block_range(n, lo, hi);
  unsigned c = 0;
  if (!status)
    for (long long i0 = lo + threadIdx.x; i0 < hi; i0 += U * NT) {
      unsigned long long kv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) kv[u] = i0 + u * NT < hi ? keys[i0 + u * NT] : ~T;
#pragma unroll
      for (int u = 0; u < U; ++u) c += (kv[u] == T);
    }
  c = __reduce_add_sync(0xffffffffu, c);
  if (lane_id() == 0 && c) atomicAdd(&s_cnt, c);
  __syncthreads();
  if (threadIdx.x == 0) {
    blk[blockIdx.x] = s_cnt;
    if (s_cnt) atomicAdd((unsigned long long*)local_ties, (unsigned long long)s_cnt);
  }
}

__global__ void __launch_bounds__(NT) finalize_kernel(const unsigned long long* __restrict__ keys,
                                                      long long n, const State* st,
                                                      const unsigned* blk,
                                                      const long long* all_ties, int rank,
                                                      uint8_t* mask) {
  __shared__ unsigned warp_sums[32];
  __shared__ unsigned long long s_before;
  long long lo, hi;
  block_range(n, lo, hi);
  if (st->status) {
    for (long long i = lo + threadIdx.x; i < hi; i += NT) mask[i] = 0;
    return;
  }
  const unsigned long long T = st->T, need = st->need_ties;
  unsigned long long b = 0;
  for (int r = threadIdx.x; r < rank; r += NT) b += (unsigned long long)all_ties[r];
  for (unsigned k = threadIdx.x; k < blockIdx.x; k += NT) b += blk[k];
  // block reduce (64-bit)
  for (int o = 16; o; o >>= 1) b += __shfl_down_sync(0xffffffffu, b, o);
  if (threadIdx.x == 0) s_before = 0;
  __syncthreads();
  if (lane_id() == 0 && b) atomicAdd(&s_before, b);
  __syncthreads();
  unsigned long long run = s_before;
  // U-element steps; the tie scan (in index order) only runs for steps that hold a tie
  for (long long c0 = lo; c0 < hi; c0 += U * NT) {
    unsigned long long kv[U];
    int any = 0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long i = c0 + u * NT + threadIdx.x;
      kv[u] = i < hi ? keys[i] : kIneligible;
      any |= kv[u] == T;
    }
    if (!__syncthreads_or(any)) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long long i = c0 + u * NT + threadIdx.x;
        if (i < hi) mask[i] = kv[u] < T;
      }
      continue;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long i = c0 + u * NT + threadIdx.x;
      const unsigned is_tie = kv[u] == T ? 1u : 0u;
      unsigned tot;
      const unsigned ex = block_exclusive_scan(is_tie, warp_sums, &tot);
      if (i < hi) mask[i] = (kv[u] < T) || (is_tie && run + ex < need);
      run += tot;
    }
  }
}

inline int set_smem() {
  static int done = 0;
  if (!done) {
    if (cudaFuncSetAttribute(keys_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             SMEM_BYTES) != cudaSuccess ||
        cudaFuncSetAttribute(hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             SMEM_BYTES) != cudaSuccess)
      return 0;
    done = 1;
  }
  return 1;
}

}  // namespace shard
}  // namespace igs

using namespace igs;

extern "C" {

int igs_select_shard_workspace_bytes(int64_t n, size_t* bytes) {
  if (!bytes || n < 0) return IGS_ERR_ARGUMENT;
  *bytes = shard::layout(n).total;
  return IGS_OK;
}

int igs_select_shard_keys(const double* grad_sum, int64_t accum_count, const double* edge_score,
                          int64_t n, double grad_threshold, int warmup, int policy, int32_t* hist,
                          void* workspace, size_t workspace_bytes, void* stream) {
  if (n < 0 || accum_count < 0 || !hist || policy < 0 || policy > 2) return IGS_ERR_ARGUMENT;
  if (n >= (1ll << 31)) return IGS_ERR_UNSUPPORTED;
  if (n > 0 && (!grad_sum || !edge_score)) return IGS_ERR_ARGUMENT;
  shard::Layout L = shard::layout(n);
  if (!workspace || workspace_bytes < L.total) return IGS_ERR_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  char* w = (char*)workspace;
  IGS_CUDA_TRY(cudaMemsetAsync(hist, 0, sizeof(int32_t) * IGS_SHARD_HIST_LEN, st));
  IGS_CUDA_TRY(cudaMemsetAsync(w + L.state, 0, sizeof(shard::State), st));
  if (n == 0) return IGS_OK;
  if (!shard::set_smem()) return IGS_ERR_CUDA;
  shard::KeyParams P{grad_sum, accum_count, edge_score, n, grad_threshold, warmup, policy,
                     (unsigned long long*)(w + L.keys), hist};
  shard::keys_kernel<<<shard::grid_for(n), shard::NT, shard::SMEM_BYTES, st>>>(P);
  IGS_LAUNCH_CHECK();
  return IGS_OK;
}

int igs_select_shard_resolve(const int32_t* global_hist, int round, int64_t take_cap,
                             void* workspace, size_t workspace_bytes, int64_t* counts,
                             void* stream) {
  if (!global_hist || round < 0 || round >= shard::ROUNDS || take_cap < 0) return IGS_ERR_ARGUMENT;
  if (!workspace || workspace_bytes < 256) return IGS_ERR_WORKSPACE;
  shard::resolve_kernel<<<1, shard::NT, 0, (cudaStream_t)stream>>>(
      global_hist, round, take_cap, (shard::State*)workspace, (long long*)counts);
  IGS_LAUNCH_CHECK();
  return IGS_OK;
}

int igs_select_shard_hist(int64_t n, int round, int32_t* hist, void* workspace,
                          size_t workspace_bytes, void* stream) {
  if (n < 0 || !hist || round < 1 || round >= shard::ROUNDS) return IGS_ERR_ARGUMENT;
  shard::Layout L = shard::layout(n);
  if (!workspace || workspace_bytes < L.total) return IGS_ERR_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  IGS_CUDA_TRY(cudaMemsetAsync(hist, 0, sizeof(int32_t) * IGS_SHARD_HIST_LEN, st));
  if (n == 0) return IGS_OK;
  if (!shard::set_smem()) return IGS_ERR_CUDA;
  char* w = (char*)workspace;
  shard::hist_kernel<<<shard::grid_for(n), shard::NT, shard::SMEM_BYTES, st>>>(
      (const unsigned long long*)(w + L.keys), n, round, (const shard::State*)(w + L.state), hist);
  IGS_LAUNCH_CHECK();
  return IGS_OK;
}

int igs_select_shard_ties(int64_t n, int64_t* local_ties, void* workspace, size_t workspace_bytes,
                          void* stream) {
  if (n < 0 || !local_ties) return IGS_ERR_ARGUMENT;
  shard::Layout L = shard::layout(n);
  if (!workspace || workspace_bytes < L.total) return IGS_ERR_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  IGS_CUDA_TRY(cudaMemsetAsync(local_ties, 0, sizeof(int64_t), st));
  if (n == 0) return IGS_OK;
  char* w = (char*)workspace;
  shard::ties_kernel<<<shard::grid_for(n), shard::NT, 0, st>>>(
      (const unsigned long long*)(w + L.keys), n, (shard::State*)(w + L.state),
      (unsigned*)(w + L.blk), (long long*)local_ties);
  IGS_LAUNCH_CHECK();
  return IGS_OK;
}

int igs_select_shard_finalize(int64_t n, const int64_t* all_ties, int rank, uint8_t* mask,
                              void* workspace, size_t workspace_bytes, void* stream) {
  if (n < 0 || rank < 0 || (rank > 0 && !all_ties)) return IGS_ERR_ARGUMENT;
  if (n == 0) return IGS_OK;
  if (!mask) return IGS_ERR_ARGUMENT;
  shard::Layout L = shard::layout(n);
  if (!workspace || workspace_bytes < L.total) return IGS_ERR_WORKSPACE;
  char* w = (char*)workspace;
  shard::finalize_kernel<<<shard::grid_for(n), shard::NT, 0, (cudaStream_t)stream>>>(
      (const unsigned long long*)(w + L.keys), n, (const shard::State*)(w + L.state),
      (const unsigned*)(w + L.blk), (const long long*)all_ties, rank, mask);
  IGS_LAUNCH_CHECK();
  return IGS_OK;
}

}  // extern "C"
