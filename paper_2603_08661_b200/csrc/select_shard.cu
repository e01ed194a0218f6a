// Sharded densify step: the per-rank kernels of the multi-GPU protocol of SURVEY.md 8(e),
// two collective rounds per densify event and no host round trip until the event is read.
//
// Every rank holds a shard of the cloud and, per row, the row's index in the reference's
// global array (gidx): contiguous ranges before the first split, then children appended in
// the reference's order (all parents, then all children in parent order).  The selection is
// bit-identical to np.argsort(-score, kind="stable")[:take] over the global array
// (/root/reference/pkg/src/splitkit/densify_controller.py:80-106): order by (key, gidx).
//
//   keys_kernel      key = order-preserving 64-bit image of the score (ascending key ==
//                    descending score, -0 == +0, NaN last; ineligible = ~0) and a 65536-bin
//                    histogram of a monotone 16-bit digit of the key (1024 bins per binade
//                    over scores in [2^-62, 4)), plus the eligible count
//                                                              -> all-reduce #1 (sum, 256 KB)
//   resolve_kernel   (1 block) take = min(#eligible, take_cap); the digit B holding rank
//                    take-1 and need = take - #(digit < B); clears this rank's record
//   compact_kernel   #(digit < B) and the OR of their LAS flags; the boundary-bucket entries
//                    (key, gidx | flags << 56) into a fixed-capacity record
//                                                              -> all-gather #2 (records)
//   final_kernel     (1 block) over every rank's record: the need-th smallest (key, gidx) of
//                    the boundary bucket by radix select -> threshold (T, G); every rank's
//                    split count k_r and the batch flags; this rank's plan (LAS guard
//                    {k_r or 0, flags}, child base = N + sum_{r' < r} k_r', status)
//   mask_kernel      mask = digit < B, or digit == B and (key, gidx) <= (T, G)
//   child_index_kernel  gidx of this rank's appended children
// A boundary bucket larger than the record capacity sets status OVERFLOW (nothing is split);
// the host re-runs compact / gather / final with a record sized from the gathered counts.
#include <cuda_runtime.h>
#include <stdint.h>

#include "igs_common.cuh"

namespace igs {
namespace shard {

constexpr int NT = 1024;
constexpr int NBINS = 1 << 16;
constexpr int U = 4;                          // elements per thread per streaming step
constexpr unsigned long long kIneligible = ~0ull;
constexpr long long MAX_PER_BLOCK = 65535;   // 16-bit packed shared-memory counters
constexpr int SMEM_BYTES = NBINS * 2;        // two 16-bit bins per 32-bit word
constexpr unsigned long long T_LO = 984064ull;      // (1023 - 62) << 10: 2^-62
constexpr unsigned long long T_HI = T_LO + 65532ull;
constexpr int DIGIT_NONPOS = 65534, DIGIT_NAN = 65535;
constexpr int RBITS = 11, RBINS = 1 << RBITS;  // final_kernel radix digits

struct State {
  unsigned long long take, n_elig, need, B;
  int status;  // 0 ok, 1 nothing to select
  int pad[7];
};
static_assert(sizeof(State) <= 256, "state fits its 256-byte slot");

struct Layout {
  size_t state, keys, klo, bidx, total;
};

inline Layout layout(long long n) {
  Layout L;
  L.state = 0;
  L.keys = 256;  // keys as two u32 arrays: high words [keys, +4n), low words from klo
  L.klo = align_up(L.keys + sizeof(unsigned) * (size_t)n, 256);
  L.bidx = align_up(L.klo + sizeof(unsigned) * (size_t)n, 256);  // u32 per row
  L.total = align_up(L.bidx + sizeof(unsigned) * (size_t)n, 256);
  return L;
}

inline int grid_for(long long n) {
  long long g = (n + MAX_PER_BLOCK - 1) / MAX_PER_BLOCK;
  long long want = (n + 4 * NT - 1) / (4 * NT);
  long long sms = sm_count() > 0 ? sm_count() : 148;
  if (want > sms) want = sms;
  if (g < want) g = want;
  if (g < 1) g = 1;
  return (int)g;
}

__device__ __forceinline__ unsigned long long score_key(double s) {
  if (s != s) return 0xFFF8000000000000ull;
  if (s == 0.0) s = 0.0;
  unsigned long long b = (unsigned long long)__double_as_longlong(s);
  unsigned long long u = (b >> 63) ? ~b : (b | 0x8000000000000000ull);
  return ~u;
}

// Monotone non-decreasing 16-bit digit of an eligible key (ascending digit == descending
// score): positive scores 1024 bins per binade over [2^-62, 4), clamped at both ends; every
// non-positive score one bin; NaN last.
__device__ __forceinline__ int key_digit(unsigned long long key) {
  if (key == 0xFFF8000000000000ull) return DIGIT_NAN;
  const unsigned long long u = ~key;
  if (!(u >> 63)) return DIGIT_NONPOS;                   // a negative score
  const unsigned long long b = u & 0x7FFFFFFFFFFFFFFFull;  // |score| bits, score >= +0
  if (b == 0) return DIGIT_NONPOS;
  unsigned long long t = b >> 42;
  t = t < T_LO ? T_LO : (t > T_HI ? T_HI : t);
  return 1 + (int)(T_HI - t);
}

// Keys live as two u32 arrays (high, low words): the passes over every row read only the high
// words; the digit needs the low word only for the NaN key and the |score| < 2^-1010 corner.
__device__ __forceinline__ unsigned long long key_at(const unsigned* __restrict__ khi,
                                                     const unsigned* __restrict__ klo, long long i) {
  return ((unsigned long long)khi[i] << 32) | klo[i];
}
// key_digit from the high word; NBINS for an ineligible row (high word 0xffffffff, which no
// eligible key has); -1 when the low word is needed.
__device__ __forceinline__ int digit_hi(unsigned h) {
  if (h == 0xFFFFFFFFu) return NBINS;
  if (h == 0xFFF80000u) return -1;                 // the NaN key, or a key sharing its high word
  const unsigned uh = ~h;
  if (!(uh >> 31)) return DIGIT_NONPOS;            // a negative score
  const unsigned bh = uh & 0x7FFFFFFFu;
  if (bh == 0) return -1;                          // |score| < 2^-1022 or zero: b == 0 needs lo
  unsigned long long t = (unsigned long long)bh >> 10;  // b >> 42
  t = t < T_LO ? T_LO : (t > T_HI ? T_HI : t);
  return 1 + (int)(T_HI - t);
}

__device__ __forceinline__ void block_range(long long n, long long& lo, long long& hi) {
  const long long per = (n + gridDim.x - 1) / gridDim.x;
  lo = min((long long)blockIdx.x * per, n);
  hi = min(lo + per, n);
}

struct KeyParams {
  const double* grad_sum;
  long long accum;
  const double* edge;
  long long n;
  double thr;
  int warmup, policy;
  unsigned* khi;
  unsigned* klo;
  int* hist;  // NBINS + 1 (last: eligible count)
};

__global__ void __launch_bounds__(NT) keys_kernel(KeyParams P) {
  extern __shared__ unsigned h[];
  for (int i = threadIdx.x; i < NBINS / 2; i += NT) h[i] = 0;
  __syncthreads();
  long long lo, hi;
  block_range(P.n, lo, hi);
  unsigned elig = 0;
  const bool need_edge = P.warmup || P.policy != IGS_POLICY_GRAD;
  for (long long i0 = lo + threadIdx.x; i0 < hi; i0 += U * NT) {
    double gs[U], ed[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {  // every load before the arithmetic
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
      P.khi[i] = (unsigned)(k >> 32);
      P.klo[i] = (unsigned)k;
      if (e) {
        ++elig;
        const unsigned d = (unsigned)key_digit(k);
        atomicAdd(&h[d >> 1], 1u << ((d & 1u) << 4));
      }
    }
  }
  elig = __reduce_add_sync(0xffffffffu, elig);
  if (lane_id() == 0 && elig) atomicAdd(&P.hist[NBINS], (int)elig);
  __syncthreads();
  for (int i = threadIdx.x; i < NBINS / 2; i += NT) {
    const unsigned v = h[i];
    if (v & 0xffffu) atomicAdd(&P.hist[2 * i], (int)(v & 0xffffu));
    if (v >> 16) atomicAdd(&P.hist[2 * i + 1], (int)(v >> 16));
  }
}

// Record of one rank (int64 words): header, then `cap` entries of two words.
enum Rec { R_LT = 0, R_BCNT = 1, R_LTFLAGS = 2, R_HDR = 4 };

// One block: take, B and need from the merged histogram; clears this rank's record header.
// Warp w owns the 2048 consecutive bins [2048 w, 2048 w + 2048), read with coalesced 16-byte
// loads (lane l: bins 4 (l + 32 k) .. + 3 of the range, k < 16).  A scan of the warp totals
// names the warp holding rank take-1; it walks its 16 chunks of 128 bins, then the lanes of
// the chunk, then the lane's 4 bins.
__global__ void __launch_bounds__(NT) resolve_kernel(const int* __restrict__ hist,
                                                     long long take_cap, State* st,
                                                     long long* record) {
  static_assert(NT == 1024 && NBINS == 32 * 2048, "32 warps x 2048 bins");
  __shared__ unsigned warp_tot[32];
  __shared__ unsigned long long s_need;
  __shared__ int s_B;
  const unsigned long long ne = (unsigned long long)(unsigned)hist[NBINS];
  const unsigned long long take = ne < (unsigned long long)take_cap ? ne : (unsigned long long)take_cap;
  const int lane = lane_id(), warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    record[R_LT] = 0;
    record[R_BCNT] = 0;
    record[R_LTFLAGS] = 0;
    record[3] = 0;
    s_B = NBINS;
    s_need = 0;
  }
  const int4* h4 = reinterpret_cast<const int4*>(hist) + warp * 512;
  unsigned cs[16];  // this lane's 4-bin sum of chunk k
  unsigned mine = 0;
#pragma unroll
  for (int half = 0; half < 2; ++half) {  // 8 loads in flight at a time (64 registers)
    int4 hv[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) hv[k] = __ldcg(h4 + lane + 32 * (8 * half + k));
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      cs[8 * half + k] = (unsigned)hv[k].x + (unsigned)hv[k].y + (unsigned)hv[k].z + (unsigned)hv[k].w;
      mine += cs[8 * half + k];
    }
  }
  const unsigned wt = __reduce_add_sync(0xffffffffu, mine);
  if (lane == 0) warp_tot[warp] = wt;
  __syncthreads();
  if (take > 0) {
    const unsigned long long r = take - 1;
    unsigned long long before = 0;
    for (int w = 0; w < warp; ++w) before += warp_tot[w];
    if (r >= before && r < before + wt) {  // warp-uniform: this warp holds rank r
      unsigned long long cum = before;
      bool done = false;
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const unsigned ck = __reduce_add_sync(0xffffffffu, cs[k]);
        if (!done && r < cum + ck) {  // chunk k (warp-uniform): lanes in order, 4 bins each
          done = true;
          unsigned x = cs[k];
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
          }
          const unsigned long long lo = cum + (x - cs[k]);
          if (r >= lo && r < lo + cs[k]) {
            const int4 hk = __ldcg(h4 + lane + 32 * k);  // the lane's 4 bins again
            const unsigned b0 = (unsigned)hk.x, b1 = (unsigned)hk.y, b2 = (unsigned)hk.z;
            unsigned long long at = lo;
            int j = 0;
            if (r >= at + b0) {
              at += b0;
              j = 1;
              if (r >= at + b1) {
                at += b1;
                j = 2;
                if (r >= at + b2) {
                  at += b2;
                  j = 3;
                }
              }
            }
            s_B = warp * 2048 + 4 * (lane + 32 * k) + j;
            s_need = take - at;
          }
        }
        cum += ck;
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    st->take = take;
    st->n_elig = ne;
    st->B = (unsigned long long)s_B;
    st->need = s_need;
    st->status = take ? 0 : 1;
  }
}

// numpy float32 LAS pre-pass flags of one parent (las.cu prepare_tile), from its loaded
// quaternion (3-D) and opacity logit.
__device__ __forceinline__ unsigned las_flags_of(bool d3, float4 q, float o, float beta) {
  unsigned f = 0;
  if (d3) {
    float s = q.x * q.x;
    s = s + q.y * q.y;
    s = s + q.z * q.z;
    s = s + q.w * q.w;
    const float nrm = sqrtf(s);
    if (!isfinite(nrm) || nrm == 0.0f) f |= IGS_LAS_BAD_QUAT;
    else if (fabsf(nrm - 1.0f) > 1e-4f) f |= IGS_LAS_RENORM;
  }
  if (las_opacity_bad(o, beta)) f |= IGS_LAS_BAD_OPACITY;
  return f;
}

constexpr int NTC = 256;  // compact_kernel block
// compact_kernel: 16-byte high-word loads per thread per trip (even: the flag gathers run in
// halves of 8 rows) and resident blocks per SM (64 registers): UC 2 at 4 blocks per SM
// measured 31 us at 6M rows against 37 us for UC 4 at 3 blocks and 45-49 us otherwise
constexpr int UC = 2;
constexpr int CMINB = 4;
static_assert(UC % 2 == 0, "compact trips are processed in halves of 8 rows");

__global__ void __launch_bounds__(NTC, CMINB) compact_kernel(const unsigned* __restrict__ khi,
                                                     const unsigned* __restrict__ klo,
                                                     const long long* __restrict__ gidx,
                                                     const float* rot, const float* opac,
                                                     float beta, long long n, const State* st,
                                                     long long cap, long long* record,
                                                     uint8_t* mask, unsigned* bidx) {
  __shared__ unsigned s_lt, s_flags;
  if (threadIdx.x == 0) {
    s_lt = 0;
    s_flags = 0;
  }
  __syncthreads();
  if (st->status) return;
  const int B = (int)st->B;
  // this block's rows, in whole trips of CROWS (16-byte aligned high-word loads)
  constexpr long long CROWS = (long long)NTC * 4 * UC;
  const long long per = ((n + gridDim.x - 1) / gridDim.x + CROWS - 1) / CROWS * CROWS;
  const long long lo = min((long long)blockIdx.x * per, n), hi = min(lo + per, n);
  unsigned lt = 0, fl = 0;
  const unsigned lanelt = lanemask_lt();
  // every lane runs the same trips, so the warp-aggregated appends see every lane
  for (long long t0 = lo; t0 < hi; t0 += CROWS) {
    // rows t0 + 4 (threadIdx.x + NTC u) + j: one 16-byte load of high words per u
    int dv[UC][4];
#pragma unroll
    for (int u = 0; u < UC; ++u) {
      const long long r0 = t0 + 4 * ((long long)threadIdx.x + (long long)NTC * u);
      uint4 hv = make_uint4(~0u, ~0u, ~0u, ~0u);
      if (r0 + 4 <= hi) {
        hv = __ldcs(reinterpret_cast<const uint4*>(khi + r0));
      } else {
        if (r0 < hi) hv.x = khi[r0];
        if (r0 + 1 < hi) hv.y = khi[r0 + 1];
        if (r0 + 2 < hi) hv.z = khi[r0 + 2];
      }
      dv[u][0] = digit_hi(hv.x);
      dv[u][1] = digit_hi(hv.y);
      dv[u][2] = digit_hi(hv.z);
      dv[u][3] = digit_hi(hv.w);
    }
#pragma unroll
    for (int u = 0; u < UC; ++u)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (dv[u][j] < 0) {  // rare: the digit needs the low word
          const long long i = t0 + 4 * ((long long)threadIdx.x + (long long)NTC * u) + j;
          dv[u][j] = key_digit(key_at(khi, klo, i));
        }
    // the mask of the rows below the boundary bucket (the boundary rows the plan takes are set
    // by boundary_mask_kernel once the threshold is known): 4 rows per 4-byte store
#pragma unroll
    for (int u = 0; u < UC; ++u) {
      const long long r0 = t0 + 4 * ((long long)threadIdx.x + (long long)NTC * u);
      const unsigned m = (dv[u][0] < B ? 1u : 0u) | (dv[u][1] < B ? 1u << 8 : 0u) |
                         (dv[u][2] < B ? 1u << 16 : 0u) | (dv[u][3] < B ? 1u << 24 : 0u);
      if (r0 + 4 <= hi) {
        *reinterpret_cast<unsigned*>(mask + r0) = m;
      } else {
        for (int j = 0; j < 4; ++j)
          if (r0 + j < hi) mask[r0 + j] = (uint8_t)((m >> (8 * j)) & 1u);
      }
    }
    // the selected and boundary rows' LAS flags (every load of a half-trip in flight first),
    // the count below the boundary bucket and the boundary-bucket records
#pragma unroll
    for (int h2 = 0; h2 < UC / 2; ++h2) {
      float4 qv[8];
      float ov[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int u = 2 * h2 + (e >> 2), j = e & 3;
        const long long i = t0 + 4 * ((long long)threadIdx.x + (long long)NTC * u) + j;
        qv[e] = make_float4(1.f, 0.f, 0.f, 0.f);
        ov[e] = 0.f;
        if (opac && dv[u][j] <= B) {
          if (rot) qv[e] = __ldg(reinterpret_cast<const float4*>(rot) + i);
          ov[e] = __ldg(opac + i);
        }
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int u = 2 * h2 + (e >> 2), j = e & 3;
        const int d = dv[u][j];
        const unsigned fu = (opac && d <= B) ? las_flags_of(rot != nullptr, qv[e], ov[e], beta) : 0u;
        if (d < B) {
          ++lt;
          fl |= fu;
        }
        const bool bnd = d == B;
        const unsigned bal = __ballot_sync(0xffffffffu, bnd);
        if (!bal) continue;
        unsigned long long base = 0;
        if ((threadIdx.x & 31) == 0)  // one append per warp
          base = atomicAdd((unsigned long long*)&record[R_BCNT], (unsigned long long)__popc(bal));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (bnd) {
          const unsigned long long slot = base + __popc(bal & lanelt);
          if ((long long)slot < cap) {
            const long long i = t0 + 4 * ((long long)threadIdx.x + (long long)NTC * u) + j;
            bidx[slot] = (unsigned)i;
            record[R_HDR + 2 * slot] = (long long)key_at(khi, klo, i);
            record[R_HDR + 2 * slot + 1] =
                (long long)((unsigned long long)gidx[i] | ((unsigned long long)fu << 56));
          }
        }
      }
    }
  }
  lt = __reduce_add_sync(0xffffffffu, lt);
  fl = __reduce_or_sync(0xffffffffu, fl);
  if (lane_id() == 0) {
    if (lt) atomicAdd(&s_lt, lt);
    if (fl) atomicOr(&s_flags, fl);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (s_lt) atomicAdd((unsigned long long*)&record[R_LT], (unsigned long long)s_lt);
    if (s_flags) atomicOr((unsigned long long*)&record[R_LTFLAGS], (unsigned long long)s_flags);
  }
}

// The plan this rank acts on (int64 words; also the host's one read per event).
enum Plan {
  P_NSPLIT = 0,   // LAS guard: this rank's split count when the split may go ahead, else 0
  P_FLAGS = 1,    // LAS guard: the batch flags (OR over every rank's selected parents)
  P_STATUS = 2,   // 0 ok, 1 nothing selected, 2 boundary bucket overflowed the records
  P_TAKE = 3,     // global split count
  P_ELIG = 4,     // global eligible count
  P_CHILD = 5,    // global index of this rank's first child
  P_KMINE = 6,    // this rank's split count
  P_MAXB = 7,     // largest boundary-bucket count over the ranks (overflow re-run size)
  P_T = 8,        // threshold key
  P_G = 9,        // threshold global index (key == T and gidx <= G is in)
  P_B = 10,       // boundary digit
  P_NEED = 11,    // boundary entries to take
  P_WORDS = 16
};
constexpr int MAX_WORLD = 64;
constexpr int EMAX = 8;             // boundary entries per thread in final_kernel
constexpr long long MAX_ENTRIES = (long long)EMAX * NT;  // world * record_cap

// Radix select (RBITS-bit digits, block-wide) of the rank-`rank` smallest of the values v[k]
// (ok[k]) each thread holds (E per thread); bits above `top` are equal in every value.
template <int E>
__device__ unsigned long long block_select64(const unsigned long long (&v)[E], const bool (&ok)[E],
                                            unsigned long long rank, int top, unsigned* h,
                                            unsigned* warp_sums, unsigned long long* s_val,
                                            int* s_bin) {
  unsigned long long prefix = 0, pmask = top >= 63 ? 0ull : (~0ull << (top + 1));
  {  // the common high bits: any valid value
    __shared__ unsigned long long s_any;
    if (threadIdx.x == 0) s_any = 0;
    __syncthreads();
    unsigned long long any = 0;
    bool have = false;
#pragma unroll
    for (int k = 0; k < E; ++k)
      if (ok[k] && !have) {
        any = v[k];
        have = true;
      }
    const unsigned hb = __ballot_sync(0xffffffffu, have);
    if (hb && lane_id() == __ffs(hb) - 1) s_any = any;  // benign race: every writer's value is valid
    __syncthreads();
    prefix = s_any & pmask;
    __syncthreads();
  }
  for (; top >= 0; top -= RBITS) {
    const int width = top + 1 < RBITS ? top + 1 : RBITS;
    const int shift = top + 1 - width;
    const unsigned dmask = (1u << width) - 1;
    for (int i = threadIdx.x; i < RBINS; i += NT) h[i] = 0;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < E; ++k)
      if (ok[k] && (v[k] & pmask) == prefix) atomicAdd(&h[(v[k] >> shift) & dmask], 1u);
    __syncthreads();
    // RBINS / NT bins per thread, block scan, the owner of `rank` publishes the digit
    constexpr int PER = RBINS / NT;
    unsigned loc[PER], sum = 0;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      loc[k] = h[threadIdx.x * PER + k];
      sum += loc[k];
    }
    unsigned tot;
    unsigned long long cum = block_exclusive_scan(sum, warp_sums, &tot);
    __shared__ unsigned s_cnt;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      if (loc[k] && rank >= cum && rank < cum + loc[k]) {
        *s_bin = threadIdx.x * PER + k;
        *s_val = rank - cum;
        s_cnt = loc[k];
      }
      cum += loc[k];
    }
    __syncthreads();
    prefix |= (unsigned long long)(*s_bin) << shift;
    pmask |= (unsigned long long)dmask << shift;
    rank = *s_val;
    const unsigned cnt = s_cnt;
    __syncthreads();
    if (cnt == 1 && top >= RBITS) {  // one value left with this prefix: it is the answer (the
                                     // boundary keys of a bucket usually separate in 1-2 rounds)
      __shared__ unsigned long long s_res;
#pragma unroll
      for (int k = 0; k < E; ++k)
        if (ok[k] && (v[k] & pmask) == prefix) s_res = v[k];
      __syncthreads();
      return s_res;
    }
  }
  return prefix;
}

__global__ void __launch_bounds__(NT) final_kernel(const long long* __restrict__ records,
                                                   int world, int rank, long long cap,
                                                   long long n_global, const State* st,
                                                   long long* plan) {
  __shared__ unsigned h[RBINS];
  __shared__ unsigned warp_sums[32];
  __shared__ unsigned long long s_val;
  __shared__ int s_bin;
  __shared__ unsigned long long s_k[MAX_WORLD];
  __shared__ unsigned s_flags;
  const long long stride = R_HDR + 2 * cap;
  const unsigned long long take = st->take, need = st->need;
  long long maxb = 0;
  int overflow = 0;
  for (int r = 0; r < world; ++r) {
    const long long b = records[r * stride + R_BCNT];
    maxb = b > maxb ? b : maxb;
    overflow |= b > cap;
  }
  if (threadIdx.x == 0) {
    for (int k = 0; k < P_WORDS; ++k) plan[k] = 0;
    plan[P_TAKE] = (long long)take;
    plan[P_ELIG] = (long long)st->n_elig;
    plan[P_MAXB] = maxb;
    plan[P_B] = (long long)st->B;
    plan[P_NEED] = (long long)need;
  }
  if (st->status || overflow || world * cap > MAX_ENTRIES) {
    if (threadIdx.x == 0) plan[P_STATUS] = st->status ? 1 : 2;
    return;
  }
  const long long m = world * cap;  // entry e: rank e / cap, slot e % cap
  // every entry in registers: thread t holds entries t + NT k
  unsigned long long kv[EMAX], gv[EMAX];
  bool ok[EMAX];
  unsigned long long kmin = ~0ull, kmax = 0;
#pragma unroll
  for (int k = 0; k < EMAX; ++k) {
    const long long e = threadIdx.x + (long long)NT * k;
    const long long r = (long long)((unsigned)e / (unsigned)cap), s = e - r * cap;  // m < 2^31
    ok[k] = e < m && s < records[r * stride + R_BCNT];
    kv[k] = ok[k] ? (unsigned long long)records[r * stride + R_HDR + 2 * s] : 0ull;
    gv[k] = ok[k] ? (unsigned long long)records[r * stride + R_HDR + 2 * s + 1] : 0ull;
    if (ok[k]) {
      kmin = kv[k] < kmin ? kv[k] : kmin;
      kmax = kv[k] > kmax ? kv[k] : kmax;
    }
  }
  // the boundary keys share their high bits (one digit bucket): start below them
  __shared__ unsigned long long s_min, s_max;
  if (threadIdx.x == 0) {
    s_min = ~0ull;
    s_max = 0;
  }
  __syncthreads();
#pragma unroll
  for (int o = 16; o; o >>= 1) {  // one shared atomic per warp
    const unsigned long long a = __shfl_down_sync(0xffffffffu, kmin, o);
    const unsigned long long b = __shfl_down_sync(0xffffffffu, kmax, o);
    kmin = a < kmin ? a : kmin;
    kmax = b > kmax ? b : kmax;
  }
  if (lane_id() == 0) {
    atomicMin(&s_min, kmin);
    atomicMax(&s_max, kmax);
  }
  __syncthreads();
  const unsigned long long diff = s_min ^ s_max;
  const int top = diff ? 63 - __clzll(diff) : 0;
  // threshold key T: the need-th smallest boundary key (rank need - 1)
  const unsigned long long T = block_select64<EMAX>(kv, ok, need - 1, top, h, warp_sums, &s_val,
                                                    &s_bin);
  unsigned long long below = 0, ties = 0;
#pragma unroll
  for (int k = 0; k < EMAX; ++k)
    if (ok[k]) {
      below += kv[k] < T;
      ties += kv[k] == T;
    }
  for (int o = 16; o; o >>= 1) {
    below += __shfl_down_sync(0xffffffffu, below, o);
    ties += __shfl_down_sync(0xffffffffu, ties, o);
  }
  __shared__ unsigned long long s_below, s_ties;
  if (threadIdx.x == 0) {
    s_below = 0;
    s_ties = 0;
  }
  __syncthreads();
  if (lane_id() == 0) {
    atomicAdd(&s_below, below);
    atomicAdd(&s_ties, ties);
  }
  __syncthreads();
  const unsigned long long need_ties = need - s_below;
  unsigned long long G = 0x00FFFFFFFFFFFFFFull;  // every tie in
  if (need_ties < s_ties) {
    unsigned long long gi[EMAX];
    bool tie[EMAX];
#pragma unroll
    for (int k = 0; k < EMAX; ++k) {
      tie[k] = ok[k] && kv[k] == T;
      gi[k] = gv[k] & 0x00FFFFFFFFFFFFFFull;
    }
    G = block_select64<EMAX>(gi, tie, need_ties - 1, 55, h, warp_sums, &s_val, &s_bin);
  }
  // every rank's split count and the batch flags
  for (int r = threadIdx.x; r < world; r += NT)
    s_k[r] = (unsigned long long)records[r * stride + R_LT];
  if (threadIdx.x == 0) {
    s_flags = 0;
    for (int r = 0; r < world; ++r) s_flags |= (unsigned)records[r * stride + R_LTFLAGS];
  }
  __syncthreads();
  unsigned fsel = 0;
#pragma unroll
  for (int k = 0; k < EMAX; ++k) {
    const unsigned long long g = gv[k] & 0x00FFFFFFFFFFFFFFull;
    const bool in = ok[k] && (kv[k] < T || (kv[k] == T && g <= G));
    if (in) fsel |= (unsigned)(gv[k] >> 56);
    // the warp's entries are consecutive: at most a few ranks, one atomic per (warp, rank)
    const unsigned e = threadIdx.x + (unsigned)NT * (unsigned)k;
    const unsigned r = e / (unsigned)cap;
    const unsigned sel = __ballot_sync(0xffffffffu, in);
    if (sel) {
      const unsigned grp = __match_any_sync(0xffffffffu, r);
      if (lane_id() == __ffs(grp) - 1 && (sel & grp)) atomicAdd(&s_k[r], (unsigned long long)__popc(sel & grp));
    }
  }
  fsel = __reduce_or_sync(0xffffffffu, fsel);
  if (lane_id() == 0 && fsel) atomicOr(&s_flags, fsel);
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long base = (unsigned long long)n_global;
    for (int r = 0; r < rank; ++r) base += s_k[r];
    const unsigned long long kmine = s_k[rank];
    plan[P_NSPLIT] = (long long)kmine;
    plan[P_FLAGS] = (long long)s_flags;
    plan[P_STATUS] = 0;
    plan[P_CHILD] = (long long)base;
    plan[P_KMINE] = (long long)kmine;
    plan[P_T] = (long long)T;
    plan[P_G] = (long long)G;
  }
}

// The mask once the plan is known: compact_kernel wrote every row's (digit < B); this sets the
// boundary rows the plan takes (this rank's boundary entries, their local rows in bidx), or
// clears the mask when nothing is selected / the records overflowed (the re-run rewrites it).
__global__ void __launch_bounds__(NT) boundary_mask_kernel(
    const unsigned* __restrict__ khi, const unsigned* __restrict__ klo,
    const long long* __restrict__ gidx, long long n,
    const long long* __restrict__ records, int rank, long long cap, const unsigned* bidx,
    const long long* plan, uint8_t* mask) {
  if (plan[P_STATUS] != 0) {
    for (long long i = blockIdx.x * (long long)NT + threadIdx.x; i < n;
         i += (long long)gridDim.x * NT)
      mask[i] = 0;
    return;
  }
  const unsigned long long T = (unsigned long long)plan[P_T];
  const unsigned long long G = (unsigned long long)plan[P_G];
  const long long stride = R_HDR + 2 * cap;
  long long nb = records[rank * stride + R_BCNT];
  nb = nb < cap ? nb : cap;
  for (long long s = blockIdx.x * (long long)NT + threadIdx.x; s < nb;
       s += (long long)gridDim.x * NT) {
    const long long i = bidx[s];
    const unsigned long long k = key_at(khi, klo, i);
    if (k < T || (k == T && (unsigned long long)gidx[i] <= G)) mask[i] = 1;
  }
}

__global__ void __launch_bounds__(NT) mask_kernel(const unsigned* __restrict__ khi,
                                                  const unsigned* __restrict__ klo,
                                                  const long long* __restrict__ gidx, long long n,
                                                  const long long* plan, uint8_t* mask) {
  const bool ok = plan[P_STATUS] == 0;
  const int B = (int)plan[P_B];
  const unsigned long long T = (unsigned long long)plan[P_T];
  const unsigned long long G = (unsigned long long)plan[P_G];
  for (long long i = blockIdx.x * (long long)NT + threadIdx.x; i < n;
       i += (long long)gridDim.x * NT) {
    const unsigned long long k = key_at(khi, klo, i);
    bool in = false;
    if (ok && k != kIneligible) {
      const int d = key_digit(k);
      in = d < B || (d == B && (k < T || (k == T && (unsigned long long)gidx[i] <= G)));
    }
    mask[i] = in;
  }
}

__global__ void child_index_kernel(long long* gidx, long long count, const long long* plan) {
  const long long k = plan[P_STATUS] == 0 ? plan[P_KMINE] : 0;
  const long long base = plan[P_CHILD];
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < k;
       j += (long long)gridDim.x * blockDim.x)
    gidx[count + j] = base + j;
}

inline int set_smem() {
  static int done = 0;
  if (!done) {
    if (cudaFuncSetAttribute(keys_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
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

int igs_shard_workspace_bytes(int64_t n, size_t* bytes) {
  if (!bytes || n < 0) return IGS_ERR_ARGUMENT;
  *bytes = shard::layout(n).total;
  return IGS_OK;
}

int igs_shard_keys(const double* grad_sum, int64_t accum_count, const double* edge_score,
                   int64_t n, double grad_threshold, int warmup, int policy, int32_t* hist,
                   void* workspace, size_t workspace_bytes, void* stream) {
  if (n < 0 || accum_count < 0 || !hist || policy < 0 || policy > 2) return IGS_ERR_ARGUMENT;
  if (n >= (1ll << 31)) return IGS_ERR_UNSUPPORTED;
  if (n > 0 && (!grad_sum || !edge_score)) return IGS_ERR_ARGUMENT;
  if ((uintptr_t)hist & 15) return IGS_ERR_ARGUMENT;
  shard::Layout L = shard::layout(n);
  if (!workspace || workspace_bytes < L.total) return IGS_ERR_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  IGS_CUDA_TRY(cudaMemsetAsync(hist, 0, sizeof(int32_t) * IGS_SHARD_HIST_LEN, st));
  if (n == 0) return IGS_OK;
  if (!shard::set_smem()) return IGS_ERR_CUDA;
  shard::KeyParams P{grad_sum, accum_count, edge_score, n, grad_threshold, warmup, policy,
                     (unsigned*)((char*)workspace + L.keys), (unsigned*)((char*)workspace + L.klo),
                     hist};
  shard::keys_kernel<<<shard::grid_for(n), shard::NT, shard::SMEM_BYTES, st>>>(P);
  IGS_LAUNCH_CHECK();
  return IGS_OK;
}

int igs_shard_boundary(const int32_t* global_hist, int64_t take_cap, const int64_t* gidx,
                       const float* rotations, const float* opacity_logits, float beta,
                       int64_t n, int64_t record_cap, int64_t* record, uint8_t* mask,
                       void* workspace, size_t workspace_bytes, void* stream) {
  if (!global_hist || !record || take_cap < 0 || n < 0 || record_cap < 1) return IGS_ERR_ARGUMENT;
  if (n > 0 && !mask) return IGS_ERR_ARGUMENT;
  if (((uintptr_t)global_hist & 15) || ((uintptr_t)rotations & 15)) return IGS_ERR_ARGUMENT;
  if (n > 0 && !gidx) return IGS_ERR_ARGUMENT;  // opacity_logits NULL: no LAS flags
  shard::Layout L = shard::layout(n);
  if (!workspace || workspace_bytes < L.total) return IGS_ERR_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  char* w = (char*)workspace;
  shard::State* S = (shard::State*)(w + L.state);
  shard::resolve_kernel<<<1, shard::NT, 0, st>>>(global_hist, take_cap, S, (long long*)record);
  IGS_LAUNCH_CHECK();
  if (n == 0) return IGS_OK;
  if (n > 0 && ((uintptr_t)mask & 3)) return IGS_ERR_ARGUMENT;  // 4-row mask stores
  long long cgrid = (n + 4LL * shard::NTC * shard::UC - 1) / (4LL * shard::NTC * shard::UC);
  const long long cmax = 8LL * (sm_count() > 0 ? sm_count() : 148);
  if (cgrid > cmax) cgrid = cmax;
  if (cgrid < 1) cgrid = 1;
  shard::compact_kernel<<<(unsigned)cgrid, shard::NTC, 0, st>>>(
      (const unsigned*)(w + L.keys), (const unsigned*)(w + L.klo), (const long long*)gidx,
      rotations, opacity_logits,
      beta, n, S, record_cap, (long long*)record, mask, (unsigned*)(w + L.bidx));
  IGS_LAUNCH_CHECK();
  return IGS_OK;
}

int igs_shard_finalize(const int64_t* records, int world, int rank, int64_t record_cap,
                       int64_t n_global, const int64_t* gidx, int64_t n, uint8_t* mask,
                       int64_t* plan, void* workspace, size_t workspace_bytes, void* stream) {
  if (!records || !plan || world < 1 || world > shard::MAX_WORLD || rank < 0 || rank >= world ||
      record_cap < 1 || n < 0 || n_global < 0)
    return IGS_ERR_ARGUMENT;
  if (n > 0 && (!gidx || !mask)) return IGS_ERR_ARGUMENT;
  shard::Layout L = shard::layout(n);
  if (!workspace || workspace_bytes < L.total) return IGS_ERR_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  char* w = (char*)workspace;
  shard::final_kernel<<<1, shard::NT, 0, st>>>((const long long*)records, world, rank,
                                               record_cap, n_global,
                                               (const shard::State*)(w + L.state),
                                               (long long*)plan);
  IGS_LAUNCH_CHECK();
  if (n == 0) return IGS_OK;
  long long grid = (n + shard::NT - 1) / shard::NT;
  const long long cap = 8LL * (sm_count() > 0 ? sm_count() : 148);
  if (grid > cap) grid = cap;
  shard::boundary_mask_kernel<<<(unsigned)grid, shard::NT, 0, st>>>(
      (const unsigned*)(w + L.keys), (const unsigned*)(w + L.klo), (const long long*)gidx, n,
      (const long long*)records, rank, record_cap, (const unsigned*)(w + L.bidx),
      (const long long*)plan, mask);
  IGS_LAUNCH_CHECK();
  return IGS_OK;
}

// The mask of a plan computed elsewhere (the large-boundary-bucket path).
int igs_shard_mask(const int64_t* gidx, int64_t n, const int64_t* plan, uint8_t* mask,
                   void* workspace, size_t workspace_bytes, void* stream) {
  if (!plan || n < 0 || (n > 0 && (!gidx || !mask))) return IGS_ERR_ARGUMENT;
  if (n == 0) return IGS_OK;
  shard::Layout L = shard::layout(n);
  if (!workspace || workspace_bytes < L.total) return IGS_ERR_WORKSPACE;
  long long grid = (n + shard::NT - 1) / shard::NT;
  const long long cap = 8LL * (sm_count() > 0 ? sm_count() : 148);
  if (grid > cap) grid = cap;
  shard::mask_kernel<<<(unsigned)grid, shard::NT, 0, (cudaStream_t)stream>>>(
      (const unsigned*)((char*)workspace + L.keys), (const unsigned*)((char*)workspace + L.klo),
      (const long long*)gidx, n,
      (const long long*)plan, mask);
  IGS_LAUNCH_CHECK();
  return IGS_OK;
}

int igs_shard_child_index(int64_t* gidx, int64_t count, const int64_t* plan, void* stream) {
  if (!gidx || !plan || count < 0) return IGS_ERR_ARGUMENT;
  shard::child_index_kernel<<<(unsigned)(2 * (sm_count() > 0 ? sm_count() : 148)), 256, 0,
                              (cudaStream_t)stream>>>((long long*)gidx, count,
                                                      (const long long*)plan);
  IGS_LAUNCH_CHECK();
  return IGS_OK;
}

}  // extern "C"
