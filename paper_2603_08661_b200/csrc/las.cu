// Long-Axis-Split on sm_100a.
//
// Replaces splitkit.las_split.las_split_batch and the helpers it calls
// (/root/reference/pkg/src/splitkit/las_split.py:52-179, core.py:17-58,151-157).
//
//   las_prepare_kernel  one pass over the 1-byte mask: per-tile split counts
//                       plus the batch flags of the masked parents (bad
//                       quaternion, logit domain, the batch-global
//                       renormalisation trigger of core.py:45-46).
//   las_scan_kernel     exclusive scan of the tile counts -> slot offsets.
//   las_apply_kernel    per tile: ballot-ranked masked parents; per parent the
//                       float32 LAS arithmetic in numpy's operation order, the
//                       in-place +offset child (positions, log_scales,
//                       opacity_logits) and the appended -offset child at slot
//                       count + rank; rotations are cloned with one 16-byte
//                       access and the SH rows with warp-cooperative 16-byte
//                       copies of the tile's compacted parent list.
//   las2d_apply_kernel  the same for 2-D scenes (las_split.py:182-197).
// Two ways to drive them: igs_las_prepare, a host read of {n_split, flags}, the host
// checks, then igs_las_apply (the sharded path, whose checks are global); or the fused
// igs_las_split / igs_las2d_split, where the apply pass reads the summary itself and writes
// nothing when the host is about to raise, so the only host read comes after the split.
// Either way BudgetError / ValueError leave every column untouched, as in the reference.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include "igs_common.cuh"

namespace igs {
namespace las {

constexpr int NT = 256;
constexpr int PER = 2;
constexpr int TILE = NT * PER;  // Gaussians per block
constexpr int SUBS = PER * NT / 32;  // (sub-tile, warp) ballot groups per tile
static_assert(SUBS <= 32, "one warp scans the tile");

constexpr int MAX_CTAS = 2048;  // fused split: per-CTA totals / flags (grid <= 8 x SMs)

struct Layout {
  size_t tile_cnt, tile_off, cta_tot, cta_flag, guard, list, total;
};

Layout layout(long long count) {
  Layout L;
  long long tiles = (count + TILE - 1) / TILE;
  L.tile_cnt = 0;
  L.tile_off = align_up(sizeof(unsigned) * (size_t)(tiles + 1), 256);
  L.cta_tot = L.tile_off + align_up(sizeof(unsigned long long) * (size_t)(tiles + 1), 256);
  L.cta_flag = L.cta_tot + sizeof(unsigned long long) * MAX_CTAS;
  L.guard = L.cta_flag + sizeof(unsigned) * MAX_CTAS;  // the summary's device copy
  L.list = align_up(L.guard + 2 * sizeof(unsigned long long), 256);  // list-mode parents
  L.total = L.list + align_up(sizeof(unsigned) * (size_t)count, 256);
  return L;
}

// numpy float32: norm = sqrt((q*q).sum(-1)), summed left to right.
__device__ __forceinline__ float quat_norm(float4 q) {
  float s = q.x * q.x;
  s = s + q.y * q.y;
  s = s + q.z * q.z;
  s = s + q.w * q.w;
  return sqrtf(s);
}

// sigmoid(o) * beta in float32 (core.py:17-21 then las_split.py:96).
__device__ __forceinline__ float raw_opacity(float o, float beta) {
  float e = expf(-o);
  float s = 1.0f / (1.0f + e);
  return s * beta;
}

// Pre-pass of one tile: its split count (returned to thread 0) and the OR of its flags
// (returned to every thread's `flags_out` lane 0 of each warp; the caller reduces).
__device__ __forceinline__ unsigned prepare_tile(const uint8_t* __restrict__ mask,
                                                 const float* __restrict__ rot,
                                                 const float* __restrict__ opac, long long count,
                                                 float beta, long long tile, unsigned* warp_cnt,
                                                 unsigned& flags_out) {
  const long long base = tile * TILE;
  unsigned local = 0, flags = 0;
  bool m[PER];
  float4 q[PER];
  float o[PER];
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const long long i = base + j * NT + threadIdx.x;
    m[j] = i < count && mask[i];
  }
#pragma unroll
  for (int j = 0; j < PER; ++j) {  // every load first, then the checks
    const long long i = base + j * NT + threadIdx.x;
    if (m[j] && opac) {  // opac NULL: counts only (the caller has the flags)
      if (rot) q[j] = reinterpret_cast<const float4*>(rot)[i];
      o[j] = opac[i];
    }
  }
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    if (!m[j]) continue;
    ++local;
    if (!opac) continue;
    if (rot) {  // 3-D scenes: quaternion checks (2-D scenes pass rot = nullptr)
      float n = quat_norm(q[j]);
      if (!isfinite(n) || n == 0.0f) flags |= IGS_LAS_BAD_QUAT;
      else if (fabsf(n - 1.0f) > 1e-4f) flags |= IGS_LAS_RENORM;
    }
    if (las_opacity_bad(o[j], beta)) flags |= IGS_LAS_BAD_OPACITY;
  }
  unsigned w = __reduce_add_sync(0xffffffffu, local);
  flags_out = __reduce_or_sync(0xffffffffu, flags);
  if (lane_id() == 0) warp_cnt[threadIdx.x >> 5] = w;
  __syncthreads();
  unsigned t = 0;
  if (threadIdx.x == 0)
    for (int k = 0; k < NT / 32; ++k) t += warp_cnt[k];
  __syncthreads();  // warp_cnt is reused by the next tile
  return t;
}

__global__ void __launch_bounds__(NT) las_prepare_kernel(const uint8_t* __restrict__ mask,
                                                         const float* __restrict__ rot,
                                                         const float* __restrict__ opac,
                                                         long long count, float beta,
                                                         unsigned* tile_cnt,
                                                         unsigned long long* summary) {
  __shared__ unsigned warp_cnt[NT / 32];
  unsigned f = 0;
  const unsigned t = prepare_tile(mask, rot, opac, count, beta, blockIdx.x, warp_cnt, f);
  if (lane_id() == 0 && f) atomicOr(&summary[1], (unsigned long long)f);
  if (threadIdx.x == 0) tile_cnt[blockIdx.x] = t;
}

// Single block: exclusive scan of the tile counts; summary[0] = total.
__global__ void __launch_bounds__(1024) las_scan_kernel(const unsigned* tile_cnt, long long tiles,
                                                        unsigned long long* tile_off,
                                                        unsigned long long* summary) {
  __shared__ unsigned warp_sums[32];
  unsigned long long carry = 0;
  for (long long b = 0; b < tiles; b += blockDim.x) {
    long long i = b + threadIdx.x;
    unsigned v = i < tiles ? tile_cnt[i] : 0u;
    unsigned tot;
    unsigned ex = block_exclusive_scan(v, warp_sums, &tot);
    if (i < tiles) tile_off[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) summary[0] = carry;
}

// Clone the SH rows (Q4 float4 each) of a tile's compacted parents src_idx[0..n) to the
// consecutive appended rows slot0 ..: 16-byte streaming loads, U in flight per thread.
template <int Q4, int U>
__device__ __forceinline__ void clone_rows(float* sh, const long long* src_idx, unsigned n,
                                           unsigned long long slot0) {
  const float4* src = reinterpret_cast<const float4*>(sh);
  float4* dstp = reinterpret_cast<float4*>(sh);
  const unsigned total = n * Q4;
  for (unsigned e0 = threadIdx.x; e0 < total; e0 += U * NT) {
    float4 v[U];
    unsigned k[U], qq[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const unsigned e = e0 + u * NT;
      k[u] = e / Q4;
      qq[u] = e - k[u] * Q4;
      if (e < total) v[u] = ld_stream_f4(src + src_idx[k[u]] * Q4 + qq[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (e0 + u * NT < total) __stcs(dstp + (long long)(slot0 + k[u]) * Q4 + qq[u], v[u]);
  }
}

struct Consts {
  float alpha, log_alpha, log_gamma, beta;
};

// The split of one parent i (las_split.py:78-99 + core.py:32-58 column l): the +offset child
// in place, the -offset child at row dst (its rotation cloned; SH is cloned by the caller).
__device__ __forceinline__ void split_parent3(float* __restrict__ pos, float* __restrict__ ls,
                                              float* __restrict__ rot, float* __restrict__ opac,
                                              long long i, long long dst, const float (&lv)[3],
                                              const float (&pv)[3], float ov, float4 qv,
                                              const Consts& c, int renorm) {
  // _split_common (las_split.py:78-99)
  const float l0 = lv[0], l1 = lv[1], l2 = lv[2];
  int l = 0;  // np.argmax: first maximum (a NaN counts as the maximum)
  float best = l0;
  if (!(best != best)) {
    if (l1 > best || l1 != l1) { l = 1; best = l1; }
    if (!(best != best) && (l2 > best || l2 != l2)) { l = 2; best = l2; }
  }
  const float offset = expf(best) * c.alpha;
  float cl0 = l0 + c.log_gamma, cl1 = l1 + c.log_gamma, cl2 = l2 + c.log_gamma;
  const float cll = best + c.log_alpha;
  if (l == 0) cl0 = cll; else if (l == 1) cl1 = cll; else cl2 = cll;
  const float raw = raw_opacity(ov, c.beta);
  const float co = logf(raw / (1.0f - raw));

  // quat_to_rotmat (core.py:32-58), column l only (axis_displacement, las_split.py:62-75)
  const float4 q = qv;
  float w = q.x, x = q.y, y = q.z, z = q.w;
  if (renorm) {
    float n = quat_norm(q);
    w = w / n; x = x / n; y = y / n; z = z / n;
  }
  float c0, c1, c2;
  if (l == 0) {
    c0 = 1.0f - 2.0f * (y * y + z * z);
    c1 = 2.0f * (x * y + w * z);
    c2 = 2.0f * (x * z - w * y);
  } else if (l == 1) {
    c0 = 2.0f * (x * y - w * z);
    c1 = 1.0f - 2.0f * (x * x + z * z);
    c2 = 2.0f * (y * z + w * x);
  } else {
    c0 = 2.0f * (x * z + w * y);
    c1 = 2.0f * (y * z - w * x);
    c2 = 1.0f - 2.0f * (x * x + y * y);
  }
  const float d0 = c0 * offset, d1 = c1 * offset, d2 = c2 * offset;
  const float p0 = pv[0], p1 = pv[1], p2 = pv[2];
  // parent slot <- +offset child
  pos[3 * i] = p0 + d0;
  pos[3 * i + 1] = p1 + d1;
  pos[3 * i + 2] = p2 + d2;
  ls[3 * i] = cl0;
  ls[3 * i + 1] = cl1;
  ls[3 * i + 2] = cl2;
  opac[i] = co;
  // appended slot <- -offset child
  pos[3 * dst] = p0 - d0;
  pos[3 * dst + 1] = p1 - d1;
  pos[3 * dst + 2] = p2 - d2;
  ls[3 * dst] = cl0;
  ls[3 * dst + 1] = cl1;
  ls[3 * dst + 2] = cl2;
  opac[dst] = co;
  reinterpret_cast<float4*>(rot)[dst] = q;
}

struct TileSmem {
  unsigned warp_cnt[SUBS];
  unsigned warp_pre[SUBS];
  long long src_idx[TILE];
  unsigned total;
};

// Split pass of one 3-D tile whose appended children start at slot0 (= count + the number
// of masked parents before the tile).
template <int CLONE_U>
__device__ __forceinline__ void apply_tile3(float* __restrict__ pos, float* __restrict__ ls,
                                            float* __restrict__ rot, float* __restrict__ opac,
                                            float* __restrict__ sh, long long sh_floats,
                                            long long count, const uint8_t* __restrict__ mask,
                                            const Consts& c, int renorm, long long tile,
                                            unsigned long long slot0, TileSmem& ts) {
  unsigned* warp_cnt = ts.warp_cnt;
  unsigned* warp_pre = ts.warp_pre;
  long long* src_idx = ts.src_idx;
  unsigned& s_total = ts.total;
  const long long base = tile * TILE;
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  bool m[PER];
  unsigned wrank[PER];
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    long long i = base + j * NT + threadIdx.x;
    m[j] = i < count && mask[i];
    unsigned bal = __ballot_sync(0xffffffffu, m[j]);
    wrank[j] = __popc(bal & lanemask_lt());
    if (lane == 0) warp_cnt[j * (NT / 32) + warp] = __popc(bal);
  }
  __syncthreads();
  if (threadIdx.x < 32) {  // exclusive scan over (sub-tile, warp) in index order
    unsigned v = threadIdx.x < (unsigned)SUBS ? warp_cnt[threadIdx.x] : 0u;
    unsigned x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      unsigned y = __shfl_up_sync(0xffffffffu, x, o);
      if (threadIdx.x >= (unsigned)o) x += y;
    }
    if (threadIdx.x < (unsigned)SUBS) warp_pre[threadIdx.x] = x - v;
    if (threadIdx.x == 31) s_total = x;
  }
  __syncthreads();

  // every load of the thread's parents first (one memory latency), then the arithmetic
  float lv[PER][3], pv[PER][3], ov[PER];
  float4 qv[PER];
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    if (!m[j]) continue;
    const long long i = base + j * NT + threadIdx.x;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      lv[j][k] = ls[3 * i + k];
      pv[j][k] = pos[3 * i + k];
    }
    ov[j] = opac[i];
    qv[j] = reinterpret_cast<const float4*>(rot)[i];
  }
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    if (!m[j]) continue;
    const long long i = base + j * NT + threadIdx.x;
    const unsigned r = warp_pre[j * (NT / 32) + warp] + wrank[j];
    const long long dst = (long long)(slot0 + r);
    src_idx[r] = i;

    split_parent3(pos, ls, rot, opac, i, dst, lv[j], pv[j], ov[j], qv[j], c, renorm);
  }
  __syncthreads();

  // SH clone of the tile's parents into consecutive appended rows.
  const unsigned n = s_total;
  if (n == 0 || sh_floats == 0) return;
  if (sh_floats == 48) {  // SH degree 3: 12 float4 per row, four loads in flight per thread
    clone_rows<12, CLONE_U>(sh, src_idx, n, slot0);
  } else if (sh_floats == 12) {  // SH degree 1
    clone_rows<3, CLONE_U>(sh, src_idx, n, slot0);
  } else if ((sh_floats & 3) == 0) {
    const long long q4 = sh_floats >> 2;
    const float4* src = reinterpret_cast<const float4*>(sh);
    float4* dstp = reinterpret_cast<float4*>(sh);
    const long long total = (long long)n * q4;
    for (long long e = threadIdx.x; e < total; e += NT) {
      long long k = e / q4, qq = e - k * q4;
      float4 v = ld_stream_f4(src + src_idx[k] * q4 + qq);
      __stcs(dstp + (long long)(slot0 + k) * q4 + qq, v);
    }
  } else {
    const long long total = (long long)n * sh_floats;
    for (long long e = threadIdx.x; e < total; e += NT) {
      long long k = e / sh_floats, qq = e - k * sh_floats;
      sh[(long long)(slot0 + k) * sh_floats + qq] = sh[src_idx[k] * sh_floats + qq];
    }
  }
}

// guard (fused split): the pre-pass summary {n_split, flags} in device memory; the apply
// returns without writing when the host is about to raise (split_guard), and renormalises
// per its RENORM flag.
__device__ __forceinline__ bool split_guard(const unsigned long long* guard, long long count,
                                            long long capacity, unsigned long long bad) {
  const unsigned long long ns = guard[0], fl = guard[1];
  return ns != 0 && (unsigned long long)count + ns <= (unsigned long long)capacity && !(fl & bad);
}

__global__ void __launch_bounds__(NT) las_apply_kernel(
    float* __restrict__ pos, float* __restrict__ ls, float* __restrict__ rot,
    float* __restrict__ opac, float* __restrict__ sh, long long sh_floats, long long count,
    const uint8_t* __restrict__ mask, Consts c, int renorm,
    const unsigned long long* __restrict__ tile_off, const unsigned long long* guard,
    long long capacity) {
  __shared__ TileSmem ts;
  if (guard) {
    if (!split_guard(guard, count, capacity, IGS_LAS_BAD_QUAT | IGS_LAS_BAD_OPACITY)) return;
    renorm = (guard[1] & IGS_LAS_RENORM) != 0;
  }
  apply_tile3<8>(pos, ls, rot, opac, sh, sh_floats, count, mask, c, renorm, blockIdx.x,
              (unsigned long long)count + tile_off[blockIdx.x], ts);
}

// 2-D Long-Axis-Split (las_split.py:109-117, 182-197): the same slot rule and scale/opacity
// update; the displacement is column l of [[cos, -sin], [sin, cos]] (theta float32).
struct TileSmem2 {
  unsigned warp_cnt[SUBS];
  unsigned warp_pre[SUBS];
};

__device__ __forceinline__ void apply_tile2(float* __restrict__ pos, float* __restrict__ ls,
                                            float* __restrict__ theta, float* __restrict__ opac,
                                            float* __restrict__ col, long long count,
                                            const uint8_t* __restrict__ mask, const Consts& c,
                                            long long tile, unsigned long long slot0,
                                            TileSmem2& ts) {
  unsigned* warp_cnt = ts.warp_cnt;
  unsigned* warp_pre = ts.warp_pre;
  const long long base = tile * TILE;
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  bool m[PER];
  unsigned wrank[PER];
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    long long i = base + j * NT + threadIdx.x;
    m[j] = i < count && mask[i];
    unsigned bal = __ballot_sync(0xffffffffu, m[j]);
    wrank[j] = __popc(bal & lanemask_lt());
    if (lane == 0) warp_cnt[j * (NT / 32) + warp] = __popc(bal);
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    unsigned v = threadIdx.x < (unsigned)SUBS ? warp_cnt[threadIdx.x] : 0u;
    unsigned x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      unsigned y = __shfl_up_sync(0xffffffffu, x, o);
      if (threadIdx.x >= (unsigned)o) x += y;
    }
    if (threadIdx.x < (unsigned)SUBS) warp_pre[threadIdx.x] = x - v;
  }
  __syncthreads();
  // every load of the thread's parents first, then the arithmetic (as the 3-D pass)
  float lv[PER][2], pv[PER][2], ov[PER], tv[PER], cv[PER][3];
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    if (!m[j]) continue;
    const long long i = base + j * NT + threadIdx.x;
    lv[j][0] = ls[2 * i];
    lv[j][1] = ls[2 * i + 1];
    pv[j][0] = pos[2 * i];
    pv[j][1] = pos[2 * i + 1];
    ov[j] = opac[i];
    tv[j] = theta[i];
#pragma unroll
    for (int k = 0; k < 3; ++k) cv[j][k] = col[3 * i + k];
  }
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    if (!m[j]) continue;
    const long long i = base + j * NT + threadIdx.x;
    const long long dst = (long long)(slot0 + warp_pre[j * (NT / 32) + warp] + wrank[j]);
    const float l0 = lv[j][0], l1 = lv[j][1];
    int l = 0;  // np.argmax: first maximum (a NaN counts as the maximum)
    float best = l0;
    if (!(best != best) && (l1 > best || l1 != l1)) {
      l = 1;
      best = l1;
    }
    const float offset = expf(best) * c.alpha;
    float cl0 = l0 + c.log_gamma, cl1 = l1 + c.log_gamma;
    const float cll = best + c.log_alpha;
    if (l == 0) cl0 = cll;
    else cl1 = cll;
    const float raw = raw_opacity(ov[j], c.beta);
    const float co = logf(raw / (1.0f - raw));
    const float th = tv[j];
    const float ct = cosf(th), st = sinf(th);
    const float d0 = (l == 0 ? ct : -st) * offset, d1 = (l == 0 ? st : ct) * offset;
    const float p0 = pv[j][0], p1 = pv[j][1];
    pos[2 * i] = p0 + d0;
    pos[2 * i + 1] = p1 + d1;
    ls[2 * i] = cl0;
    ls[2 * i + 1] = cl1;
    opac[i] = co;
    pos[2 * dst] = p0 - d0;
    pos[2 * dst + 1] = p1 - d1;
    ls[2 * dst] = cl0;
    ls[2 * dst + 1] = cl1;
    theta[dst] = th;
    opac[dst] = co;
    col[3 * dst] = cv[j][0];
    col[3 * dst + 1] = cv[j][1];
    col[3 * dst + 2] = cv[j][2];
  }
}

__global__ void __launch_bounds__(NT) las2d_apply_kernel(
    float* __restrict__ pos, float* __restrict__ ls, float* __restrict__ theta,
    float* __restrict__ opac, float* __restrict__ col, long long count,
    const uint8_t* __restrict__ mask, Consts c, const unsigned long long* __restrict__ tile_off,
    const unsigned long long* guard, long long capacity) {
  __shared__ TileSmem2 ts;
  if (guard && !split_guard(guard, count, capacity, IGS_LAS_BAD_OPACITY)) return;
  apply_tile2(pos, ls, theta, opac, col, count, mask, c, blockIdx.x,
              (unsigned long long)count + tile_off[blockIdx.x], ts);
}

// ------------------------------------------------------------ fused split
// igs_las_split / igs_las2d_split = las_prepare_coop_kernel + the guarded apply kernel, back to
// back on the stream with no host round trip and no memset:
//   las_prepare_coop_kernel  one cooperative launch, each CTA owning a contiguous range of
//     tiles.  Phase 1: the pre-pass of its tiles (tile counts; the CTA's total and flags to its
//     own slot, so no zero-initialised memory).  Grid barrier.  Phase 2: every CTA reads all CTA
//     totals / flags, writes the slot offsets of its tiles, and CTA 0 writes the summary
//     {n_split, flags} to the workspace (the apply's guard) and to the caller's summary.
//   las_apply_kernel / las2d_apply_kernel with that guard: every block returns before writing
//     when the host is about to raise, so the scene is untouched as in the reference.
// One warp's view of a 512-parent tile: lane L holds mask bytes [16 L, 16 L + 16) of the tile
// as a 16-bit set of masked parents (ascending index = lane-major bit order).
__device__ __forceinline__ unsigned tile_lane_bits(const uint8_t* __restrict__ mask,
                                                   long long count, long long tile, bool vec) {
  const long long i0 = tile * TILE + 16 * (long long)lane_id();
  unsigned bits = 0;
  if (vec && i0 + 16 <= count) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(mask + i0));
    const unsigned w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const unsigned r = __vcmpne4(w[k], 0u);  // 0xff per nonzero byte
      bits |= (((r >> 7) & 1u) | ((r >> 14) & 2u) | ((r >> 21) & 4u) | ((r >> 28) & 8u)) << (4 * k);
    }
  } else {
#pragma unroll
    for (int k = 0; k < 16; ++k)
      if (i0 + k < count && mask[i0 + k]) bits |= 1u << k;
  }
  return bits;
}

// Fused split pre-pass, one cooperative launch; each CTA owns tiles [t0, t1), one warp per tile
// (no block barrier per tile).  Phase 1: per tile, the masked count (tile_cnt) and the batch
// flags of its masked parents; the CTA's total and flags to its own slot.  Grid barrier.
// Phase 2: every CTA reads all CTA totals / flags, scans its own tiles into slot offsets
// (tile_off), and CTA 0 writes the summary.  Phase 3 (list mode): each warp writes its tiles'
// masked parents, in index order, at their slots.
template <bool D3>
__global__ void __launch_bounds__(NT) las_prepare_coop_kernel(
    const uint8_t* __restrict__ mask, const float* __restrict__ rot,
    const float* __restrict__ opac, long long count, float beta, long long tiles,
    unsigned* tile_cnt, unsigned long long* tile_off, unsigned long long* cta_tot,
    unsigned* cta_flag, unsigned long long* guard, int64_t* summary, unsigned* list) {
  constexpr int NW = NT / 32;
  __shared__ unsigned long long wtot[NW];
  __shared__ unsigned wflag[NW];
  __shared__ unsigned long long s_pre, s_tot;
  __shared__ unsigned s_flags;
  const long long G = gridDim.x, b = blockIdx.x;
  const long long t0 = b * tiles / G, t1 = (b + 1) * tiles / G;
  const int lane = lane_id(), warp = threadIdx.x >> 5;
  const bool vec = (((uintptr_t)mask) & 15) == 0;
  unsigned long long tot = 0;
  unsigned flags = 0;
  if (t1 - t0 <= 2) {  // few tiles per CTA (small batches): the whole CTA on each tile
    __shared__ unsigned warp_cnt[NW];
    for (long long t = t0; t < t1; ++t) {
      unsigned f = 0;
      const unsigned n = prepare_tile(mask, D3 ? rot : nullptr, opac, count, beta, t, warp_cnt, f);
      flags |= f;
      if (threadIdx.x == 0) tile_cnt[t] = n;
      tot += n;  // block-uniform
    }
    if (warp != 0) tot = 0;  // counted once, by warp 0
  }
  for (long long t = t0 + warp; t1 - t0 > 2 && t < t1; t += NW) {
    const unsigned bits = tile_lane_bits(mask, count, t, vec);
    unsigned f = 0;
    if (opac && __any_sync(0xffffffffu, bits != 0u)) {  // opac NULL: counts only
      // the flag inputs in coalesced order: row tile * 512 + 32 k + lane, its mask bit from
      // the lane holding it (lane 2k + lane / 16, bit lane % 16); two halves of 8 loads each
      const long long tb = t * TILE;
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        float4 q[8];
        float o[8];
        bool m[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {  // every load of the half first, then the checks
          const int k = 8 * half + j;
          const unsigned ob = __shfl_sync(0xffffffffu, bits, 2 * k + (lane >> 4));
          m[j] = (ob >> (lane & 15)) & 1u;
          const long long i = tb + 32 * k + lane;
          if (m[j]) {
            if (D3) q[j] = __ldg(reinterpret_cast<const float4*>(rot) + i);
            o[j] = __ldg(opac + i);
          }
        }
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (m[j]) {
            if (D3) {
              const float n = quat_norm(q[j]);
              if (!isfinite(n) || n == 0.0f) f |= IGS_LAS_BAD_QUAT;
              else if (fabsf(n - 1.0f) > 1e-4f) f |= IGS_LAS_RENORM;
            }
            if (las_opacity_bad(o[j], beta)) f |= IGS_LAS_BAD_OPACITY;
          }
      }
    }
    const unsigned cnt = __reduce_add_sync(0xffffffffu, (unsigned)__popc(bits));
    flags |= __reduce_or_sync(0xffffffffu, f);
    if (lane == 0) tile_cnt[t] = cnt;
    tot += cnt;
  }
  if (lane == 0) {
    wtot[warp] = tot;
    wflag[warp] = flags;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long ct = 0;
    unsigned cf = 0;
#pragma unroll
    for (int k = 0; k < NW; ++k) {
      ct += wtot[k];
      cf |= wflag[k];
    }
    cta_tot[b] = ct;
    cta_flag[b] = cf;
    s_pre = 0;
    s_tot = 0;
    s_flags = 0;
  }
  cooperative_groups::this_grid().sync();
  unsigned long long pre = 0, all = 0;
  unsigned fl = 0;
  for (long long k = threadIdx.x; k < G; k += NT) {
    const unsigned long long v = __ldcg(&cta_tot[k]);
    all += v;
    if (k < b) pre += v;
    fl |= __ldcg(&cta_flag[k]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    pre += __shfl_down_sync(0xffffffffu, pre, o);
    all += __shfl_down_sync(0xffffffffu, all, o);
  }
  fl = __reduce_or_sync(0xffffffffu, fl);
  if (lane == 0) {
    atomicAdd(&s_pre, pre);
    atomicAdd(&s_tot, all);
    atomicOr(&s_flags, fl);
  }
  __syncthreads();
  if (b == 0 && threadIdx.x == 0) {
    guard[0] = s_tot;
    guard[1] = s_flags;
    // summary[1] last: a host polling it (igs_wait_host_word) then reads a complete summary
    summary[0] = (int64_t)s_tot;
    __threadfence_system();
    summary[1] = (int64_t)s_flags;
  }
  // slot offsets of this CTA's tiles: a block scan of their counts, NT tiles per round
  unsigned long long carry = s_pre;
  for (long long base = t0; base < t1; base += NT) {
    const long long t = base + threadIdx.x;
    const unsigned long long v = t < t1 ? (unsigned long long)__ldcg(&tile_cnt[t]) : 0ull;
    unsigned long long x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wtot[warp] = x;
    __syncthreads();
    unsigned long long wpre = 0, round = 0;
#pragma unroll
    for (int k = 0; k < NW; ++k) {
      if (k < warp) wpre += wtot[k];
      round += wtot[k];
    }
    if (t < t1) tile_off[t] = carry + wpre + x - v;
    carry += round;
    __syncthreads();
  }
  if (!list) return;
  __syncthreads();  // this CTA's tile_off writes -> its warps' reads below
  for (long long t = t0 + warp; t < t1; t += NW) {
    const unsigned bits = tile_lane_bits(mask, count, t, vec);
    const unsigned c = (unsigned)__popc(bits);
    unsigned x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    unsigned long long at = __ldcg(&tile_off[t]) + (x - c);
    const unsigned i0 = (unsigned)(t * TILE + 16 * (long long)lane);
    unsigned rest = bits;
    while (rest) {
      const int k = __ffs(rest) - 1;
      rest &= rest - 1u;
      list[at++] = i0 + (unsigned)k;
    }
  }
}

// List-mode split (sparse masks): persistent blocks walk the compacted parent list in chunks
// of NT; child j of the list goes to row count + j (ascending parent order, as the tile
// mode).  Coalesced list reads, one gather per parent record, the chunk's SH rows cloned with
// cooperative 16-byte copies.  Guarded by {n_split, flags} like las_apply_kernel.
template <int CLONE_U>
__global__ void __launch_bounds__(NT, 4) las_apply_list_kernel(
    float* __restrict__ pos, float* __restrict__ ls, float* __restrict__ rot,
    float* __restrict__ opac, float* __restrict__ sh, long long sh_floats, long long count,
    const unsigned* __restrict__ list, Consts c, const unsigned long long* guard,
    long long capacity) {
  __shared__ long long src[NT];
  if (!split_guard(guard, count, capacity, IGS_LAS_BAD_QUAT | IGS_LAS_BAD_OPACITY)) return;
  const int renorm = (guard[1] & IGS_LAS_RENORM) != 0;
  const long long ns = (long long)guard[0];
  for (long long b0 = (long long)blockIdx.x * NT; b0 < ns; b0 += (long long)gridDim.x * NT) {
    const long long j = b0 + threadIdx.x;
    const bool v = j < ns;
    const long long i = v ? (long long)list[j] : 0;
    float lv[3], pv[3], ov = 0.0f;
    float4 qv = make_float4(0.f, 0.f, 0.f, 0.f);
    if (v) {
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        lv[k] = ls[3 * i + k];
        pv[k] = pos[3 * i + k];
      }
      ov = opac[i];
      qv = reinterpret_cast<const float4*>(rot)[i];
      split_parent3(pos, ls, rot, opac, i, count + j, lv, pv, ov, qv, c, renorm);
    }
    src[threadIdx.x] = i;
    __syncthreads();
    const unsigned n = (unsigned)min((long long)NT, ns - b0);
    const unsigned long long slot0 = (unsigned long long)(count + b0);
    if (sh_floats == 48) clone_rows<12, CLONE_U>(sh, src, n, slot0);
    else if (sh_floats == 12) clone_rows<3, CLONE_U>(sh, src, n, slot0);
    else if ((sh_floats & 3) == 0) {
      const long long q4 = sh_floats >> 2;
      const float4* s4 = reinterpret_cast<const float4*>(sh);
      float4* d4 = reinterpret_cast<float4*>(sh);
      for (long long e = threadIdx.x; e < (long long)n * q4; e += NT) {
        const long long k = e / q4, qq = e - k * q4;
        __stcs(d4 + (long long)(slot0 + k) * q4 + qq, ld_stream_f4(s4 + src[k] * q4 + qq));
      }
    } else {
      for (long long e = threadIdx.x; e < (long long)n * sh_floats; e += NT) {
        const long long k = e / sh_floats, qq = e - k * sh_floats;
        sh[(long long)(slot0 + k) * sh_floats + qq] = sh[src[k] * sh_floats + qq];
      }
    }
    __syncthreads();
  }
}

inline int list_grid() {
  static int g = 0;
  if (!g) {
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, las_apply_list_kernel<4>, NT, 0) !=
        cudaSuccess || n < 1)
      n = 1;
    g = n * (sm_count() > 0 ? sm_count() : 148);
  }
  return g;
}

template <bool D3>
int launch_prepare_coop(const uint8_t* mask, const float* rot, const float* opac, long long count,
                        float beta, void* workspace, size_t workspace_bytes, int64_t* summary,
                        cudaStream_t s, const unsigned long long** guard_out,
                        const unsigned long long** tile_off_out, bool want_list = false) {
  Layout L = layout(count);
  if (!workspace || workspace_bytes < L.total) return IGS_ERR_WORKSPACE;
  char* w = (char*)workspace;
  const long long tiles = (count + TILE - 1) / TILE;
  static int per_sm[2] = {-1, -1};
  int& bps = per_sm[D3 ? 1 : 0];
  if (bps < 0) {
    int n = 0;
    IGS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, las_prepare_coop_kernel<D3>, NT, 0));
    bps = n;
  }
  long long grid = (long long)bps * sm_count();
  if (grid > MAX_CTAS) grid = MAX_CTAS;
  if (grid > tiles) grid = tiles;
  if (grid < 1) return IGS_ERR_CUDA;
  unsigned* tile_cnt = (unsigned*)(w + L.tile_cnt);
  unsigned long long* tile_off = (unsigned long long*)(w + L.tile_off);
  unsigned long long* cta_tot = (unsigned long long*)(w + L.cta_tot);
  unsigned* cta_flag = (unsigned*)(w + L.cta_flag);
  unsigned long long* guard = (unsigned long long*)(w + L.guard);
  unsigned* list = want_list ? (unsigned*)(w + L.list) : nullptr;
  void* args[] = {&mask, &rot, &opac, &count, &beta, (void*)&tiles, &tile_cnt, &tile_off,
                  &cta_tot, &cta_flag, &guard, &summary, &list};
  IGS_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)las_prepare_coop_kernel<D3>,
                                           dim3((unsigned)grid), dim3(NT), args, 0, s));
  *guard_out = guard;
  *tile_off_out = tile_off;
  return IGS_OK;
}

}  // namespace las
}  // namespace igs

using namespace igs;

extern "C" {

int igs_las_workspace_bytes(int64_t count, size_t* bytes) {
  if (!bytes || count < 0) return IGS_ERR_ARGUMENT;
  *bytes = las::layout(count).total;
  return IGS_OK;
}

int igs_las_prepare(const uint8_t* mask, const float* rotations, const float* opacity_logits,
                    int64_t count, float beta, void* workspace, size_t workspace_bytes,
                    int64_t* summary, void* stream) {
  if (count < 0 || !summary) return IGS_ERR_ARGUMENT;
  if (count > 0 && (!mask || !opacity_logits)) return IGS_ERR_ARGUMENT;
  if (count > 0 && ((uintptr_t)rotations & 15)) return IGS_ERR_ARGUMENT;  // nullable: 2-D
  las::Layout L = las::layout(count);
  if (!workspace || workspace_bytes < L.total) return IGS_ERR_WORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  IGS_CUDA_TRY(cudaMemsetAsync(summary, 0, 2 * sizeof(int64_t), s));
  if (count == 0) return IGS_OK;
  long long tiles = (count + las::TILE - 1) / las::TILE;
  unsigned* tile_cnt = (unsigned*)((char*)workspace + L.tile_cnt);
  unsigned long long* tile_off = (unsigned long long*)((char*)workspace + L.tile_off);
  las::las_prepare_kernel<<<(unsigned)tiles, las::NT, 0, s>>>(
      mask, rotations, opacity_logits, count, beta, tile_cnt, (unsigned long long*)summary);
  IGS_LAUNCH_CHECK();
  las::las_scan_kernel<<<1, 1024, 0, s>>>(tile_cnt, tiles, tile_off,
                                          (unsigned long long*)summary);
  IGS_LAUNCH_CHECK();
  return IGS_OK;
}

int igs_las_apply(float* positions, float* log_scales, float* rotations, float* opacity_logits,
                  float* sh, int64_t sh_floats, int64_t count, int64_t capacity,
                  const uint8_t* mask, float alpha, float log_alpha, float log_gamma, float beta,
                  int renormalize, void* workspace, size_t workspace_bytes, void* stream) {
  if (count < 0 || capacity < count || sh_floats < 0) return IGS_ERR_ARGUMENT;
  if (count == 0) return IGS_OK;
  if (!positions || !log_scales || !rotations || !opacity_logits || !mask) return IGS_ERR_ARGUMENT;
  if (sh_floats > 0 && !sh) return IGS_ERR_ARGUMENT;
  if (((uintptr_t)rotations & 15) || (sh_floats % 4 == 0 && ((uintptr_t)sh & 15)))
    return IGS_ERR_ARGUMENT;
  las::Layout L = las::layout(count);
  if (!workspace || workspace_bytes < L.total) return IGS_ERR_WORKSPACE;
  long long tiles = (count + las::TILE - 1) / las::TILE;
  las::Consts c{alpha, log_alpha, log_gamma, beta};
  las::las_apply_kernel<<<(unsigned)tiles, las::NT, 0, (cudaStream_t)stream>>>(
      positions, log_scales, rotations, opacity_logits, sh, sh_floats, count, mask, c,
      renormalize, (const unsigned long long*)((char*)workspace + L.tile_off), nullptr, 0);
  IGS_LAUNCH_CHECK();
  return IGS_OK;
}

int igs_las2d_apply(float* positions, float* log_scales, float* thetas, float* opacity_logits,
                    float* colors, int64_t count, int64_t capacity, const uint8_t* mask,
                    float alpha, float log_alpha, float log_gamma, float beta, void* workspace,
                    size_t workspace_bytes, void* stream) {
  if (count < 0 || capacity < count) return IGS_ERR_ARGUMENT;
  if (count == 0) return IGS_OK;
  if (!positions || !log_scales || !thetas || !opacity_logits || !colors || !mask)
    return IGS_ERR_ARGUMENT;
  las::Layout L = las::layout(count);
  if (!workspace || workspace_bytes < L.total) return IGS_ERR_WORKSPACE;
  long long tiles = (count + las::TILE - 1) / las::TILE;
  las::Consts c{alpha, log_alpha, log_gamma, beta};
  las::las2d_apply_kernel<<<(unsigned)tiles, las::NT, 0, (cudaStream_t)stream>>>(
      positions, log_scales, thetas, opacity_logits, colors, count, mask, c,
      (const unsigned long long*)((char*)workspace + L.tile_off), nullptr, 0);
  IGS_LAUNCH_CHECK();
  return IGS_OK;
}

static int las_split_impl(float* positions, float* log_scales, float* rotations,
                          float* opacity_logits, float* sh, int64_t sh_floats, int64_t count,
                          int64_t capacity, const uint8_t* mask, float alpha, float log_alpha,
                          float log_gamma, float beta, void* workspace, size_t workspace_bytes,
                          int64_t* summary, void* stream, bool list_mode) {
  if (count < 0 || capacity < count || sh_floats < 0 || !summary) return IGS_ERR_ARGUMENT;
  if (count > 0 && (!positions || !log_scales || !rotations || !opacity_logits || !mask))
    return IGS_ERR_ARGUMENT;
  if (sh_floats > 0 && count > 0 && !sh) return IGS_ERR_ARGUMENT;
  if (((uintptr_t)rotations & 15) || (sh_floats % 4 == 0 && ((uintptr_t)sh & 15)))
    return IGS_ERR_ARGUMENT;
  cudaStream_t s = (cudaStream_t)stream;
  if (count == 0) {
    IGS_CUDA_TRY(cudaMemsetAsync(summary, 0, 2 * sizeof(int64_t), s));
    return IGS_OK;
  }
  const unsigned long long *guard = nullptr, *tile_off = nullptr;
  int st = las::launch_prepare_coop<true>(mask, rotations, opacity_logits, count, beta, workspace,
                                          workspace_bytes, summary, s, &guard, &tile_off,
                                          list_mode);
  if (st != IGS_OK) return st;
  const long long tiles = (count + las::TILE - 1) / las::TILE;
  las::Consts c{alpha, log_alpha, log_gamma, beta};
  las::Layout L = las::layout(count);
  if (list_mode)
    las::las_apply_list_kernel<4><<<las::list_grid(), las::NT, 0, s>>>(
        positions, log_scales, rotations, opacity_logits, sh, sh_floats, count,
        (const unsigned*)((char*)workspace + L.list), c, guard, capacity);
  else
    las::las_apply_kernel<<<(unsigned)tiles, las::NT, 0, s>>>(
        positions, log_scales, rotations, opacity_logits, sh, sh_floats, count, mask, c, 0,
        tile_off, guard, capacity);
  IGS_LAUNCH_CHECK();
  return IGS_OK;
}

int igs_las_split(float* positions, float* log_scales, float* rotations, float* opacity_logits,
                  float* sh, int64_t sh_floats, int64_t count, int64_t capacity,
                  const uint8_t* mask, float alpha, float log_alpha, float log_gamma, float beta,
                  void* workspace, size_t workspace_bytes, int64_t* summary, void* stream) {
  return las_split_impl(positions, log_scales, rotations, opacity_logits, sh, sh_floats, count,
                        capacity, mask, alpha, log_alpha, log_gamma, beta, workspace,
                        workspace_bytes, summary, stream, false);
}

int igs_las_split_packed(const IgsLasSplitArgs* a) {
  if (!a) return IGS_ERR_ARGUMENT;
  return las_split_impl(a->positions, a->log_scales, a->rotations, a->opacity_logits, a->sh,
                        a->sh_floats, a->count, a->capacity, a->mask, a->alpha, a->log_alpha,
                        a->log_gamma, a->beta, a->workspace, a->workspace_bytes, a->summary,
                        a->stream, a->sparse != 0);
}

int igs_las_split_sparse(float* positions, float* log_scales, float* rotations,
                         float* opacity_logits, float* sh, int64_t sh_floats, int64_t count,
                         int64_t capacity, const uint8_t* mask, float alpha, float log_alpha,
                         float log_gamma, float beta, void* workspace, size_t workspace_bytes,
                         int64_t* summary, void* stream) {
  return las_split_impl(positions, log_scales, rotations, opacity_logits, sh, sh_floats, count,
                        capacity, mask, alpha, log_alpha, log_gamma, beta, workspace,
                        workspace_bytes, summary, stream, true);
}

int igs_las2d_split(float* positions, float* log_scales, float* thetas, float* opacity_logits,
                    float* colors, int64_t count, int64_t capacity, const uint8_t* mask,
                    float alpha, float log_alpha, float log_gamma, float beta, void* workspace,
                    size_t workspace_bytes, int64_t* summary, void* stream) {
  if (count < 0 || capacity < count || !summary) return IGS_ERR_ARGUMENT;
  if (count > 0 && (!positions || !log_scales || !thetas || !opacity_logits || !colors || !mask))
    return IGS_ERR_ARGUMENT;
  cudaStream_t s = (cudaStream_t)stream;
  if (count == 0) {
    IGS_CUDA_TRY(cudaMemsetAsync(summary, 0, 2 * sizeof(int64_t), s));
    return IGS_OK;
  }
  const unsigned long long *guard = nullptr, *tile_off = nullptr;
  int st = las::launch_prepare_coop<false>(mask, nullptr, opacity_logits, count, beta, workspace,
                                           workspace_bytes, summary, s, &guard, &tile_off);
  if (st != IGS_OK) return st;
  const long long tiles = (count + las::TILE - 1) / las::TILE;
  las::Consts c{alpha, log_alpha, log_gamma, beta};
  las::las2d_apply_kernel<<<(unsigned)tiles, las::NT, 0, s>>>(
      positions, log_scales, thetas, opacity_logits, colors, count, mask, c, tile_off, guard,
      capacity);
  IGS_LAUNCH_CHECK();
  return IGS_OK;
}

// The split of one shard under a decision taken elsewhere (the sharded densify step): the
// cooperative pre-pass for this shard's slot offsets, then the apply pass guarded by the
// device words guard = {n_split or 0, batch flags} (RENORM / domain flags over every rank's
// selected parents) against the shard's reserved rows.
int igs_las_split_guarded(float* positions, float* log_scales, float* rotations,
                          float* opacity_logits, float* sh_or_colors, int64_t sh_floats,
                          int dims, int64_t count, int64_t reserved_rows, const uint8_t* mask,
                          float alpha, float log_alpha, float log_gamma, float beta,
                          const int64_t* guard, void* workspace, size_t workspace_bytes,
                          void* stream) {
  if (count < 0 || reserved_rows < count || !guard || (dims != 2 && dims != 3))
    return IGS_ERR_ARGUMENT;
  if (count == 0) return IGS_OK;
  if (!positions || !log_scales || !rotations || !opacity_logits || !sh_or_colors || !mask)
    return IGS_ERR_ARGUMENT;
  if (dims == 3 && (((uintptr_t)rotations & 15) || (sh_floats % 4 == 0 && ((uintptr_t)sh_or_colors & 15))))
    return IGS_ERR_ARGUMENT;
  cudaStream_t s = (cudaStream_t)stream;
  las::Layout L = las::layout(count);
  if (!workspace || workspace_bytes < L.total) return IGS_ERR_WORKSPACE;
  int64_t* local_summary = (int64_t*)((char*)workspace + L.guard);
  const unsigned long long *local_guard = nullptr, *tile_off = nullptr;
  const int st = dims == 3
      ? las::launch_prepare_coop<true>(mask, nullptr, nullptr, count, beta, workspace,
                                       workspace_bytes, local_summary, s, &local_guard, &tile_off,
                                       true)  // counts and the parent list: the flags are in guard
      : las::launch_prepare_coop<false>(mask, nullptr, opacity_logits, count, beta, workspace,
                                        workspace_bytes, local_summary, s, &local_guard,
                                        &tile_off);
  if (st != IGS_OK) return st;
  const long long tiles = (count + las::TILE - 1) / las::TILE;
  las::Consts c{alpha, log_alpha, log_gamma, beta};
  if (dims == 3)
    las::las_apply_list_kernel<4><<<las::list_grid(), las::NT, 0, s>>>(
        positions, log_scales, rotations, opacity_logits, sh_or_colors, sh_floats, count,
        (const unsigned*)((char*)workspace + L.list), c, (const unsigned long long*)guard,
        reserved_rows);
  else
    las::las2d_apply_kernel<<<(unsigned)tiles, las::NT, 0, s>>>(
        positions, log_scales, rotations, opacity_logits, sh_or_colors, count, mask, c, tile_off,
        (const unsigned long long*)guard, reserved_rows);
  IGS_LAUNCH_CHECK();
  return IGS_OK;
}

}  // extern "C"
