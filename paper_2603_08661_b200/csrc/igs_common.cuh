// Shared device helpers for the sm_100a densification kernels.
//
// The whole library is compiled with --fmad=false: every a*b+c written in
// this code is two IEEE-rounded operations, as numpy/scipy evaluate them on
// the CPU.  Where a fused multiply-add is wanted it is written as fma().
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/igs_b200.h"

namespace igs {

void set_cuda_error(cudaError_t e);

#define IGS_CUDA_TRY(expr)                       \
  do {                                           \
    cudaError_t _e = (expr);                     \
    if (_e != cudaSuccess) {                     \
      ::igs::set_cuda_error(_e);                 \
      return IGS_ERR_CUDA;                       \
    }                                            \
  } while (0)

#define IGS_LAUNCH_CHECK() IGS_CUDA_TRY(cudaGetLastError())

inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

int sm_count();

// ---- memory-model helpers -------------------------------------------------

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned long long ld_acquire64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void spin_until_geq(const unsigned* p, unsigned target) {
  while (ld_acquire(p) < target) __nanosleep(64);
}

// Streaming 16-byte access (data touched once): keep it out of L1.
__device__ __forceinline__ float4 ld_stream_f4(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  return r;
}

// ---- numpy float semantics --------------------------------------------------

// np.clip(x, 0, 1) == minimum(maximum(x, 0), 1) with NaN propagation (numpy 2 clip loop).
__device__ __forceinline__ double np_clip01(double x) {
  if (x != x) return x;
  double m = x > 0.0 ? x : 0.0;
  return m < 1.0 ? m : 1.0;
}

// np.minimum(x, 1.0): (x <= 1 || isnan(x)) ? x : 1
__device__ __forceinline__ double np_min1(double x) { return (x <= 1.0 || x != x) ? x : 1.0; }

// np.mod(a, b) for float64 (npy_divmod): fmod, then shift into the divisor's sign.
__device__ __forceinline__ double np_mod(double a, double b) {
  double m = fmod(a, b);
  if (m != 0.0) {
    if ((b < 0.0) != (m < 0.0)) m = m + b;
  } else {
    m = copysign(0.0, b);
  }
  return m;
}

// floor((theta + pi/8) / (pi/4)) mod 4, edge_pipeline.py:102, evaluated as numpy does.
__device__ __forceinline__ int np_orientation_bin(double theta) {
  const double pi = 3.141592653589793;
  double q = floor((theta + pi / 8.0) / (pi / 4.0));
  long long b = (long long)q;  // astype(int)
  long long r = b % 4;
  if (r < 0) r += 4;           // python modulo
  return (int)r;
}

// glibc >= 2.35 __hypot (non-FMA x86-64 build), restated from libm.so.6 (glibc 2.39).
// Bit-exact with np.hypot; oracle/edge.py:hypot_glibc is the CPU restatement.
__device__ __forceinline__ double hypot_kernel(double ax, double ay) {
  double h = sqrt(ax * ax + ay * ay);  // correctly rounded sqrt (no fast-math)
  double t1, t2;
  if (h <= ay + ay) {
    double d = h - ay;
    t1 = ((d + d) - ax) * ax;
    double two_diff = (ax - ay) + (ax - ay);
    t2 = (d - two_diff) * d;
  } else {
    double d = h - ax;
    t1 = (d + d) * (ax - (ay + ay));
    t2 = ((4.0 * d) - ay) * ay + d * d;
  }
  return h - (t1 + t2) / (h + h);
}

static __device__ __noinline__ double hypot_glibc_slow(double x, double y);

// glibc hypot: the common range inline, the scaled / non-finite / trivial cases out of line.
__device__ __forceinline__ double hypot_glibc(double x, double y) {
  double ax = fabs(x), ay = fabs(y);
  if (ax < ay) {
    double t = ax;
    ax = ay;
    ay = t;
  }
  if (ay >= 0x1p-459 && ax <= 0x1p+511 && ay > ax * 0x1p-54) return hypot_kernel(ax, ay);
  return hypot_glibc_slow(x, y);
}

static __device__ __noinline__ double hypot_glibc_slow(double x, double y) {
  double ax = fabs(x), ay = fabs(y);
  if (!isfinite(ax) || !isfinite(ay)) {
    if (isinf(ax) || isinf(ay)) return __longlong_as_double(0x7ff0000000000000LL);
    return ax + ay;
  }
  if (ax < ay) {
    double t = ax;
    ax = ay;
    ay = t;
  }
  const double kLarge = 0x1p+511, kTiny = 0x1p-459, kEps = 0x1p-54;
  if (ax > kLarge) {
    if (ay <= ax * kEps) return ax + ay;
    return hypot_kernel(ax * 0x1p-600, ay * 0x1p-600) * 0x1p+600;
  }
  if (ay < kTiny) {
    if (ax >= ay * 0x1p+54) return ax + ay;
    return hypot_kernel(ax * 0x1p+600, ay * 0x1p+600) * 0x1p-600;
  }
  if (ay <= ax * kEps) return ax + ay;
  return hypot_kernel(ax, ay);
}

// The LAS logit-domain check of one parent (las_split.py: logit(sigmoid(o) * beta) needs the
// float32 value strictly inside (0, 1)), as the pre-pass computes it: e = expf(-o),
// r = (1 / (1 + e)) * beta.  Fast path without expf: for |o| <= 80, e is finite and positive, so
// 1 / (1 + e) lies in [1.8e-35, 1]; with 1e-6 <= beta < 1 the rounded product is then > 0 and
// <= beta < 1.  Anything else (NaN, large |o|, other beta) is evaluated exactly.
__device__ __forceinline__ bool las_opacity_bad(float o, float beta) {
  if (fabsf(o) <= 80.0f && beta >= 1e-6f && beta < 1.0f) return false;
  const float e = expf(-o);
  const float r = (1.0f / (1.0f + e)) * beta;
  return !(r > 0.0f && r < 1.0f);
}

// np.clip(x, 0, 1) on the bit pattern (integer pipe): NaN kept, x <= 0 (incl. -0) -> +0.
__device__ __forceinline__ double np_clip01_int(double x) {
  long long b = __double_as_longlong(x);
  if ((b & 0x7fffffffffffffffLL) > 0x7ff0000000000000LL) return x;  // NaN
  if (b <= 0) return 0.0;                                             // +0, -0, negatives
  return b > 0x3ff0000000000000LL ? 1.0 : x;
}

// Correctly rounded x / d given rd = RN(1/d) (Markstein: one FMA-residual correction).
__device__ __forceinline__ double div_by(double x, double d, double rd) {
  double q = x * rd;
  double r = fma(-q, d, x);
  return fma(r, rd, q);
}

// NMS direction bin of the gradient (gx, gy) -- identical to
// np_orientation_bin(np_mod(atan2(gy, gx), pi)) except within ~1e-12 rad of a
// bin boundary, where it falls back to evaluating that expression.
static __device__ __noinline__ int gradient_bin(double gx, double gy) {
  double ax = fabs(gx), ay = fabs(gy);
  if (ay == 0.0) return 0;         // theta in {0, pi, -pi} -> folded to 0 -> bin 0
  if (ax == 0.0 && isfinite(ay)) return 2;  // theta = +-pi/2 -> pi/2 -> bin 2
  const double kTan = 0.41421356237309503;  // tan(pi/8)
  double s = ax + ay;
  double d0 = fma(-kTan, ax, ay);   // > 0  <=> angle above pi/8 from the x axis
  double d2 = fma(-kTan, ay, ax);   // > 0  <=> angle below 3pi/8
  double tol = 1e-12 * s;
  if (!(fabs(d0) > tol) || !(fabs(d2) > tol)) {  // near a boundary, or non-finite
    return np_orientation_bin(np_mod(atan2(gy, gx), 3.141592653589793));
  }
  if (d0 < 0.0) return 0;
  if (d2 < 0.0) return 2;
  return ((gx > 0.0) == (gy > 0.0)) ? 1 : 3;
}

// ---- block helpers ----------------------------------------------------------

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Exclusive block-wide scan of one unsigned per thread (blockDim.x <= 1024).
// `warp_sums` must hold 32 entries.  Returns the exclusive prefix; *total gets the sum.
__device__ __forceinline__ unsigned block_exclusive_scan(unsigned v, unsigned* warp_sums,
                                                         unsigned* total) {
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  const unsigned nwarps = (blockDim.x + 31) >> 5;
  unsigned x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    unsigned y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= (unsigned)o) x += y;
  }
  if (lane == 31) warp_sums[warp] = x;
  __syncthreads();
  if (warp == 0) {
    unsigned s = lane < nwarps ? warp_sums[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      unsigned y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= (unsigned)o) s += y;
    }
    if (lane < nwarps) warp_sums[lane] = s;  // inclusive warp prefix
  }
  __syncthreads();
  unsigned base = warp ? warp_sums[warp - 1] : 0u;
  *total = warp_sums[nwarps - 1];
  __syncthreads();
  return base + x - v;
}

}  // namespace igs
