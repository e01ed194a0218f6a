// Densification statistics on sm_100a: fold one iteration's positional gradients into the
// per-primitive running sums, fused with their norm.
//
// Replaces the trainer's `accumulate_grads(stats, np.hypot(g[:, 0], g[:, 1]))`
// (/root/reference/pkg/src/splitkit/splat2d.py:393-394 with densify_controller.py:54-63):
// grad_sum[i] += hypot(gx, gy) with glibc's hypot / hypotf for float64 / float32 gradients
// (bit-exact with np.hypot on the same dtype) and one rounded float64 add, so the statistics
// the selection reads never leave the device.
#include <cuda_runtime.h>
#include <stdint.h>

#include "igs_common.cuh"

namespace igs {
namespace stats {

constexpr int NT = 256;

// np.hypot on float32 pairs is glibc's hypotf: the double sqrt of the double sum of squares,
// rounded to float (inf wins over NaN).
__device__ __forceinline__ float hypotf_glibc(float x, float y) {
  if (isinf(x) || isinf(y)) return __int_as_float(0x7f800000);
  const double dx = x, dy = y;
  return (float)sqrt(dx * dx + dy * dy);
}

constexpr int U = 4;  // primitives per thread, every load issued before the arithmetic

template <typename T>
struct Pair;
template <>
struct Pair<double> { using V = double2; };
template <>
struct Pair<float> { using V = float2; };

// PAIR: g is aligned for one (gx, gy) vector load per primitive.
// STORE: the first accumulation after a reset (grad_sum holds no values yet): grad_sum[i] =
// 0.0 + h, what numpy's zeros + h gives, without reading the stale buffer.
template <typename T, bool PAIR, bool STORE>
__global__ void __launch_bounds__(NT) accumulate_kernel(double* __restrict__ grad_sum,
                                                        const T* __restrict__ g, long long n) {
  const long long base = (long long)blockIdx.x * NT * U + threadIdx.x;
  T gx[U], gy[U];
  double sum[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const long long i = base + (long long)u * NT;
    if (i < n) {
      if (PAIR) {
        const typename Pair<T>::V v = __ldcs(reinterpret_cast<const typename Pair<T>::V*>(g) + i);
        gx[u] = v.x;
        gy[u] = v.y;
      } else {
        gx[u] = g[2 * i];
        gy[u] = g[2 * i + 1];
      }
      sum[u] = STORE ? 0.0 : grad_sum[i];
    }
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const long long i = base + (long long)u * NT;
    if (i >= n) break;
    double h;
    if (sizeof(T) == 8) h = hypot_glibc((double)gx[u], (double)gy[u]);
    else h = (double)hypotf_glibc((float)gx[u], (float)gy[u]);
    grad_sum[i] = sum[u] + h;
  }
}

}  // namespace stats
}  // namespace igs

using namespace igs;

extern "C" {

int igs_accumulate_grad_norms(double* grad_sum, const void* grads, int dtype, int64_t n,
                              void* stream) {
  const bool store = (dtype & IGS_ACCUM_STORE) != 0;
  dtype &= ~IGS_ACCUM_STORE;
  if (n < 0 || (dtype != IGS_F32 && dtype != IGS_F64)) return IGS_ERR_ARGUMENT;
  if (n == 0) return IGS_OK;
  if (!grad_sum || !grads) return IGS_ERR_ARGUMENT;
  const unsigned blocks = (unsigned)((n + stats::NT * stats::U - 1) / (stats::NT * stats::U));
  cudaStream_t st = (cudaStream_t)stream;
  const uintptr_t a = (uintptr_t)grads;
  const bool pair = a % (dtype == IGS_F64 ? 16 : 8) == 0;
#define IGS_ACCUM(T, P, S) \
  stats::accumulate_kernel<T, P, S><<<blocks, stats::NT, 0, st>>>(grad_sum, (const T*)grads, n)
  if (dtype == IGS_F64) {
    if (store) { if (pair) IGS_ACCUM(double, true, true); else IGS_ACCUM(double, false, true); }
    else { if (pair) IGS_ACCUM(double, true, false); else IGS_ACCUM(double, false, false); }
  } else {
    if (store) { if (pair) IGS_ACCUM(float, true, true); else IGS_ACCUM(float, false, true); }
    else { if (pair) IGS_ACCUM(float, true, false); else IGS_ACCUM(float, false, false); }
  }
#undef IGS_ACCUM
  IGS_LAUNCH_CHECK();
  return IGS_OK;
}

}  // extern "C"
