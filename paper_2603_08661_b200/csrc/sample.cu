// Score sampling on sm_100a: bilinear samples of importance maps at primitive positions.
//
// Replaces splitkit.edge_pipeline.sample_scores
// (/root/reference/pkg/src/splitkit/edge_pipeline.py:138-164), the bridge from the edge map
// to the per-primitive edge_score that selection consumes (splat2d.py:397), batched over
// views: position i samples map view[i] (or map 0).  One thread per position; the four
// taps are read-only loads through L1 (neighbouring primitives share map lines).
//
// Arithmetic (float64, separately rounded, numpy's left-to-right order):
//   inside = 0 <= x <= W-1 and 0 <= y <= H-1          (else the score is 0)
//   xc, yc = clip(x, 0, W-1), clip(y, 0, H-1);  x0, y0 = floor;  x1, y1 = min(+1, edge)
//   fx, fy = xc - x0, yc - y0
//   value = ((1-fy) * ((1-fx) v00 + fx v01)) + (fy * ((1-fx) v10 + fx v11))
// NaN positions set a device flag: numpy indexes with INT64_MIN there and the reference
// raises IndexError, which the Python wrapper re-raises.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "igs_common.cuh"

namespace igs {
namespace sample {

constexpr int NT = 256;

__global__ void __launch_bounds__(NT) sample_kernel(const double* __restrict__ maps, long long B,
                                                    long long H, long long W,
                                                    const double* __restrict__ pos,
                                                    const int32_t* __restrict__ view, long long n,
                                                    double* __restrict__ out, int* flags) {
  const long long i = (long long)blockIdx.x * NT + threadIdx.x;
  if (i >= n) return;
  const double2 xy = __ldg(reinterpret_cast<const double2*>(pos) + i);
  const double x = xy.x, y = xy.y;
  if (x != x || y != y) {
    atomicOr(flags, 1);
    out[i] = 0.0;
    return;
  }
  long long b = 0;
  if (view) {
    b = __ldg(view + i);
    if (b < 0 || b >= B) {
      atomicOr(flags, 2);
      out[i] = 0.0;
      return;
    }
  }
  const double wm = (double)(W - 1), hm = (double)(H - 1);
  const bool inside = x >= 0.0 && x <= wm && y >= 0.0 && y <= hm;
  if (!inside) {
    out[i] = 0.0;
    return;
  }
  // inside: clip is the identity (it only matters for the discarded outside branch)
  const double x0f = floor(x), y0f = floor(y);
  const long long x0 = (long long)x0f, y0 = (long long)y0f;
  const long long x1 = x0 + 1 < W - 1 ? x0 + 1 : W - 1;
  const long long y1 = y0 + 1 < H - 1 ? y0 + 1 : H - 1;
  const double fx = x - x0f, fy = y - y0f;
  const double* m = maps + b * H * W;
  const double v00 = __ldg(m + y0 * W + x0), v01 = __ldg(m + y0 * W + x1);
  const double v10 = __ldg(m + y1 * W + x0), v11 = __ldg(m + y1 * W + x1);
  const double gx = 1.0 - fx, gy = 1.0 - fy;
  const double top = (gx * v00) + (fx * v01);
  const double bot = (gx * v10) + (fx * v11);
  out[i] = (gy * top) + (fy * bot);
}

}  // namespace sample
}  // namespace igs

using namespace igs;

extern "C" {

int igs_sample_scores(const double* maps, int64_t batch, int64_t height, int64_t width,
                      const double* positions, const int32_t* view, int64_t n, double* scores,
                      int32_t* flags, void* stream) {
  if (n < 0 || batch < 1 || height < 1 || width < 1 || !flags) return IGS_ERR_ARGUMENT;
  cudaStream_t st = (cudaStream_t)stream;
  IGS_CUDA_TRY(cudaMemsetAsync(flags, 0, sizeof(int32_t), st));
  if (n == 0) return IGS_OK;
  if (!maps || !positions || !scores) return IGS_ERR_ARGUMENT;
  if (((uintptr_t)positions & 15) != 0) return IGS_ERR_ARGUMENT;
  const long long blocks = (n + sample::NT - 1) / sample::NT;
  sample::sample_kernel<<<(unsigned)blocks, sample::NT, 0, st>>>(maps, batch, height, width,
                                                                 positions, view, n, scores,
                                                                 (int*)flags);
  IGS_LAUNCH_CHECK();
  return IGS_OK;
}

}  // extern "C"
