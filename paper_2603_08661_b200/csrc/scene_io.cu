// Scene-file support on sm_100a: the device half of `.igsp` loading.
//
// Replaces the quaternion renormalisation of splitkit.io_cli.read_scene
// (/root/reference/pkg/src/splitkit/io_cli.py:122-127).  The Python loader
// (paper_2603_08661_b200/scene_io.py) copies the file's column blocks to the device
// with one H2D transfer; this kernel then renormalises the rotation block in place:
//   norm = sqrt(((q0^2 + q1^2) + q2^2) + q3^2)     float64, left to right
//                                                  (np.linalg.norm(q.astype(f64), axis=1))
//   q    = float32(float64(q) / norm)              (quats / norms[:, None]).astype(float32)
// Every square of a float32 is exact in float64, and sqrt / division are correctly
// rounded on both sides, so the result is bit-identical to numpy.  A zero or non-finite
// norm sets bit 1 of *flags (the reference raises SceneFormatError).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "igs_common.cuh"

namespace igs {
namespace scene_io {

constexpr int NT = 256;

constexpr int U = 4;  // quaternions per thread, loads first

__global__ void __launch_bounds__(NT) normalize_quats_kernel(float4* __restrict__ q, long long n,
                                                              int* flags) {
  const long long base = (long long)blockIdx.x * NT * U + threadIdx.x;
  float4 v[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const long long i = base + (long long)u * NT;
    if (i < n) v[u] = q[i];
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const long long i = base + (long long)u * NT;
    if (i >= n) break;
    const double x = v[u].x, y = v[u].y, z = v[u].z, w = v[u].w;
    double s = x * x;
    s = s + y * y;
    s = s + z * z;
    s = s + w * w;
    const double norm = sqrt(s);
    if (!(norm > 0.0) || !isfinite(norm)) {
      atomicOr(flags, 1);
      continue;
    }
    q[i] = make_float4((float)(x / norm), (float)(y / norm), (float)(z / norm), (float)(w / norm));
  }
}

}  // namespace scene_io
}  // namespace igs

using namespace igs;

extern "C" {

int igs_normalize_quaternions(float* quats, int64_t n, int32_t* flags, void* stream) {
  if (n < 0 || !flags) return IGS_ERR_ARGUMENT;
  if (n > 0 && (!quats || ((uintptr_t)quats & 15))) return IGS_ERR_ARGUMENT;
  cudaStream_t s = (cudaStream_t)stream;
  IGS_CUDA_TRY(cudaMemsetAsync(flags, 0, sizeof(int32_t), s));
  if (n == 0) return IGS_OK;
  const long long blocks = (n + scene_io::NT * scene_io::U - 1) / (scene_io::NT * scene_io::U);
  scene_io::normalize_quats_kernel<<<(unsigned)blocks, scene_io::NT, 0, s>>>(
      reinterpret_cast<float4*>(quats), n, flags);
  IGS_LAUNCH_CHECK();
  return IGS_OK;
}

}  // extern "C"
