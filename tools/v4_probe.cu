// Probe: 256-bit global stores with an L2 cache hint on sm_100a, all lanes and divergent lanes.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void st4(double* a, double v0, double v1, double v2, double v3) {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("st.global.L2::cache_hint.v4.f64 [%0], {%1, %2, %3, %4}, %5;" ::"l"(a), "d"(v0),
               "d"(v1), "d"(v2), "d"(v3), "l"(pol) : "memory");
}
__global__ void k(double* a, const int* sel) {
  const int t = threadIdx.x;
  double v0 = t * 4 + 1, v1 = v0 + 1, v2 = v0 + 2, v3 = v0 + 3;
  if (sel[t]) st4(a + t * 4, v0, v1, v2, v3);
}
int main() {
  const int N = 256;
  double* d; int* s; cudaMalloc(&d, N * 32); cudaMalloc(&s, N * 4);
  int hs[N]; for (int i = 0; i < N; ++i) hs[i] = (i * 7 + i / 3) % 3 == 0;
  cudaMemcpy(s, hs, sizeof(hs), cudaMemcpyHostToDevice);
  cudaMemset(d, 0, N * 32);
  k<<<1, N>>>(d, s); cudaDeviceSynchronize();
  double h[N * 4]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < N * 4; ++i) {
    double want = hs[i / 4] ? i + 1 : 0;
    if (h[i] != want) { if (bad < 8) printf("bad %d got %g want %g\n", i, h[i], want); ++bad; }
  }
  printf("divergent v4 store probe: %d bad of %d (%s)\n", bad, N * 4, cudaGetErrorString(cudaGetLastError()));
}
