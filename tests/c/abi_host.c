/*
 * A plain-C host program on the C ABI (include/igs_b200.h): what a non-Python integrator
 * of libigs_b200.so writes.  Test infrastructure, driven by tests/test_cabi_c.py.
 *
 *   abi_host query                       host-only calls: ABI version, status strings,
 *                                        workspace sizes, argument errors (no GPU needed)
 *   abi_host edge IN OUT B H W SIGMA_W   reads B*H*W*3 float64 views and the 25 blur weights
 *                                        (IN = views then weights, raw little-endian), runs
 *                                        igs_edge_importance on the default stream, writes the
 *                                        B*H*W float64 maps to OUT
 *
 * The GPU mode uses the CUDA runtime only for memory (cudaMalloc / cudaMemcpy), as a caller
 * that owns its buffers would; the library never allocates.
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "igs_b200.h"

/* the few CUDA runtime entry points the GPU mode needs (libcudart, C linkage) */
typedef int cudaError_t;
extern cudaError_t cudaMalloc(void** p, size_t n);
extern cudaError_t cudaFree(void* p);
extern cudaError_t cudaMemcpy(void* dst, const void* src, size_t n, int kind);
extern cudaError_t cudaDeviceSynchronize(void);
enum { H2D = 1, D2H = 2 };

static int query(void) {
  size_t n = 0;
  if (igs_abi_version() < 1) return 1;
  if (strcmp(igs_strerror(IGS_OK), "ok") != 0) return 2;
  if (igs_edge_workspace_bytes(200, 822, 1237, 0, &n) != IGS_OK || n == 0) return 3;
  if (igs_edge_workspace_bytes(-1, 8, 8, 0, &n) != IGS_ERR_ARGUMENT) return 4;
  if (igs_select_workspace_bytes(1000000, &n) != IGS_OK || n < 8000000) return 5;
  if (igs_las_workspace_bytes(1000000, &n) != IGS_OK || n == 0) return 6;
  /* host-checked argument errors return before any launch */
  if (igs_edge_importance(NULL, IGS_F64, 3, 1, 2, 2, NULL, 0, NULL, NULL, 0, NULL) !=
      IGS_ERR_ARGUMENT)
    return 7;
  printf("abi %d ok\n", igs_abi_version());
  return 0;
}

static int edge(const char* in_path, const char* out_path, long long B, long long H, long long W) {
  const size_t npx = (size_t)(B * H * W);
  double* host_in = malloc(npx * 3 * sizeof(double));
  double w25[25];
  double* host_out = malloc(npx * sizeof(double));
  FILE* f = fopen(in_path, "rb");
  if (!f || !host_in || !host_out) return 10;
  if (fread(host_in, sizeof(double), npx * 3, f) != npx * 3) return 11;
  if (fread(w25, sizeof(double), 25, f) != 25) return 12;
  fclose(f);
  size_t ws_bytes = 0;
  if (igs_edge_workspace_bytes(B, H, W, 0, &ws_bytes) != IGS_OK) return 13;
  void *d_in = NULL, *d_out = NULL, *d_ws = NULL;
  if (cudaMalloc(&d_in, npx * 3 * sizeof(double)) || cudaMalloc(&d_out, npx * sizeof(double)) ||
      cudaMalloc(&d_ws, ws_bytes))
    return 14;
  if (cudaMemcpy(d_in, host_in, npx * 3 * sizeof(double), H2D)) return 15;
  int st = igs_edge_importance(d_in, IGS_F64, 3, B, H, W, w25, 0, (double*)d_out, d_ws, ws_bytes,
                               NULL);
  if (st != IGS_OK) {
    fprintf(stderr, "igs_edge_importance: %s (%s)\n", igs_strerror(st), igs_last_cuda_error());
    return 16;
  }
  if (cudaDeviceSynchronize() || cudaMemcpy(host_out, d_out, npx * sizeof(double), D2H)) return 17;
  f = fopen(out_path, "wb");
  if (!f || fwrite(host_out, sizeof(double), npx, f) != npx) return 18;
  fclose(f);
  cudaFree(d_in);
  cudaFree(d_out);
  cudaFree(d_ws);
  free(host_in);
  free(host_out);
  printf("edge ok\n");
  return 0;
}

int main(int argc, char** argv) {
  if (argc >= 2 && strcmp(argv[1], "query") == 0) return query();
  if (argc >= 7 && strcmp(argv[1], "edge") == 0)
    return edge(argv[2], argv[3], atoll(argv[4]), atoll(argv[5]), atoll(argv[6]));
  fprintf(stderr, "usage: abi_host query | edge IN OUT B H W\n");
  return 64;
}
