// C-ABI housekeeping: status strings, CUDA error capture, device queries.
#include <cuda_runtime.h>

#include <chrono>
#include <stdio.h>

#include "igs_common.cuh"

namespace igs {

static thread_local char g_cuda_error[256] = "";

void set_cuda_error(cudaError_t e) {
  snprintf(g_cuda_error, sizeof(g_cuda_error), "%s: %s", cudaGetErrorName(e),
           cudaGetErrorString(e));
}

int sm_count() {
  static int cached = 0;
  if (!cached) {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess)
      cached = n;
  }
  return cached;
}

}  // namespace igs

extern "C" {

const char* igs_strerror(int status) {
  switch (status) {
    case IGS_OK: return "ok";
    case IGS_ERR_ARGUMENT: return "invalid argument";
    case IGS_ERR_CUDA: return "CUDA error";
    case IGS_ERR_WORKSPACE: return "workspace too small";
    case IGS_ERR_UNSUPPORTED: return "unsupported";
    default: return "unknown status";
  }
}

const char* igs_last_cuda_error(void) { return igs::g_cuda_error; }

// 2: igs_shard_boundary takes the mask (round 2); igs_las_split_packed, igs_las_split_sparse,
//    igs_wait_host_word, igs_publish_words added
int igs_abi_version(void) { return 2; }

// Wait for `stream` (the host half of a synchronous call such as las_split_batch, whose
// kernels write their summary into pinned host memory).
int igs_stream_synchronize(void* stream) {
  IGS_CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
  return IGS_OK;
}

// Copy n int64 words of device memory into pinned host memory, then (system-scope fence)
// set host[n] = 1: a host spinning on host[n] (igs_wait_host_word) reads complete words while
// the stream runs on (e.g. the sharded plan, before the split it guards has finished).
__global__ void publish_words_kernel(const int64_t* src, int64_t* host, int64_t n) {
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) host[i] = src[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    *(volatile int64_t*)(host + n) = 1;
  }
}

int igs_publish_words(const int64_t* src, int64_t* host, int64_t n, void* stream) {
  if (!src || !host || n < 0) return IGS_ERR_ARGUMENT;
  publish_words_kernel<<<1, 128, 0, (cudaStream_t)stream>>>(src, host, n);
  IGS_LAUNCH_CHECK();
  return IGS_OK;
}

// Spin until the host word (pinned memory a kernel writes) differs from `sentinel`; after
// `timeout_ns` fall back to synchronising `stream` (so an asynchronous kernel fault surfaces
// as its CUDA error) and fail with IGS_ERR_CUDA if the word is still unwritten.
int igs_wait_host_word(const int64_t* word, int64_t sentinel, int64_t timeout_ns, void* stream) {
  if (!word) return IGS_ERR_ARGUMENT;
  const volatile int64_t* w = word;
  if (*w != sentinel) return IGS_OK;
  const auto t0 = std::chrono::steady_clock::now();
  for (unsigned spin = 1;; ++spin) {
    if (*w != sentinel) return IGS_OK;
    if ((spin & 1023u) == 0 &&
        std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0)
                .count() > timeout_ns)
      break;
  }
  IGS_CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
  return *w != sentinel ? IGS_OK : IGS_ERR_CUDA;
}

// L2 set-aside for persisting (evict_last) lines on the current device; returns the granted
// size in *granted (nullable).  Device-wide setting (cudaLimitPersistingL2CacheSize).
int igs_l2_set_aside(size_t bytes, size_t* granted) {
  int dev = 0;
  IGS_CUDA_TRY(cudaGetDevice(&dev));
  int maxp = 0;
  IGS_CUDA_TRY(cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev));
  if (bytes > (size_t)maxp) bytes = (size_t)maxp;
  IGS_CUDA_TRY(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, bytes));
  if (granted) IGS_CUDA_TRY(cudaDeviceGetLimit(granted, cudaLimitPersistingL2CacheSize));
  return IGS_OK;
}


// The tail of a sharded densify event in one call (include/igs_b200.h IgsShardEventArgs).
int igs_shard_event(const IgsShardEventArgs* a) {
  if (!a || !a->host_plan || a->plan_words < 0) return IGS_ERR_ARGUMENT;
  int rc = igs_shard_finalize(a->records, a->world, a->rank, a->record_cap, a->n_global, a->gidx,
                              a->n, a->mask, a->plan, a->shard_workspace,
                              a->shard_workspace_bytes, a->stream);
  if (rc) return rc;
  *(volatile int64_t*)(a->host_plan + a->plan_words) = -1;  // the previous read is complete
  rc = igs_publish_words(a->plan, a->host_plan, a->plan_words, a->stream);
  if (rc || !a->split) return rc;
  rc = igs_las_split_guarded(a->positions, a->log_scales, a->rotations, a->opacity_logits,
                             a->sh_or_colors, a->sh_floats, a->dims, a->n, a->reserved_rows,
                             a->mask, a->alpha, a->log_alpha, a->log_gamma, a->beta, a->plan,
                             a->las_workspace, a->las_workspace_bytes, a->stream);
  if (rc) return rc;
  return igs_shard_child_index(a->gidx, a->n, a->plan, a->stream);
}

}  // extern "C"
