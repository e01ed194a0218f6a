/*
 * igs_b200.h -- C ABI of the B200 (sm_100a) densification hot path of ImprovedGS+.
 *
 * One shared library, libigs_b200.so, built from every .cu file in paper_2603_08661_b200/csrc/.
 * Every entry point takes plain device pointers, sizes and a cudaStream_t
 * (passed as void*), returns an igs_status (0 == IGS_OK) and never allocates:
 * the caller owns every buffer, including the workspace, whose size the
 * matching *_workspace_bytes() query reports.  All launches are asynchronous
 * on `stream`; the functions that must report device-detected conditions
 * write them to caller-provided DEVICE counters (no hidden host syncs).
 *
 * The reference (`splitkit`, /root/reference/pkg/src/splitkit) is pure
 * Python; there is no reference C ABI.  Each entry point names the reference
 * function it replaces (file:line); the Python drop-in in
 * paper_2603_08661_b200/ keeps the reference names, arguments and exceptions
 * and binds these symbols through ctypes.
 */
#ifndef IGS_B200_H
#define IGS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------ */
enum igs_status {
  IGS_OK = 0,
  IGS_ERR_ARGUMENT = 1,     /* bad shape / size / pointer / flag combination   */
  IGS_ERR_CUDA = 2,         /* a CUDA runtime call failed (see igs_last_cuda_error) */
  IGS_ERR_WORKSPACE = 3,    /* workspace smaller than *_workspace_bytes()      */
  IGS_ERR_UNSUPPORTED = 4   /* valid request this build does not implement      */
};

enum igs_dtype { IGS_F32 = 0, IGS_F64 = 1 };

/* igs_edge_importance flags (io_cli.py:315-323 --no-nms / --no-median) */
enum igs_edge_flags { IGS_EDGE_NO_NMS = 1, IGS_EDGE_NO_MEDIAN = 2 };

/* selection policy (schedule.py:94, densify_controller.py:72-77) */
enum igs_policy { IGS_POLICY_PRODUCT = 0, IGS_POLICY_EDGE = 1, IGS_POLICY_GRAD = 2 };

/* LAS pre-pass flags (core.py:43-46, core.py:27-28) */
enum igs_las_flags {
  IGS_LAS_BAD_QUAT = 1,     /* zero or non-finite quaternion norm -> ValueError */
  IGS_LAS_BAD_OPACITY = 2,  /* sigmoid(o)*beta outside (0,1)    -> ValueError   */
  IGS_LAS_RENORM = 4        /* some |norm-1| > 1e-4: renormalise the whole batch */
};

const char* igs_strerror(int status);
const char* igs_last_cuda_error(void);
/* 2 since round 2 (igs_shard_boundary takes the mask; the packed LAS call and the pinned-word
 * helpers were added). */
int igs_abi_version(void);
/* cudaStreamSynchronize(stream): the host half of a synchronous call whose kernels write
 * their result into pinned host memory (e.g. igs_las_split's summary). */
int igs_stream_synchronize(void* stream);
/* Spin until *word (pinned host memory a kernel writes, e.g. igs_las_split's summary[1]) is no
 * longer `sentinel`.  After timeout_ns the stream is synchronised instead (an asynchronous
 * kernel fault returns its CUDA error); IGS_ERR_CUDA if the word is still unwritten. */
int igs_wait_host_word(const int64_t* word, int64_t sentinel, int64_t timeout_ns, void* stream);
/* Stream-ordered copy of n int64 words from device memory into pinned host memory, then
 * host[n] = 1 (after a system-scope fence): the host spins on host[n] instead of a stream
 * synchronise (the sharded step reads its plan while the guarded split still runs). */
int igs_publish_words(const int64_t* src, int64_t* host, int64_t n, void* stream);

/* L2 set-aside for persisting (evict_last) lines: the fused edge kernel keeps the in-flight
 * views' thinned maps evict_last.  Device-wide (cudaLimitPersistingL2CacheSize), clamped to
 * the device maximum; *granted (nullable) receives the size in effect. */
int igs_l2_set_aside(size_t bytes, size_t* granted);

/* ---- edge-importance map (edge_pipeline.py) ----------------------------- */

/* Workspace for igs_edge_importance / igs_median_normalize over `batch` views of height x width. */
int igs_edge_workspace_bytes(int64_t batch, int64_t height, int64_t width, int flags,
                             size_t* bytes);

/* importance_pipeline (edge_pipeline.py:128-135), batched over views with per-view medians.
 * image: (batch, height, width, channels) contiguous, channels 3 (RGB -> Rec.601 gray,
 * :42-49) or 1 (already gray, not clipped, :134), dtype IGS_F32/IGS_F64.
 * blur_w25: the 5x5 weights of blur_kernel_5x5(sigma) (:52-59), host memory, row-major.
 * out: (batch, height, width) float64.  height, width >= 3.  One fused persistent launch:
 * gray -> blur -> Sobel -> NMS (-> median histogram -> radix select -> normalise). */
int igs_edge_importance(const void* image, int in_dtype, int channels,
                        int64_t batch, int64_t height, int64_t width,
                        const double* blur_w25, int flags, double* out,
                        void* workspace, size_t workspace_bytes, void* stream);

/* Stage entry points, one kernel each (edge_pipeline.py:42-125); batched over views. */
int igs_to_grayscale(const void* image, int in_dtype, int64_t batch, int64_t height,
                     int64_t width, double* gray, void* stream);                 /* :42-49  */
int igs_gaussian_blur_5x5(const double* gray, int64_t batch, int64_t height, int64_t width,
                          const double* blur_w25, double* out, void* stream);    /* :62-67  */
int igs_sobel_gradients(const double* gray, int64_t batch, int64_t height, int64_t width,
                        double* magnitude, double* orientation, void* stream);   /* :70-83  */
int igs_nms_thin(const double* magnitude, const double* orientation, int64_t batch,
                 int64_t height, int64_t width, double* out, void* stream);      /* :86-114 */
/* median_normalize (:117-125) of `batch` independent arrays of n values (in may == out).
 * medians (device, nullable): receives each array's positive median (1.0 if none). */
int igs_median_normalize(const double* in, int64_t batch, int64_t n, double* out,
                         double* medians, void* workspace, size_t workspace_bytes,
                         void* stream);

/* sample_scores (edge_pipeline.py:138-164): bilinear samples of importance maps at
 * positions (n, 2) float64 (x, y) -- 16-byte aligned -- of map view[i] (view nullable: map 0)
 * of maps (batch, height, width) float64; outside [0, W-1] x [0, H-1] -> 0.  flags (device
 * int32) receives bit 1 for a NaN position (the reference raises IndexError), bit 2 for a
 * view index outside [0, batch). */
int igs_sample_scores(const double* maps, int64_t batch, int64_t height, int64_t width,
                      const double* positions, const int32_t* view, int64_t n, double* scores,
                      int32_t* flags, void* stream);

/* Debug: record {start_ns, end_ns, kind, view, index, smid} (32 bytes) per task of later
 * igs_edge_importance launches into the device buffer buf (NULL disables); *written (nullable)
 * receives the number of records the previous launches produced. */
int igs_debug_edge_trace(void* buf, int64_t capacity, int64_t* written);

/* Debug: per-phase nanoseconds of the fused kernel's band sub-steps, summed over blocks
 * (gray, blur, Sobel, NMS decide, NMS finish), in a library built with -DIGS_PHASE_PROF;
 * IGS_ERR_UNSUPPORTED otherwise.  reset != 0 clears the counters after reading. */
int igs_debug_edge_phases(uint64_t* out8, int reset);

/* ---- budgeted candidate selection (densify_controller.py:66-106) -------- */

int igs_select_workspace_bytes(int64_t n, size_t* bytes);

/* grad_norm = grad_sum / accum_count (0 if accum_count == 0, :40-43).  Eligible: all
 * (warmup != 0) or grad_norm > grad_threshold.  take = min(#eligible, take_cap) where the
 * host computes take_cap = min(headroom, max(ceil(growth_cap*count - 1e-9), 0)) (:99-100).
 * mask[i] = 1 for the `take` eligible entries ranked first by (score desc, index asc),
 * i.e. np.argsort(-score, kind="stable") (:104).  counts (device int64[2]) receives
 * {#eligible, take}. */
int igs_select_candidates(const double* grad_sum, int64_t accum_count, const double* edge_score,
                          int64_t n, double grad_threshold, int warmup, int policy,
                          int64_t take_cap, uint8_t* mask, int64_t* counts,
                          void* workspace, size_t workspace_bytes, void* stream);

/* Trainer-side statistics (splat2d.py:393-394 + densify_controller.py:54-63): grad_sum[i] +=
 * hypot(grads[2i], grads[2i+1]) in float64 (glibc hypot, as np.hypot); grads (n, 2) of dtype
 * IGS_F32 / IGS_F64.  The caller increments the accumulation count.  dtype | IGS_ACCUM_STORE:
 * the first accumulation after a reset, grad_sum[i] = 0.0 + hypot(...) without reading
 * grad_sum (the reset's zeros are never written). */
#define IGS_ACCUM_STORE 0x100
int igs_accumulate_grad_norms(double* grad_sum, const void* grads, int dtype, int64_t n,
                              void* stream);

/* ---- sharded densify step (multi-GPU) ------------------- *
 * select_candidates + las_split_batch of densify_step (densify_controller.py:80-106,
 * 125-147) over a cloud sharded across ranks, bit-identical to the single-process step on the
 * reference's global array.  Each row carries its global index gidx (int64; contiguous ranges
 * before the first split, children appended in the reference's order afterwards); ties break
 * by gidx.  Per event, all stream-ordered, two collectives, one host read at the end:
 *   igs_shard_keys        -> all-reduce(sum) hist (int32[IGS_SHARD_HIST_LEN]: 65536 bins of a
 *                            monotone 16-bit digit of the score key, then the eligible count)
 *   igs_shard_boundary    resolve take / boundary digit / need, compact this rank's
 *                            boundary-bucket entries into its record, and write the mask of
 *                            its rows below the boundary bucket
 *                         -> all-gather records (int64[4 + 2 record_cap] per rank)
 *   igs_shard_finalize    threshold (key, gidx) by radix select over every record; the plan
 *                            (int64[16]); completes this rank's mask (the boundary rows taken;
 *                            cleared when nothing is selected or the records overflowed)
 *   igs_las_split_guarded the split of this shard, guarded by plan[0..1]
 *   igs_shard_child_index gidx of this rank's appended children
 * plan words: [0] this rank's split count if the split may go ahead else 0, [1] batch LAS
 * flags, [2] status (0 ok, 1 nothing selected, 2 boundary bucket larger than record_cap:
 * nothing split, re-run boundary/gather/finalize with record_cap >= plan[7]), [3] global
 * split count, [4] global eligible count, [5] global index of this rank's first child,
 * [6] this rank's split count, [7] largest boundary-bucket count over the ranks, [8] threshold
 * key, [9] threshold global index, [10] boundary digit, [11] boundary entries to take.  With
 * more than 32768 boundary entries over all ranks igs_shard_finalize sets status 2 as well
 * and the caller selects from the gathered records itself, then calls igs_shard_mask. */
#define IGS_SHARD_HIST_LEN 65537
int igs_shard_workspace_bytes(int64_t n, size_t* bytes);
int igs_shard_keys(const double* grad_sum, int64_t accum_count, const double* edge_score,
                   int64_t n, double grad_threshold, int warmup, int policy, int32_t* hist,
                   void* workspace, size_t workspace_bytes, void* stream);
int igs_shard_boundary(const int32_t* global_hist, int64_t take_cap, const int64_t* gidx,
                       const float* rotations, const float* opacity_logits, float beta,
                       int64_t n, int64_t record_cap, int64_t* record, uint8_t* mask,
                       void* workspace, size_t workspace_bytes, void* stream);
int igs_shard_finalize(const int64_t* records, int world, int rank, int64_t record_cap,
                       int64_t n_global, const int64_t* gidx, int64_t n, uint8_t* mask,
                       int64_t* plan, void* workspace, size_t workspace_bytes, void* stream);
int igs_shard_child_index(int64_t* gidx, int64_t count, const int64_t* plan, void* stream);
/* The rest of an event in one call (igs_shard_finalize, then igs_publish_words of the plan into
 * the pinned host_plan[0..plan_words) with host_plan[plan_words] = -1 beforehand and 1 last,
 * then -- when `split` -- igs_las_split_guarded of the shard under the plan and
 * igs_shard_child_index): the same launches in the same stream order as the four calls, one
 * host->library transition instead of four. */
typedef struct IgsShardEventArgs {
  const int64_t* records;
  int32_t world, rank;
  int64_t record_cap, n_global;
  int64_t* gidx;
  int64_t n;
  uint8_t* mask;
  int64_t* plan;
  void* shard_workspace;
  size_t shard_workspace_bytes;
  int64_t* host_plan;
  int64_t plan_words;
  int32_t split, dims;
  float* positions;
  float* log_scales;
  float* rotations;
  float* opacity_logits;
  float* sh_or_colors;
  int64_t sh_floats, reserved_rows;
  float alpha, log_alpha, log_gamma, beta;
  void* las_workspace;
  size_t las_workspace_bytes;
  void* stream;
} IgsShardEventArgs;
int igs_shard_event(const IgsShardEventArgs* args);
/* This rank's mask for a plan computed outside igs_shard_finalize (the path for boundary
 * buckets of more than 32768 entries over all ranks, e.g. every score equal). */
int igs_shard_mask(const int64_t* gidx, int64_t n, const int64_t* plan, uint8_t* mask,
                   void* workspace, size_t workspace_bytes, void* stream);

/* ---- Long-Axis-Split (las_split.py:146-179) ----------------------------- */

int igs_las_workspace_bytes(int64_t count, size_t* bytes);

/* Pre-pass over the mask (1 byte per Gaussian): per-block split counts and their exclusive
 * scan (slot ranks), plus the flags of enum igs_las_flags over the MASKED parents
 * (rotations may be NULL: a 2-D scene, no quaternion checks).
 * summary (device int64[2]) receives {n_split, flags}.  Nothing in the scene is written. */
int igs_las_prepare(const uint8_t* mask, const float* rotations, const float* opacity_logits,
                    int64_t count, float beta, void* workspace, size_t workspace_bytes,
                    int64_t* summary, void* stream);

/* Split pass (run after igs_las_prepare on the same workspace and a host check of the
 * summary): parent i <- +offset child (positions, log_scales, opacity_logits written in
 * place); slot count + rank(i) <- -offset child with the parent's rotation and SH cloned.
 * Columns are SoA float32 with capacity rows: positions (cap,3), log_scales (cap,3),
 * rotations (cap,4), opacity_logits (cap,), sh (cap, sh_floats).  renormalize != 0 applies
 * the batch-global quaternion renormalisation of core.py:45-46. */
int igs_las_apply(float* positions, float* log_scales, float* rotations, float* opacity_logits,
                  float* sh, int64_t sh_floats, int64_t count, int64_t capacity,
                  const uint8_t* mask, float alpha, float log_alpha, float log_gamma,
                  float beta, int renormalize, void* workspace, size_t workspace_bytes,
                  void* stream);

/* The whole split in ONE cooperative launch, no host round trip between the passes: the
 * pre-pass of every tile, a grid barrier, then the apply pass guarded on the device by the
 * pre-pass totals.  If count + n_split > capacity or a domain flag (BAD_QUAT / BAD_OPACITY) is
 * set, nothing in the scene is written; the caller reads summary {n_split, flags} afterwards
 * and raises (BudgetError / ValueError) or adds n_split to its count.  Renormalisation follows
 * the RENORM flag.  summary may be device memory or pinned host memory (written directly).
 * Replaces las_split.py:158-179 (the reference's las_split_batch) in one call. */
int igs_las_split(float* positions, float* log_scales, float* rotations, float* opacity_logits,
                  float* sh, int64_t sh_floats, int64_t count, int64_t capacity,
                  const uint8_t* mask, float alpha, float log_alpha, float log_gamma, float beta,
                  void* workspace, size_t workspace_bytes, int64_t* summary, void* stream);

/* igs_las_split (sparse = 0) / igs_las_split_sparse (sparse != 0) with the arguments in one
 * struct: for bindings whose per-argument call cost matters at small sizes (one pointer
 * instead of 17 converted arguments; the Python drop-in keeps one per scene and updates
 * count / capacity / mask / summary per call). */
typedef struct IgsLasSplitArgs {
  float* positions;
  float* log_scales;
  float* rotations;
  float* opacity_logits;
  float* sh;
  int64_t sh_floats;
  int64_t count;
  int64_t capacity;
  const uint8_t* mask;
  float alpha, log_alpha, log_gamma, beta;
  void* workspace;
  size_t workspace_bytes;
  int64_t* summary;
  void* stream;
  int32_t sparse;
  int32_t reserved;
} IgsLasSplitArgs;
int igs_las_split_packed(const IgsLasSplitArgs* args);

/* igs_las_split for sparse masks (e.g. densify_step's top-5% selection): the pre-pass also
 * lists the masked parents in slot order and the apply pass walks that list (one gather per
 * parent) instead of every tile of the mask.  Same results, same guard. */
int igs_las_split_sparse(float* positions, float* log_scales, float* rotations,
                         float* opacity_logits, float* sh, int64_t sh_floats, int64_t count,
                         int64_t capacity, const uint8_t* mask, float alpha, float log_alpha,
                         float log_gamma, float beta, void* workspace, size_t workspace_bytes,
                         int64_t* summary, void* stream);

/* 2-D Long-Axis-Split (las_split.py:182-197), after igs_las_prepare with rotations = NULL
 * (no quaternion checks).  Columns: positions (cap,2), log_scales (cap,2), thetas (cap,),
 * opacity_logits (cap,), colors (cap,3), float32; the same slot rule as igs_las_apply. */
int igs_las2d_apply(float* positions, float* log_scales, float* thetas, float* opacity_logits,
                    float* colors, int64_t count, int64_t capacity, const uint8_t* mask,
                    float alpha, float log_alpha, float log_gamma, float beta, void* workspace,
                    size_t workspace_bytes, void* stream);

/* igs_las_split for a 2-D scene (las_split.py:182-197): same guard (BAD_OPACITY only). */
int igs_las2d_split(float* positions, float* log_scales, float* thetas, float* opacity_logits,
                    float* colors, int64_t count, int64_t capacity, const uint8_t* mask,
                    float alpha, float log_alpha, float log_gamma, float beta, void* workspace,
                    size_t workspace_bytes, int64_t* summary, void* stream);

/* The split of one shard under the sharded step's plan: the pre-pass for this shard's slot
 * offsets, then the apply pass guarded by the device words guard = {n_split or 0, batch
 * flags} against reserved_rows.  dims 3: rotations (cap,4), sh_or_colors = sh (cap,
 * sh_floats); dims 2: rotations = thetas (cap,), sh_or_colors = colors (cap,3). */
int igs_las_split_guarded(float* positions, float* log_scales, float* rotations,
                          float* opacity_logits, float* sh_or_colors, int64_t sh_floats,
                          int dims, int64_t count, int64_t reserved_rows, const uint8_t* mask,
                          float alpha, float log_alpha, float log_gamma, float beta,
                          const int64_t* guard, void* workspace, size_t workspace_bytes,
                          void* stream);

/* ---- scene files (io_cli.py:83-134) ------------------------------------- */

/* read_scene's quaternion renormalisation (io_cli.py:122-127), in place on n float32
 * quaternions (16-byte aligned): q = float32(float64(q) / ||float64(q)||), the norm summed
 * left to right (np.linalg.norm).  flags (device int32) receives bit 1 for a zero or
 * non-finite norm (SceneFormatError). */
int igs_normalize_quaternions(float* quats, int64_t n, int32_t* flags, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* IGS_B200_H */
