// Edge-importance map on sm_100a: one persistent, task-queued launch per batch of views.
//
// Replaces splitkit.edge_pipeline.importance_pipeline and its stages
// (/root/reference/pkg/src/splitkit/edge_pipeline.py:42-135).
//
// Task kinds (one persistent cooperative grid, 256-thread blocks):
//   E(v,t)  fused band: gray -> 5x5 blur -> Sobel -> direction bin -> NMS over a
//           band of <= 124 columns x <= 128 rows, walked top to bottom in 16-row
//           sub-steps with the context rows kept in shared memory (see run_band);
//           writes the thinned map and merges a per-view histogram of the
//           positive survivors.  The last E task of a view locates the median
//           histogram bin(s).                                 (:42-114, :123)
//   C(v,c)  collect: gathers the values falling in the median bin(s) into a
//           candidate buffer plus a level-2 histogram.  The last C task of a view
//           selects the exact order statistic(s) -> median m (np.median: (a+b)/2
//           for an even count).                                          (:124)
//   A(v,c)  apply: out = min(v / (2 m), 1) in place.                     (:125)
// Scheduling is dependency driven (claim_task): A work of views whose median is
// published first, then C work of views whose bins are published, else the next
// E band -- at most `ahead` views past the A front, so only a few views' thinned
// maps are live.  Those are stored with an L2 evict_last policy (the input
// streams with evict_first), so E, C and A meet in L2 and the final map is
// written back to HBM once.  Work is claimed only when ready: no task waits.
//
// Arithmetic: float64 in scipy's order (see oracle/edge.py): taps summed in
// row-major order from 0.0 with separately rounded multiply and add; glibc's
// hypot (exact, IEEE division) for every stored magnitude; the NMS compares
// ordered by |g|^2 keys with an exact-hypot fallback (see band_nms); the NMS direction
// bin from exact comparisons against tan(pi/8) with a fallback to numpy's
// floor((mod(atan2)+pi/8)/(pi/4)) within 1e-12 rad of a boundary.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <type_traits>

#include "igs_common.cuh"

namespace igs {
namespace edge {

constexpr int NT = 256;                      // threads per block
constexpr int NWARP = NT / 32;
#ifndef IGS_SR
#define IGS_SR 16
#endif
constexpr int SR = IGS_SR;                   // output rows per band sub-step
constexpr int SH = SR / 2;                   // rows per blur / Sobel strip (two strips)
#ifndef IGS_MINB
#define IGS_MINB 3
#endif
constexpr int TWM = 124;                     // max output columns per band
constexpr int BAND_H = 256;                  // max rows per band (tuning override)
constexpr int BAND_H_DEFAULT = 112;          // rows per band (7 sub-steps; measured best of
                                             // 80-208 for 200 x 822-row views)
constexpr int GWP = TWM + 8, BWP = 128, MWP = 128;  // row pitches (cells); the blur /
                                                    // Sobel lanes cover 128 columns
constexpr int GR = SR + 8, BR = SR + 4, QR = SR + 2;        // rows per sub-step + context
static_assert(TWM * BAND_H < 65536, "16-bit shared histogram counters per band");
static_assert(TWM + 4 <= 128 && 2 * SH == SR && SR <= 16, "blur / Sobel: 128 columns x 2 strips");
static_assert(TWM + 8 <= 132, "gray: 4 x 32 lanes + 4 columns");

constexpr int NB = 4096;                     // level-1 median histogram: 64 bins per octave
constexpr int HIST_SHIFT = 46;               // bin = (bits >> 46) - HIST_BASE (18 top bits)
constexpr int HIST_BASE = 963 << 6;          // bins cover [2^-60, 2^4); outside -> end bins
constexpr int NBR = 2048;                    // radix-select digit bins (11 bits)
constexpr int SUB_SHIFT = 34;                // level-2 bin = bits 45..34 inside a level-1 bin
constexpr int SLOTS = 8;                     // candidates kept per level-2 bin
constexpr int NB2 = 4096;                    // level-2 histogram: bits 47..36 inside a bin
constexpr int CHUNK = 16384;                 // values per collect/apply task (< 65536)
constexpr int RING = 16;                     // candidate buffers / level-2 histograms in flight
constexpr int SEL_CAP = GR * GWP + BR * BWP;  // doubles of smem the select may use

enum Mode { MODE_FUSED = 0, MODE_MEDIAN_ONLY = 1 };

struct ViewCtl {            // per-view control block, zeroed before launch
  unsigned tiles_done;      // E tasks finished
  unsigned binfound;        // 1 once the median bins are known
  unsigned collect_done;    // C tasks finished
  unsigned select_done;     // 1 once denom is published
  unsigned cnt1, cnt2;      // candidate append counters (front / back)
  int b1, b2;               // level-1 bins of ranks k1, k2
  unsigned long long r1, r2;// ranks within those bins
  unsigned long long npos;  // positive count
  double denom;             // 2 * median
  double median;
  unsigned c_claim, a_claim;// C / A chunks handed out
  unsigned nsurv;           // fused mode: positive survivors appended by the E tasks
  unsigned tca;             // C / A tasks of this view (fused: survivor chunks)
  unsigned a_done;          // A tasks finished: the view's ring slot is free once a_done == tca
  unsigned pad[9];
};
static_assert(sizeof(ViewCtl) == 128, "one ViewCtl per 128-byte line");

struct Params {
  const void* img;          // (B,H,W,C) input (fused) or (B,n) values (median-only)
  int in_f64;
  int channels;             // 3 or 1
  int mode;
  int nms;                  // 0: keep all magnitudes (--no-nms)
  int median;               // 0: no normalisation (--no-median)
  int sym;                  // blur weights dihedrally symmetric -> 6 unique values
  int skip;                 // some taps have |w| <= DBL_EPSILON (NI_Correlate skips them)
  unsigned keep_mask;       // bit t: tap t kept
  long long B, H, W;        // fused: image dims; median-only: H = 1, W = n
  long long npx;            // H * W
  double w25[25];
  double w6[3][3];          // w6[|di|][|dj|] for the symmetric case
  double* out;              // (B, npx) float64
  double* medians;          // optional (B,) output of the medians
  // scheduling
  int tw, ncols, band_h, TE, TC, TA;
  int chunk;                // fused mode: survivor entries per C / A task (<= CHUNK)
  int ahead;                // E may run at most `ahead` views past the A front (< RING)
  double kgray[3];          // Rec.601 weights (edge_pipeline.py:22), in the constant bank
  double ktan, ktol;        // tan(pi/8) and the 1e-12 relative margin of the direction bin
  // workspace
  unsigned* sched;          // [1] C front view, [2] A front view, [4..5] next E task (u64)
  ViewCtl* ctl;
  unsigned* hist;           // (B, NB)
  unsigned* hist2;          // (RING, 2, NB2)
  double* slots;            // (RING, 2, NB2, SLOTS) candidates bucketed by level-2 bin
  double* cand;             // (RING, slot): fused mode: survivor values [0, npx), survivor
                            // indices (u32) [npx, 1.5 npx), candidate lists [2 npx, 3 npx);
                            // median-only mode: candidate lists [0, npx)
  long long slot;           // doubles per ring slot
};

// Ring slot of view v (3 * npx_e doubles, npx_e = npx rounded up to even).  Fused mode:
//   [0, npx_e)               survivor-list values (one column-ordered segment per band row)
//   [npx_e, 2 npx_e)         the collect pass's two candidate lists
//   from 2 npx_e             survivor-list pixel indices (u32)
// Median-only mode: the candidate lists at [0, npx).
__device__ __forceinline__ double* ring_slot(const Params& p, int v) {
  return p.cand + (long long)(v % RING) * p.slot;
}
__device__ __forceinline__ double* cand_lists(const Params& p, int v) {
  return ring_slot(p, v) + (p.mode == MODE_FUSED ? p.slot / 3 : 0);
}
__device__ __forceinline__ unsigned* surv_idx(const Params& p, int v) {
  return reinterpret_cast<unsigned*>(ring_slot(p, v) + 2 * (p.slot / 3));
}


struct __align__(16) Smem {
  double g[GR * GWP];       // gray rows of a band sub-step; C/A stream buffers, select scratch
  double b[BR * BWP];       // blurred rows (contiguous with g)
  unsigned q[(QR + 1) * MWP];  // Sobel cells: (|grad|^2 key << 2) | direction bin; one pad
                               // row: the NMS neighbour reads of the unused columns past the
                               // band stay inside the array
  unsigned short list[SR * TWM];  // compacted NMS survivors / undecided pixels of a sub-step
  unsigned list_n[2];       // list lengths (double-buffered by sub-step parity)
  unsigned rowl[SR];        // median mode: first s.list entry of each sub-step row
  unsigned rowg[SR];        // median mode: its position in the view's survivor list
  unsigned hist[NB / 2];    // level-1 counts packed two 16-bit bins per word; radix scratch
  unsigned warp_sums[32];
  int task_kind, task_view, task_idx, flag;
  int ivals[4];
  int scratch[4];
  unsigned long long mbar[4];  // bulk-copy barriers of the C / A streams (NBUF), initialised once
  unsigned mbar_seq;           // bulk-copy pieces issued by this CTA so far (barrier phases)
  int pend_valid, pend_view, pend_idx;  // a claimed band deferred until its ring slot is free
  unsigned long long u64[2];
};

// ---- L2 cache policies (input streamed once: evict_first; thinned map: evict_last) ----
__device__ __forceinline__ unsigned long long policy_evict_first() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ unsigned long long policy_evict_last() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double ld_hint(const double* a, unsigned long long pol) {
  double v;
  asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_hint(const float* a, unsigned long long pol) {
  float v;
  asm("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(a), "l"(pol));
  return (double)v;
}
__device__ __forceinline__ void st_hint(double* a, double v, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(a), "d"(v), "l"(pol) : "memory");
}
// predicated form: no divergent branch (BSSY/BSYNC) around the store
__device__ __forceinline__ void st_hint_if(bool pred, double* a, double v, unsigned long long pol) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %3, 0;\n\t"
               "@p st.global.L2::cache_hint.f64 [%0], %1, %2;\n\t}" ::"l"(a), "d"(v), "l"(pol),
               "r"((int)pred) : "memory");
}
__device__ __forceinline__ double ld_cg_hint(const double* a, unsigned long long pol) {
  double v;
  asm volatile("ld.global.cg.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
  return v;
}

// ---- TMA bulk copies (cp.async.bulk global -> shared, completion on an mbarrier) ----
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes,
                                          unsigned long long* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  asm volatile(
      "{\n .reg .pred P;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      " @!P bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// generic-proxy writes of other CTAs (survivor lists, acquired through the view's control
// block) -> async-proxy reads (bulk copies from global memory)
__device__ __forceinline__ void fence_proxy_async_all() {
  asm volatile("fence.proxy.async;" ::: "memory");
}

__device__ __forceinline__ double2 ld_cg2(const double* a) {
  double2 r;
  asm volatile("ld.global.cg.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(a));
  return r;
}

__device__ __forceinline__ int clamp_i(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }
__device__ __forceinline__ long long clampi(long long v, long long lo, long long hi) {
  return v < lo ? lo : (v > hi ? hi : v);
}


__device__ __forceinline__ int hist_bin(double v) {
  long long hb = (long long)((unsigned long long)__double_as_longlong(v) >> HIST_SHIFT) - HIST_BASE;
  return hb < 0 ? 0 : (hb >= NB ? NB - 1 : (int)hb);
}

// Shared-memory level-1 histogram: two 16-bit counters per word (a task adds < 65536).
__device__ __forceinline__ void hist_add(Smem& s, int b) {
  atomicAdd(&s.hist[b >> 1], 1u << ((b & 1) << 4));
}

// ---------------------------------------------------------------- E: fused band
// An E task owns a band of the view: output columns [x0, x0 + xw) (xw <= TWM) and rows
// [ya, yb).  It walks the band top to bottom in sub-steps of n <= SR output rows; shared
// memory holds each stage's rows for the current sub-step plus the context rows the next
// one needs (shifted down between sub-steps), so every row is computed once per band:
//   gray    rows [Y-4, Y+4+n)   s.g  (row 0 = Y-4;  columns x0-4 .., clamped coordinates)
//   blur    rows [Y-2, Y+2+n)   s.b  (row 0 = Y-2;  columns x0-2 ..)
//   Sobel   rows [Y-1, Y+1+n)   s.q  (row 0 = Y-1;  columns x0-1 ..: packed |g|^2 key + bin)
//   NMS     rows [Y,   Y+n)     decide from the keys; survivors and undecided pixels are
//                               compacted into s.list and finished by all threads (exact
//                               glibc hypot, map store, median histogram)
// Hot loops run over full 128-lane column sets without per-cell bounds tests: columns past
// the band compute harmless values that nothing reads.
//
// Exactness.  NMS compares glibc hypot values.  A cell's key is the top 30 bits of the IEEE
// pattern of |g|^2 = fma(gx, gx, gy*gy); two keys more than one unit apart order the
// magnitudes with a margin of ~2^-19 relative (the rounding of |g|^2 and the <= 1 ulp error
// of hypot are below 2^-50).  Keys within one unit, exact-zero ties, tiny or non-finite
// gradients (KEY_EXACT) fall back to the exact hypot of the cells involved, recomputed from
// the blurred rows.  Surviving pixels always store the exact glibc hypot value.

constexpr unsigned KEY_EXACT = 0x3fffffffu;  // key field of a cell whose order needs hypot

// Packed Sobel cell: (key << 2) | direction bin.  The key is the high word of |g|^2 >> 2 when
// 2^-960 <= |g|^2 < 2^1000 (range test on the integer high word), 0 for an exactly zero
// gradient, KEY_EXACT otherwise (tiny, huge or NaN: order by the exact hypot).
__device__ __forceinline__ unsigned pack_cell(double gx, double gy, int bin) {
  const double q = fma(gx, gx, gy * gy);
  const unsigned hi = (unsigned)__double2hiint(q);
  unsigned key = hi >> 2;
  if (hi - 0x03f00000u >= 0x7e700000u - 0x03f00000u)
    key = (gx == 0.0 && gy == 0.0) ? 0u : KEY_EXACT;
  return (key << 2) | (unsigned)bin;
}

// Gray rows [y_first, y_first + cnt) into s.g rows [r_first, r_first + cnt) (cnt <= 16).
// Warp w handles rows w and w + NWARP; lanes handle columns lane + 32 k (k < 4) and
// columns 128..131 in one combined pass.
__device__ __forceinline__ void ld_rgb(const double* a, unsigned long long pol, double& r,
                                       double& g, double& b) {
  asm("ld.global.nc.L2::cache_hint.f64 %0, [%3], %4;\n\t"
      "ld.global.nc.L2::cache_hint.f64 %1, [%3+8], %4;\n\t"
      "ld.global.nc.L2::cache_hint.f64 %2, [%3+16], %4;"
      : "=d"(r), "=d"(g), "=d"(b) : "l"(a), "l"(pol));
}
__device__ __forceinline__ void ld_rgb(const float* a, unsigned long long pol, double& r,
                                       double& g, double& b) {
  float x, y, z;
  asm("ld.global.nc.L2::cache_hint.f32 %0, [%3], %4;\n\t"
      "ld.global.nc.L2::cache_hint.f32 %1, [%3+4], %4;\n\t"
      "ld.global.nc.L2::cache_hint.f32 %2, [%3+8], %4;"
      : "=f"(x), "=f"(y), "=f"(z) : "l"(a), "l"(pol));
  r = x;
  g = y;
  b = z;
}

template <int CH, bool F64, int RPW = 2>  // RPW: rows per warp (cnt <= 8 RPW)
__device__ void band_gray(const Params& p, Smem& s, int v, int x0, int y_first, int r_first,
                          int cnt, unsigned long long pol) {
  using T = typename std::conditional<F64, double, float>::type;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int H = (int)p.H, W = (int)p.W;
  const T* img = (const T*)p.img + (long long)v * p.npx * CH;
  auto gray = [&](const T* px) -> double {
    if (CH == 3) {
      double rr, gg, bb;
      ld_rgb(px, pol, rr, gg, bb);
      double g = ((p.kgray[0] * rr) + (p.kgray[1] * gg)) + (p.kgray[2] * bb);
      g = g > 1.0 ? 1.0 : g;  // np.clip(., 0, 1); NaN passes; the sign of a zero cannot
      return g < 0.0 ? 0.0 : g;  // reach the output (blur sums start from +0, clip again)
    }
    return ld_hint(px, pol);  // a gray input is not clipped (edge_pipeline.py:134)
  };
  int xo[5];
#pragma unroll
  for (int k = 0; k < 4; ++k) xo[k] = clamp_i(x0 - 4 + lane + 32 * k, 0, W - 1) * CH;
  xo[4] = clamp_i(x0 - 4 + 128 + (lane & 3), 0, W - 1) * CH;
#pragma unroll
  for (int h = 0; h < RPW; ++h) {
    const int r = warp + NWARP * h;
    if (r < cnt) {
      const T* row = img + (long long)clamp_i(y_first + r, 0, H - 1) * W * CH;
      double* dst = s.g + (r_first + r) * GWP + lane;
#pragma unroll
      for (int k = 0; k < 4; ++k) dst[32 * k] = gray(row + xo[k]);
    }
  }
  const int r = warp + NWARP * (lane >> 2);
  if (lane < 4 * RPW && r < cnt)
    s.g[(r_first + r) * GWP + 128 + (lane & 3)] =
        gray(img + (long long)clamp_i(y_first + r, 0, H - 1) * W * CH + xo[4]);
}

// 5x5 blur of rows [y_first, y_first + cnt) (cnt <= 16) into s.b rows [rb_first, ...);
// blurred s.b row R sums s.g rows R .. R+4.  Thread (c, h): blurred column c (x = x0-2+c,
// computed at the clamped column), rows h*8 .. h*8+7, streaming the input rows top to bottom
// so every output sums its taps in NI_Correlate's row-major order.  Rows outside the image
// take the value of the clamped in-image row (mode="nearest" on the blurred image).
// Blurred rows outside the image take the value of the clamped in-image row (mode="nearest"
// on the blurred image): computed directly at the clamped row (band edges only).
template <bool FAST, int CH>
__device__ __noinline__ void blur_edge_rows(const Params& p, const double* gin, double* bout,
                                            int y0, int nr) {
  const int H = (int)p.H;
  for (int o = 0; o < nr; ++o) {
    const int y = y0 + o;
    if (y >= 0 && y < H) continue;
    const double* row = gin + (o + (clamp_i(y, 0, H - 1) - y)) * GWP;
    double a = 0.0;
    for (int di = 0; di < 5; ++di)
      for (int dj = 0; dj < 5; ++dj) {
        const int t25 = di * 5 + dj;
        const double w = p.w25[t25];
        if (FAST) a = (t25 == 0) ? row[di * GWP + dj] * w : a + row[di * GWP + dj] * w;
        else if ((p.keep_mask >> t25) & 1u) a = a + row[di * GWP + dj] * w;
      }
    bout[o * BWP] = (CH == 3) ? (a > 1.0 ? 1.0 : a) : np_clip01_int(a);
  }
}

template <bool FAST, int CH, int RT = SH>  // RT: output rows per thread (the prologue: 2)
__device__ void band_blur(const Params& p, Smem& s, int x0, int y_first, int rb_first, int cnt,
                          bool shift = false) {
  const int c = threadIdx.x & 127, h = threadIdx.x >> 7;
  const int H = (int)p.H, W = (int)p.W;
  const int r0 = h * RT;
  if (shift && h == 1) {  // the previous sub-step's last 4 blurred rows -> context rows 0..3;
                          // this thread overwrites their sources (rows 16..19) below
#pragma unroll
    for (int j = 0; j < 4; ++j) s.b[j * BWP + c] = s.b[(SR + j) * BWP + c];
  }
  if (r0 >= cnt) return;
  const int nr = min(RT, cnt - r0);
  const int gc = clamp_i(x0 - 2 + c, 0, W - 1) - x0 + 2;  // s.g column of the leftmost tap
  const double* gin = s.g + (rb_first + r0) * GWP + gc;
  auto wsym = [&](int di, int dj) { return p.w6[di < 2 ? 2 - di : di - 2][dj < 2 ? 2 - dj : dj - 2]; };
  auto finish = [&](double x) { return (CH == 3) ? (x > 1.0 ? 1.0 : x) : np_clip01_int(x); };
  double acc[RT];
#pragma unroll
  for (int r = 0; r < RT + 4; ++r) {
    double xv[5];
#pragma unroll
    for (int dj = 0; dj < 5; ++dj) xv[dj] = gin[r * GWP + dj];
    // innermost over the outputs: consecutive adds go to independent accumulators; each
    // output still sums its taps in row-major (di, dj) order
#pragma unroll
    for (int dj = 0; dj < 5; ++dj) {
#pragma unroll
      for (int o = 0; o < RT; ++o) {
        const int di = r - o;
        if (di < 0 || di > 4) continue;
        const int t25 = di * 5 + dj;
        if (FAST) {
          const double prod = xv[dj] * wsym(di, dj);
          acc[o] = (t25 == 0) ? prod : acc[o] + prod;
        } else {
          if (t25 == 0) acc[o] = 0.0;
          if ((p.keep_mask >> t25) & 1u) acc[o] = acc[o] + xv[dj] * p.w25[t25];
        }
      }
    }
  }
  double* bout = s.b + (rb_first + r0) * BWP + c;
  const int y0 = y_first + r0;
  if (nr == RT) {
#pragma unroll
    for (int o = 0; o < RT; ++o) bout[o * BWP] = finish(acc[o]);
  } else {
#pragma unroll
    for (int o = 0; o < RT; ++o)
      if (o < nr) bout[o * BWP] = finish(acc[o]);
  }
  if (y0 < 0 || y0 + nr > H) blur_edge_rows<FAST, CH>(p, gin, bout, y0, nr);  // rare
}

__device__ __forceinline__ void sobel_at(const double* t, const double* m, const double* d,
                                         double& gx, double& gy) {
  // NI_Correlate tap order with the zero taps skipped; the exact x2 taps as FMAs.
  gx = t[2] - t[0];
  gx = fma(-2.0, m[0], gx);
  gx = fma(2.0, m[2], gx);
  gx = gx - d[0];
  gx = gx + d[2];
  gy = fma(-2.0, t[1], -t[0]);
  gy = gy - t[2];
  gy = gy + d[0];
  gy = fma(2.0, d[1], gy);
  gy = gy + d[2];
}

// Direction bin (gradient_bin) with the common case inline and its constants in the
// kernel parameters.
__device__ __forceinline__ int dir_bin(const Params& p, double gx, double gy) {
  const double ax = fabs(gx), ay = fabs(gy);
  const double d0 = fma(-p.ktan, ax, ay);   // > 0: above pi/8 from the x axis
  const double d2 = fma(-p.ktan, ay, ax);   // > 0: below 3 pi/8
  const double tol = p.ktol * (ax + ay);
  if (fabs(d0) > tol && fabs(d2) > tol) {
    const int q13 = ((__double2hiint(gx) ^ __double2hiint(gy)) >= 0) ? 1 : 3;
    return d0 < 0.0 ? 0 : (d2 < 0.0 ? 2 : q13);
  }
  return gradient_bin(gx, gy);  // zero, near a boundary, or non-finite
}

// Sobel of rows [y_first, y_first + cnt) into s.q rows [rq_first, ...); s.q row R uses s.b
// rows R .. R+2.  Thread (c, h): magnitude column c (x = x0 - 1 + c), rows h*8 .. h*8+7,
// sliding a 3x3 window down s.b.  Cells outside the image hold 0 (edge_pipeline.py:97).
template <bool NMS>
__device__ void band_sobel(const Params& p, Smem& s, int x0, int y_first, int rq_first, int cnt,
                           bool shift = false) {
  const int c = threadIdx.x & 127, h = threadIdx.x >> 7;
  const int H = (int)p.H, W = (int)p.W;
  const int r0 = h * SH;
  if (shift && h == 1) {  // the previous sub-step's last 2 Sobel rows -> context rows 0..1;
                          // this thread overwrites their sources (rows 16..17) below
    s.q[c] = s.q[SR * MWP + c];
    s.q[MWP + c] = s.q[(SR + 1) * MWP + c];
  }
  if (r0 >= cnt) return;
  const int nr = min(SH, cnt - r0);
  const int x = x0 - 1 + c;
  const bool xin = x >= 0 && x < W;
  const int y0 = y_first + r0;
  const double* bin_ = s.b + (rq_first + r0) * BWP + c;
  unsigned* qout = s.q + (rq_first + r0) * MWP + c;
  double t[3], m[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    t[k] = bin_[k];
    m[k] = bin_[BWP + k];
  }
  auto row = [&](int j, bool check) {
    double d[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) d[k] = bin_[(j + 2) * BWP + k];
    double gx, gy;
    sobel_at(t, m, d, gx, gy);
    unsigned cellv = pack_cell(gx, gy, NMS ? dir_bin(p, gx, gy) : 0);
    const int y = y0 + j;
    if (!xin || (check && (y < 0 || y >= H))) cellv = 0u;
    qout[j * MWP] = cellv;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      t[k] = m[k];
      m[k] = d[k];
    }
  };
  if (nr == SH && y0 >= 0 && y0 + SH <= H) {
    // common case: straight-line code, so the window shift is register renaming
#pragma unroll
    for (int j = 0; j < SH; ++j) row(j, false);
  } else {
#pragma unroll
    for (int j = 0; j < SH; ++j)
      if (j < nr) row(j, true);
  }
}

// Exact glibc hypot at magnitude cell (s.q row rq, column c) of image row y (0 outside).
__device__ __forceinline__ double mag_exact(const Params& p, const Smem& s, int x0, int y,
                                            int rq, int c) {
  const int x = x0 - 1 + c;
  if (y < 0 || y >= (int)p.H || x < 0 || x >= (int)p.W) return 0.0;
  const double* b = s.b + rq * BWP + c;
  double gx, gy;
  sobel_at(b, b + BWP, b + 2 * BWP, gx, gy);
  return hypot_glibc(gx, gy);
}

// NMS decisions of output rows [y_first, y_first + cnt) (s.q row r + 1): warp w rows w and
// w + NWARP, lane l columns l + 32 k.  Suppressed pixels store 0 here; survivors and
// undecided pixels are appended to s.list as (r << 12) | (c << 2) | (undecided prev << 1) |
// undecided next (warp-aggregated).
template <bool NMS, bool MED>
__device__ void band_nms_decide(const Params& p, Smem& s, int v, int x0, int xw, int cb,
                                int y_first, int cnt, int parity, unsigned long long pol_mid) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long vbase = (long long)v * p.npx;
  const unsigned lt = lanemask_lt();
  unsigned bal[2][4];
  unsigned short entry[2][4];
  unsigned tot[2] = {0u, 0u};
#pragma unroll
  for (int hh = 0; hh < 2; ++hh) {
    const int r = warp + NWARP * hh;
    const bool row_ok = r < cnt;  // warp-uniform
    const unsigned* qrow = s.q + (r + 1) * MWP + 1;  // output column c at qrow[c]
    double* orow = p.out + vbase + (long long)(y_first + r) * p.W + x0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int c = lane + 32 * k;
      bool need = false;
      entry[hh][k] = 0;
      if (row_ok) {
        const unsigned qc = qrow[c];
        if (NMS) {
          const int bn = (int)(qc & 3u);
          // prev (dy, dx): bin0 (0,-1), bin1 (-1,-1), bin2 (-1,0), bin3 (-1,+1); next = -prev
          const int po = bn == 0 ? -1 : bn - MWP - 2;  // prev as an offset in s.q cells
          const int kc = (int)(qc >> 2), kp = (int)(qrow[c + po] >> 2), kn = (int)(qrow[c - po] >> 2);
          const int d1 = kc - kp, d2 = kc - kn;
          const bool sent = max(kc, max(kp, kn)) == (int)KEY_EXACT;
          const bool u1 = sent || ((unsigned)(d1 + 1) <= 2u && (kc | kp) != 0);
          const bool u2 = sent || ((unsigned)(d2 + 1) <= 2u && (kc | kn) != 0);
          // suppressed for sure: prev decided >= self, or next decided > self
          need = !((!u1 && d1 <= 0) || (!u2 && d2 < 0));
          entry[hh][k] = (unsigned short)(((unsigned)r << 12) | ((unsigned)c << 2) | (u1 ? 2u : 0u) |
                                          (u2 ? 1u : 0u));
        } else {
          need = (qc >> 2) != 0;
          entry[hh][k] = (unsigned short)(((unsigned)r << 12) | ((unsigned)c << 2));
        }
        const bool in = c < xw;
        need = need && in;
        // every pixel gets a full-line store here (0); survivors are overwritten by finish
        // (no median) or by the apply pass (median), so no line is ever partially written
        st_hint_if((MED || !need) && in, orow + c, 0.0, pol_mid);
      }
      bal[hh][k] = __ballot_sync(0xffffffffu, need);
      tot[hh] += __popc(bal[hh][k]);
    }
  }
  // one shared-list chunk per row (column order) and ONE survivor-list reservation per warp
  unsigned lbase0 = 0, lbase1 = 0, gbase = 0;
  if (lane == 0) {
    if (tot[0] + tot[1]) {
      lbase0 = atomicAdd(&s.list_n[parity], tot[0] + tot[1]);
      if (MED) gbase = atomicAdd(&p.ctl[v].nsurv, tot[0] + tot[1]);
    }
    lbase1 = lbase0 + tot[0];
  }
  lbase0 = __shfl_sync(0xffffffffu, lbase0, 0);
  lbase1 = __shfl_sync(0xffffffffu, lbase1, 0);
#pragma unroll
  for (int hh = 0; hh < 2; ++hh) {
    unsigned pre = hh ? lbase1 : lbase0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if ((bal[hh][k] >> lane) & 1u) s.list[pre + __popc(bal[hh][k] & lt)] = entry[hh][k];
      pre += __popc(bal[hh][k]);
    }
  }
  if (lane == 0 && MED) {  // row r's entries: list [rowl, ...) -> survivor list [rowg, ...)
    const int r0 = warp, r1 = warp + NWARP;
    if (r0 < cnt) { s.rowl[r0] = lbase0; s.rowg[r0] = gbase; }
    if (r1 < cnt) { s.rowl[r1] = lbase1; s.rowg[r1] = gbase + tot[0]; }
  }
}

// Finish the compacted pixels with all threads: exact magnitude, the undecided comparisons,
// the map store (L2 evict_last) and the median histogram.
__device__ void band_nms_finish(const Params& p, Smem& s, int v, int x0, int y_first, int parity,
                                unsigned long long pol_mid) {
  const unsigned n = s.list_n[parity];
  const long long vbase = (long long)v * p.npx;
  double* sval = ring_slot(p, v);
  unsigned* sidx = surv_idx(p, v);
  for (unsigned i = threadIdx.x; i < n; i += NT) {
    const unsigned e = s.list[i];
    const int r = (int)(e >> 12), c = (int)((e >> 2) & 0x3ffu);
    const int y = y_first + r;
    const double m = mag_exact(p, s, x0, y, r + 1, c + 1);
    bool keep = true;
    if (e & 3u) {
      const int bn = (int)(s.q[(r + 1) * MWP + 1 + c] & 3u);
      const int dy = bn == 0 ? 0 : -1, dx = bn == 0 ? -1 : bn - 2;
      if (e & 2u) keep = m > mag_exact(p, s, x0, y + dy, r + 1 + dy, c + 1 + dx);
      if (keep && (e & 1u)) keep = m >= mag_exact(p, s, x0, y - dy, r + 1 - dy, c + 1 - dx);
    }
    const double outv = keep ? m : 0.0;
    if (p.median) {
      // the entry's slot in its row segment of the view's survivor list; the apply pass
      // rebuilds the row from the segment (0 everywhere else)
      const unsigned at = s.rowg[r] + (i - s.rowl[r]);
      sval[at] = outv;
      sidx[at] = (unsigned)((long long)y * p.W + x0 + c);
      if (outv > 0.0) hist_add(s, hist_bin(outv));
    } else {
      st_hint(p.out + vbase + (long long)y * p.W + x0 + c, outv, pol_mid);
    }
  }
}

template <int CH, bool F64>
__device__ void prefetch_rows(const Params& p, int v, int x0, int xw, int y_lo, int y_hi,
                              unsigned long long pol);

template <int CH, bool F64>
__device__ void claim_next(const Params& p, Smem& s, unsigned long long pol_in);

// Copy rows [from, from + n) (n <= NWARP) of a shared array of pitch P to rows [0, n):
// warp wbase + r copies row r, lanes the columns.
template <typename E, int P>
__device__ __forceinline__ void shift_rows(E* a, int from, int n, int wbase = 0) {
  const int lane = threadIdx.x & 31, r = (int)(threadIdx.x >> 5) - wbase;
  if (r >= 0 && r < n) {
    const E* src = a + (from + r) * P;
    E* dst = a + r * P;
#pragma unroll
    for (int c = lane; c < P; c += 32) dst[c] = src[c];
  }
}

#ifdef IGS_PHASE_PROF
__device__ unsigned long long g_phase_ns[8];
#define PHASE_MARK(i)                                                             \
  do {                                                                            \
    if (threadIdx.x == 0) {                                                       \
      unsigned long long _t;                                                      \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t));                      \
      atomicAdd(&g_phase_ns[i], _t - t_prev);                                     \
      t_prev = _t;                                                                \
    }                                                                             \
  } while (0)
#else
#define PHASE_MARK(i) \
  do {                \
  } while (0)
#endif

template <bool FAST, int CH, bool F64>
__device__ void run_band(const Params& p, Smem& s, int v, int t, unsigned long long pol_in,
                         unsigned long long pol_mid) {
  const int H = (int)p.H, W = (int)p.W;
  const int cb = t % p.ncols, rb = t / p.ncols;
  const int x0 = cb * p.tw, xw = min(p.tw, W - x0);
  const int ya = rb * p.band_h, yb = min(ya + p.band_h, H);
#ifdef IGS_PHASE_PROF
  unsigned long long t_prev = 0;
  if (threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_prev));
#endif
  // prologue: gray rows [ya-4, ya+4+n0) -> s.g rows 0..; blurred [ya-2, ya+2) -> s.b rows 0..3;
  // Sobel rows [ya-1, ya+1) -> s.q rows 0..1
  if (threadIdx.x == 0) s.list_n[0] = 0;
  const int n0 = min(SR, yb - ya);
  band_gray<CH, F64, 3>(p, s, v, x0, ya - 4, 0, 8 + n0, pol_in);  // every row's loads in flight
  __syncthreads();
  band_blur<FAST, CH, 2>(p, s, x0, ya - 2, 0, 4);  // 2 rows per strip
  __syncthreads();
  if (p.nms) band_sobel<true>(p, s, x0, ya - 1, 0, 2);
  else band_sobel<false>(p, s, x0, ya - 1, 0, 2);
  int parity = 0;
  PHASE_MARK(6);  // prologue (gray 8 + n0 rows, blur 4, Sobel 2)
  // Sub-step: four barriers.  The gray rows of sub-step k+1 are converted in sub-step k's finish
  // phase (s.g rows 8.. are free once the Sobel phase has shifted the context rows), and the
  // blurred / Sobel context rows are shifted by the threads that overwrite their sources.
  for (int Y = ya; Y < yb; Y += SR) {
    const int n = min(SR, yb - Y);
    const bool more = Y + SR < yb;
    const bool first = Y == ya;
    if (threadIdx.x < 32) {  // warp 0: L2 prefetch of the next sub-step's input rows, or
                             // (last sub-step) the claim of the next task
      if (more) prefetch_rows<CH, F64>(p, v, x0, xw, Y + SR + 4, min(Y + 2 * SR, yb) + 4, pol_in);
      else claim_next<CH, F64>(p, s, pol_in);
    }
    if (threadIdx.x == 32) s.list_n[parity ^ 1] = 0;  // the next sub-step's list
    // s.b rows 0..3 hold blurred [Y-2, Y+2) (shifted here); new rows [Y+2, Y+2+n) -> rows 4 ..
    // (the prologue's Sobel rows 0..1 read only s.b rows 0..3)
    band_blur<FAST, CH>(p, s, x0, Y + 2, 4, n, !first);
    __syncthreads();
    if (more) PHASE_MARK(1);
    else PHASE_MARK(5);  // the last sub-step's blur phase carries the next-task claim
    // s.q rows 0..1 hold Sobel [Y-1, Y+1) (shifted here); new rows [Y+1, Y+1+n) -> rows 2 ..;
    // meanwhile keep gray rows [Y+n-4, Y+n+4) for the next sub-step
    if (p.nms) band_sobel<true>(p, s, x0, Y + 1, 2, n, !first);
    else band_sobel<false>(p, s, x0, Y + 1, 2, n, !first);
    if (more) shift_rows<double, GWP>(s.g, n, 8);
    __syncthreads();
    PHASE_MARK(2);
    if (p.nms) {
      if (p.median) band_nms_decide<true, true>(p, s, v, x0, xw, cb, Y, n, parity, pol_mid);
      else band_nms_decide<true, false>(p, s, v, x0, xw, cb, Y, n, parity, pol_mid);
    } else {
      if (p.median) band_nms_decide<false, true>(p, s, v, x0, xw, cb, Y, n, parity, pol_mid);
      else band_nms_decide<false, false>(p, s, v, x0, xw, cb, Y, n, parity, pol_mid);
    }
    __syncthreads();
    PHASE_MARK(3);
    // the next sub-step's gray rows [Y+SR+4, ...) -> s.g rows 8 .., with this sub-step's finish
    if (more) band_gray<CH, F64>(p, s, v, x0, Y + SR + 4, 8, min(SR, yb - Y - SR), pol_in);
    band_nms_finish(p, s, v, x0, Y, parity, pol_mid);
    parity ^= 1;
    __syncthreads();
    PHASE_MARK(4);
  }
}

// ------------------------------------------------ histogram-only chunk (median-only mode)
__device__ __noinline__ void run_hist_chunk(const Params& p, Smem& s, int v, int c) {
  const long long lo = (long long)c * CHUNK, hi = min(lo + (long long)CHUNK, p.npx);
  const double* src = (const double*)p.img + (long long)v * p.npx;
  for (long long i = lo + threadIdx.x; i < hi; i += NT) {
    double x = __ldg(src + i);
    if (x > 0.0) hist_add(s, hist_bin(x));
  }
}

// Flush the block histogram into the view's global histogram and clear it.
__device__ void flush_hist(const Params& p, Smem& s, int v) {
  __syncthreads();
  unsigned* gh = p.hist + (long long)v * NB;
  for (int i = threadIdx.x; i < NB / 2; i += NT) {
    const unsigned h = s.hist[i];
    if (h) {
      if (h & 0xffffu) atomicAdd(&gh[2 * i], h & 0xffffu);
      if (h >> 16) atomicAdd(&gh[2 * i + 1], h >> 16);
      s.hist[i] = 0;
    }
  }
}

// Locate the bin holding rank `rank` in a histogram of nb bins (nb % NT == 0, <= 16 * NT).
// Every thread returns the same (bin, rank within bin) via smem.
template <int NBINS>
__device__ __noinline__ void locate(const unsigned* h, Smem& s, unsigned long long rank, int& bin,
                       unsigned long long& rin, bool global_mem) {
  constexpr int PER = NBINS / NT;
  unsigned loc[PER], sum = 0;
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    loc[k] = global_mem ? __ldcg(&h[threadIdx.x * PER + k]) : h[threadIdx.x * PER + k];
    sum += loc[k];
  }
  unsigned total;
  unsigned before = block_exclusive_scan(sum, s.warp_sums, &total);
  unsigned long long cum = before;
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    if (loc[k] && rank >= cum && rank < cum + loc[k]) {
      s.ivals[0] = threadIdx.x * PER + k;
      s.u64[0] = rank - cum;
    }
    cum += loc[k];
  }
  __syncthreads();
  bin = s.ivals[0];
  rin = s.u64[0];
  __syncthreads();
}

// Last E task of a view: locate the level-1 bins holding ranks k1 = (n-1)/2 and k2 = n/2.
__device__ __noinline__ void find_median_bins(const Params& p, Smem& s, int v) {
  const unsigned* gh = p.hist + (long long)v * NB;
  constexpr int PER = NB / NT;
  unsigned local = 0;
#pragma unroll
  for (int k = 0; k < PER; ++k) local += __ldcg(&gh[threadIdx.x * PER + k]);
  unsigned total = __reduce_add_sync(0xffffffffu, local);
  if ((threadIdx.x & 31) == 0) s.warp_sums[threadIdx.x >> 5] = total;
  __syncthreads();
  total = 0;
#pragma unroll
  for (int w = 0; w < NWARP; ++w) total += s.warp_sums[w];
  __syncthreads();
  ViewCtl& ctl = p.ctl[v];
  if (total == 0) {
    if (threadIdx.x == 0) {
      ctl.npos = 0;
      ctl.median = 1.0;
      ctl.denom = 2.0 * 1.0;
      if (p.medians) p.medians[v] = 1.0;
    }
  } else {
    int b1, b2;
    unsigned long long r1, r2;
    locate<NB>(gh, s, (total - 1) / 2, b1, r1, true);
    locate<NB>(gh, s, total / 2, b2, r2, true);
    if (threadIdx.x == 0) {
      ctl.npos = total;
      ctl.b1 = b1;
      ctl.r1 = r1;
      ctl.b2 = b2;
      ctl.r2 = r2;
    }
  }
  if (threadIdx.x == 0) {  // C tasks: chunks of the survivor list (fused) or of the input
    const unsigned long long ns = p.mode == MODE_FUSED ? __ldcg(&ctl.nsurv) : 0ull;
    ctl.tca = p.mode == MODE_FUSED ? (unsigned)((ns + p.chunk - 1) / p.chunk) : (unsigned)p.TC;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (total == 0) atomicExch(&ctl.select_done, 1u);
    atomicExch(&ctl.binfound, 1u);
  }
}

__device__ __forceinline__ int sub_bin(unsigned long long bits) {
  return (int)((bits >> SUB_SHIFT) & (NB2 - 1));
}

// ---------------------------------------------------- streamed chunks for C and A tasks
// A C/A task streams its chunk of the thinned map through shared memory in PIECE-sized
// pieces with TMA bulk copies (two buffers in flight, mbarrier completion), so the task is
// not limited by register-held loads.  Unaligned views fall back to plain loads.
constexpr int PIECE = 1280;                     // doubles per piece (10 KB)
constexpr int NBUF = 4;                         // pieces in flight
constexpr int STAGE = 512;                      // staged candidates per list in a C task
constexpr int APIECE = 1024;                    // survivor entries per apply piece (12 KB)
static_assert(NBUF * APIECE * 12 <= (GR * GWP + BR * BWP) * 8 + QR * MWP * 4, "apply pieces fit in g + b + q");
static_assert(CHUNK % APIECE == 0 && APIECE % 4 == 0, "apply pieces tile a chunk");
static_assert(NBUF * PIECE + 2 * STAGE <= GR * GWP + BR * BWP + QR * MWP / 2,
              "stream buffers fit in g + b + q");

// g, b and q are contiguous at the start of Smem: one arena for C/A/select scratch.
__device__ __forceinline__ double* arena(Smem& s) { return reinterpret_cast<double*>(&s); }

template <typename Visit>
__device__ void stream_chunk(Smem& s, const double* src, long long lo, long long hi,
                             Visit visit) {
  const long long n = hi - lo;
  const bool aligned = ((((uintptr_t)(src + lo)) & 15) == 0);
  if (!aligned) {
    for (long long i = lo + threadIdx.x; i < hi; i += NT) visit(i, __ldcg(src + i));
    __syncthreads();  // same exit contract as the bulk path: every visit has completed
    return;
  }
  const long long nfull = n & ~1ll;  // bulk part: a multiple of 16 bytes
  const int npieces = (int)((nfull + PIECE - 1) / PIECE);
  // barriers initialised once per CTA (kernel prologue); piece j of the CTA's bulk-copy
  // sequence uses barrier j % NBUF at parity (j / NBUF) & 1
  __syncthreads();
  const unsigned seq = s.mbar_seq;
  auto issue = [&](int k) {
    const long long off = (long long)k * PIECE;
    const unsigned len = (unsigned)min((long long)PIECE, nfull - off);
    bulk_load(arena(s) + (k % NBUF) * PIECE, src + lo + off, len * 8u, &s.mbar[(seq + k) % NBUF]);
  };
  if (threadIdx.x == 0) {
    fence_proxy_async();      // earlier generic smem accesses of the arena -> async-proxy writes
    fence_proxy_async_all();  // survivor lists written by other CTAs -> async-proxy reads
    for (int k = 0; k < NBUF && k < npieces; ++k) issue(k);
  }
  __syncthreads();
  for (int k = 0; k < npieces; ++k) {
    const double* buf = arena(s) + (k % NBUF) * PIECE;
    mbar_wait(&s.mbar[(seq + k) % NBUF], ((seq + k) / NBUF) & 1u);
    const long long off = (long long)k * PIECE;
    const int len = (int)min((long long)PIECE, nfull - off);
    for (int i = threadIdx.x; i < len; i += NT) visit(lo + off + i, buf[i]);
    __syncthreads();
    if (threadIdx.x == 0 && k + NBUF < npieces) {
      fence_proxy_async();
      issue(k + NBUF);
    }
  }
  if (threadIdx.x == 0) s.mbar_seq = seq + (unsigned)npieces;  // read again after a barrier
  if ((n & 1) && threadIdx.x == 0) visit(hi - 1, __ldcg(src + hi - 1));
  __syncthreads();
}

// ------------------------------------------------------------- C: collect candidates
// Candidates are bucketed by level-2 bin (returning atomics on the level-2 histogram) and
// also appended to a flat per-view list: staged in shared memory, then ONE global atomic per
// task reserves the space.
// Stage candidate x of list `list` in shared memory; false (spilled straight to the global
// list) once STAGE are staged.
__device__ __forceinline__ bool stage(Smem& s, double x, int list, double* overflow_base,
                                      int dir, unsigned* gcounter) {
  double* buf = arena(s) + NBUF * PIECE + list * STAGE;
  const int k = atomicAdd(&s.ivals[1 + list], 1);
  if (k < STAGE) {
    buf[k] = x;
    return true;
  }
  const unsigned g = atomicAdd(gcounter, 1u);  // rare: more than STAGE candidates in a chunk
  overflow_base[dir * (long long)g] = x;
  return false;
}

__device__ __noinline__ void run_collect(const Params& p, Smem& s, int v, int c) {
  ViewCtl& ctl = p.ctl[v];
  if (threadIdx.x == 0) {  // claimed only once binfound (and the ring slot) is published
    s.ivals[0] = __ldcg(&ctl.npos) ? 1 : 0;
    s.ivals[1] = 0;
    s.ivals[2] = 0;
    s.scratch[0] = __ldcg(&ctl.b1);
    s.scratch[1] = __ldcg(&ctl.b2);
  }
  __syncthreads();
  const int npos = s.ivals[0], b1 = s.scratch[0], b2 = s.scratch[1];
  __syncthreads();
  if (!npos) return;
  // fused: a chunk of the view's survivor list; median-only: a chunk of the input array
  const bool fused = p.mode == MODE_FUSED;
  const double* src = fused ? ring_slot(p, v) : (const double*)p.img + (long long)v * p.npx;
  const long long nsrc = fused ? (long long)__ldcg(&ctl.nsurv) : p.npx;
  const int slot = v % RING;
  double* cand = cand_lists(p, v);
  double* cand2 = cand + p.npx - 1;
  unsigned* h2a = p.hist2 + (long long)slot * 2 * NB2;
  unsigned* h2b = h2a + NB2;
  double* sla = p.slots + (long long)slot * 2 * NB2 * SLOTS;
  double* slb = sla + NB2 * SLOTS;
  const long long lo = (long long)c * p.chunk, hi = min(lo + (long long)p.chunk, nsrc);
  auto bucket = [&](double x, int list) {  // level-2 bucket (returning global atomic)
    const int sb = sub_bin((unsigned long long)__double_as_longlong(x));
    const unsigned k = atomicAdd(&(list ? h2b : h2a)[sb], 1u);
    if (k < (unsigned)SLOTS) (list ? slb : sla)[sb * SLOTS + k] = x;
  };
  // the scan only stages candidates in shared memory; their global atomics are issued
  // together afterwards (one round trip per task instead of one per hit)
  stream_chunk(s, src, lo, hi, [&](long long, double x) {
    if (!(x > 0.0)) return;
    const int hb = hist_bin(x);
    if (hb != b1 && hb != b2) return;
    const int list = hb == b1 ? 0 : 1;
    if (!stage(s, x, list, list ? cand2 : cand, list ? -1 : 1, list ? &ctl.cnt2 : &ctl.cnt1))
      bucket(x, list);  // rare: spilled past STAGE, bucketed right away
  });
  const int n1 = min(s.ivals[1], STAGE), n2s = min(s.ivals[2], STAGE);
  const double* st = arena(s) + NBUF * PIECE;
  for (int k = threadIdx.x; k < n1 + n2s; k += NT) {
    if (k < n1) bucket(st[k], 0);
    else bucket(st[STAGE + k - n1], 1);
  }
  // append the staged lists: one reservation per list
  if (threadIdx.x == 0) {
    s.u64[0] = n1 ? atomicAdd(&ctl.cnt1, (unsigned)n1) : 0u;
    s.u64[1] = n2s ? atomicAdd(&ctl.cnt2, (unsigned)n2s) : 0u;
  }
  __syncthreads();
  const unsigned long long o1 = s.u64[0], o2 = s.u64[1];
  for (int k = threadIdx.x; k < n1; k += NT) cand[o1 + k] = st[k];
  for (int k = threadIdx.x; k < n2s; k += NT) cand2[-(long long)(o2 + k)] = st[STAGE + k];
}

// Block-wide radix select over n positive doubles (bit order == value order) stored at
// src[dir * i] (global or shared).  Bits above `top` are already known to be equal.
__device__ __noinline__ unsigned long long block_radix_select(Smem& s, const double* src, long long n, int dir,
                                                 unsigned long long rank, int top, bool global_mem) {
  unsigned long long prefix = 0, pmask = top >= 63 ? 0ull : (~0ull << (top + 1));
  unsigned* h = s.hist;  // reused; cleared on exit
  if (n > 0 && pmask) {
    double x0 = global_mem ? __ldcg(src) : src[0];
    prefix = (unsigned long long)__double_as_longlong(x0) & pmask;
  }
  for (int hb = top; hb >= 0; hb -= 11) {
    const int width = hb + 1 < 11 ? hb + 1 : 11;
    const int shift = hb + 1 - width;
    const unsigned dmask = (1u << width) - 1;
    for (int i = threadIdx.x; i < NBR; i += NT) h[i] = 0;
    __syncthreads();
    for (long long i = threadIdx.x; i < n; i += NT) {
      const double x = global_mem ? __ldcg(src + dir * i) : src[dir * i];
      const unsigned long long bits = (unsigned long long)__double_as_longlong(x);
      if ((bits & pmask) == prefix) atomicAdd(&h[(bits >> shift) & dmask], 1u);
    }
    __syncthreads();
    int d;
    unsigned long long r;
    locate<NBR>(h, s, rank, d, r, false);
    rank = r;
    prefix |= (unsigned long long)d << shift;
    pmask |= (unsigned long long)dmask << shift;
  }
  for (int i = threadIdx.x; i < NBR; i += NT) h[i] = 0;
  __syncthreads();
  return prefix;
}

// Exact order statistics of the median.  For each wanted rank (one for an odd count, two for
// an even one) the level-2 histogram of its level-1 bin names a sub-bin (bits 47..36); one
// unrolled pass over the candidate list stages the members of the (at most two) sub-bins in
// shared memory, where a radix select over bits 35..0 finishes.  Clamped level-1 bins
// (0, NB-1) and oversize sub-bins fall back to a full-width select over the candidates.
struct Want {
  const double* src;   // candidate region, element i at src[dir * i]
  long long n;
  int dir;
  int bin;             // level-1 bin
  unsigned long long rank;
  const unsigned* h2;
  int sb;              // level-2 bin (-1: generic path)
  unsigned long long r2;
  unsigned cnt;
};

__device__ __noinline__ void gather_subbins(Smem& s, const double* src, long long n, int dir, int sbA,
                               double* bufA, int sbB, double* bufB) {
  constexpr int U = 8;
  for (long long base = 0; base < n; base += NT * U) {
    double x[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const long long i = base + k * NT + threadIdx.x;
      x[k] = i < n ? __ldcg(src + dir * i) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      if (base + k * NT + threadIdx.x >= n) continue;
      const int sb = sub_bin((unsigned long long)__double_as_longlong(x[k]));
      if (sb == sbA) bufA[atomicAdd(&s.ivals[1], 1)] = x[k];
      else if (sb == sbB) bufB[atomicAdd(&s.ivals[2], 1)] = x[k];
    }
  }
}

// Rank selection for a short shared-memory list (n <= NT): element t's rank is the number of
// smaller elements plus equal ones before it; the owner of rank `rank` publishes its bits.
__device__ __noinline__ unsigned long long small_select(Smem& s, const double* buf, int n,
                                           unsigned long long rank) {
  const int t = threadIdx.x;
  if (t < n) {
    const unsigned long long x = (unsigned long long)__double_as_longlong(buf[t]);
    unsigned r = 0;
    for (int j = 0; j < n; ++j) {
      const unsigned long long y = (unsigned long long)__double_as_longlong(buf[j]);
      r += (y < x) || (y == x && j < t);
    }
    if (r == rank) s.u64[1] = x;
  }
  __syncthreads();
  const unsigned long long res = s.u64[1];
  __syncthreads();
  return res;
}

__device__ __noinline__ unsigned long long select_staged(Smem& s, const double* buf, unsigned n,
                                            unsigned long long rank) {
  if (n <= (unsigned)NT) return small_select(s, buf, (int)n, rank);
  return block_radix_select(s, buf, n, 1, rank, 35, false);
}

__device__ __noinline__ void plan(Smem& s, Want& w) {
  w.sb = -1;
  if (w.bin == 0 || w.bin == NB - 1) return;
  int sb;
  unsigned long long r2;
  locate<NB2>(w.h2, s, w.rank, sb, r2, true);
  w.sb = sb;
  w.r2 = r2;
  w.cnt = __ldcg(&w.h2[sb]);
}

// Order statistic of one Want: from the bucketed slots when the level-2 bin holds at most
// SLOTS candidates (the common case: ~1 per bin), else by staging the level-2 bin from the
// flat candidate list, else (clamped level-1 bin) by a full-width select over the list.
__device__ __noinline__ double resolve(Smem& s, const Want& w, const double* slots) {
  if (w.sb < 0)
    return __longlong_as_double(block_radix_select(s, w.src, w.n, w.dir, w.rank, 63, true));
  double* buf = s.g;
  if (w.cnt <= (unsigned)SLOTS) {
    if (threadIdx.x < w.cnt) buf[threadIdx.x] = __ldcg(slots + w.sb * SLOTS + threadIdx.x);
    __syncthreads();
    return __longlong_as_double(small_select(s, buf, (int)w.cnt, w.r2));
  }
  if (w.cnt > (unsigned)SEL_CAP)
    return __longlong_as_double(block_radix_select(s, w.src, w.n, w.dir, w.rank, 63, true));
  if (threadIdx.x == 0) {
    s.ivals[1] = 0;
    s.ivals[2] = 0;
  }
  __syncthreads();
  gather_subbins(s, w.src, w.n, w.dir, w.sb, buf, -2, buf);
  __syncthreads();
  return __longlong_as_double(select_staged(s, buf, w.cnt, w.r2));
}

__device__ __noinline__ void run_select(const Params& p, Smem& s, int v) {
  ViewCtl& ctl = p.ctl[v];
  const int slot = v % RING;
  const double* cand = cand_lists(p, v);
  const unsigned* h2a = p.hist2 + (long long)slot * 2 * NB2;
  const unsigned* h2b = h2a + NB2;
  const double* sla = p.slots + (long long)slot * 2 * NB2 * SLOTS;
  const double* slb = sla + NB2 * SLOTS;
  const unsigned n1 = __ldcg(&ctl.cnt1), n2 = __ldcg(&ctl.cnt2);
  const int b1 = __ldcg(&ctl.b1), b2 = __ldcg(&ctl.b2);
  const unsigned long long npos = __ldcg(&ctl.npos);
  const bool even = (npos & 1ull) == 0;
  Want w1{cand, n1, 1, b1, __ldcg(&ctl.r1), h2a, -1, 0, 0};
  plan(s, w1);
  const double a = resolve(s, w1, sla);
  double m = a;
  if (even) {
    Want w2 = (b2 == b1) ? Want{cand, n1, 1, b1, __ldcg(&ctl.r2), h2a, -1, 0, 0}
                         : Want{cand + p.npx - 1, n2, -1, b2, __ldcg(&ctl.r2), h2b, -1, 0, 0};
    plan(s, w2);
    const double b = resolve(s, w2, b2 == b1 ? sla : slb);
    m = (a + b) / 2.0;
  }
  // clear this slot's level-2 histograms for view v + RING
  unsigned* h2w = p.hist2 + (long long)slot * 2 * NB2;
  for (int i = threadIdx.x; i < 2 * NB2; i += NT) h2w[i] = 0;
  if (threadIdx.x == 0) {
    ctl.median = m;
    ctl.denom = 2.0 * m;
    if (p.medians) p.medians[v] = m;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicExch(&ctl.select_done, 1u);
  }
}

// ------------------------------------------------------------------ A: apply
__device__ __forceinline__ double normalise(double x, double denom, double rd, bool plain) {
  double q;
  if (plain && x == 0.0) q = x * rd;                       // +-0 / denom, sign kept
  else if (plain && fabs(x) < 0x1p+900 && fabs(x) > 0x1p-900) q = div_by(x, denom, rd);
  else q = x / denom;
  return np_min1(q);
}

__device__ __noinline__ void run_apply(const Params& p, Smem& s, int v, int c, unsigned long long pol_out) {
  ViewCtl& ctl = p.ctl[v];  // claimed only once select_done is published
  const double denom = __ldcg(&ctl.denom);
  const double rd = __drcp_rn(denom);
  const bool plain = isfinite(denom) && denom > 0x1p-1000 && denom < 0x1p+1000;
  double* dst = p.out + (long long)v * p.npx;
  if (p.mode == MODE_FUSED) {
    // a chunk of the survivor list: the normalised values overwrite their pixels (the E task
    // wrote full lines of zeros, so these stores merge into lines still in L2)
    // values and pixel indices arrive by TMA bulk copies, NBUF pieces of APIECE entries in
    // flight (the list is 16-byte aligned at every chunk start; a piece's copy may run past the
    // chunk end inside the list allocation -- those entries are not visited)
    const double* sval = ring_slot(p, v);
    const unsigned* sidx = surv_idx(p, v);
    const long long n = (long long)__ldcg(&ctl.nsurv);
    const long long lo = (long long)c * p.chunk, hi = min(lo + (long long)p.chunk, n);
    const int npieces = (int)((hi - lo + APIECE - 1) / APIECE);
    double* vbuf = arena(s);
    unsigned* ibuf = reinterpret_cast<unsigned*>(arena(s) + NBUF * APIECE);
    __syncthreads();
    const unsigned seq = s.mbar_seq;
    auto issue = [&](int k) {
      const long long off = lo + (long long)k * APIECE;
      const unsigned len = (unsigned)min((long long)APIECE, hi - off);
      const unsigned len4 = (len + 3u) & ~3u;  // 16-byte multiple for the index copy
      unsigned long long* bar = &s.mbar[(seq + k) % NBUF];
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                   "r"(len4 * 12u)
                   : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
              "r"(smem_u32(vbuf + (k % NBUF) * APIECE)),
          "l"(sval + off), "r"(len4 * 8u), "r"(smem_u32(bar))
          : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
              "r"(smem_u32(ibuf + (k % NBUF) * APIECE)),
          "l"(sidx + off), "r"(len4 * 4u), "r"(smem_u32(bar))
          : "memory");
    };
    if (threadIdx.x == 0) {
      fence_proxy_async();
      fence_proxy_async_all();
      for (int k = 0; k < NBUF && k < npieces; ++k) issue(k);
    }
    __syncthreads();
    for (int k = 0; k < npieces; ++k) {
      mbar_wait(&s.mbar[(seq + k) % NBUF], ((seq + k) / NBUF) & 1u);
      const long long off = lo + (long long)k * APIECE;
      const int len = (int)min((long long)APIECE, hi - off);
      const double* vb = vbuf + (k % NBUF) * APIECE;
      const unsigned* ib = ibuf + (k % NBUF) * APIECE;
      for (int i = threadIdx.x; i < len; i += NT) {
        const double x = vb[i];
        st_hint_if(x != 0.0, dst + ib[i], normalise(x, denom, rd, plain), pol_out);
      }
      __syncthreads();
      if (threadIdx.x == 0 && k + NBUF < npieces) {
        fence_proxy_async();
        issue(k + NBUF);
      }
    }
    if (threadIdx.x == 0) s.mbar_seq = seq + (unsigned)npieces;
    return;
  }
  const double* src = (const double*)p.img + (long long)v * p.npx;
  const long long lo = (long long)c * CHUNK, hi = min(lo + (long long)CHUNK, p.npx);
  stream_chunk(s, src, lo, hi, [&](long long i, double x) {
    st_hint(dst + i, normalise(x, denom, rd, plain), pol_out);
  });
}

// ------------------------------------------------------------- scheduler
// Thread 0 claims the next task, in priority order: an A chunk of the oldest view whose
// median is published, a C chunk of the oldest view whose bins are published (and whose
// candidate ring slot is free), else the next E band if it is at most `ahead` views past the
// A front (bounding the L2-resident thinned maps).  A/C work is claimed only when ready, so
// no task ever waits; TASK_NONE means "nothing ready right now".
enum TaskKind { TASK_END = 0, TASK_E = 1, TASK_C = 2, TASK_A = 3, TASK_NONE = 4 };

// Optional per-task trace (igs_debug_edge_trace): {start_ns, end_ns, kind, view, idx, smid}.
struct TraceRec {
  unsigned long long t0, t1;
  int kind, view, idx, sm;
};
__device__ TraceRec* g_trace = nullptr;
__device__ unsigned long long g_trace_cap = 0;
__device__ unsigned long long g_trace_n = 0;

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Ring slot v % RING is free for view v once view v - RING has retired: its median is
// published and every one of its apply tasks (the last readers of the slot) has finished.
__device__ __forceinline__ bool ring_free(const Params& p, unsigned v) {
  if (v < (unsigned)RING) return true;
  const ViewCtl& old = p.ctl[v - RING];
  return ld_acquire(&old.select_done) && ld_acquire(&old.a_done) >= __ldcg(&old.tca);
}

__device__ void claim_task(const Params& p, Smem& s, int& kind, int& view, int& idx) {
  unsigned* sched = p.sched;
  const unsigned B = (unsigned)p.B;
  // a band claimed earlier whose ring slot was still in use runs as soon as the slot is free
  if (s.pend_valid && ring_free(p, (unsigned)s.pend_view)) {
    kind = TASK_E; view = s.pend_view; idx = s.pend_idx;
    s.pend_valid = 0;
    return;
  }
  if (p.median) {
    for (;;) {  // A
      const unsigned v = ld_acquire(&sched[2]);
      if (v >= B || !ld_acquire(&p.ctl[v].select_done)) break;
      const unsigned c = atomicAdd(&p.ctl[v].a_claim, 1u);
      if (c < (p.mode == MODE_FUSED ? __ldcg(&p.ctl[v].tca) : (unsigned)p.TC)) {
        kind = TASK_A; view = (int)v; idx = (int)c;
        return;
      }
      atomicCAS(&sched[2], v, v + 1);
    }
    for (;;) {  // C
      const unsigned v = ld_acquire(&sched[1]);
      if (v >= B || !ld_acquire(&p.ctl[v].binfound)) break;
      if (v >= (unsigned)RING && !ld_acquire(&p.ctl[v - RING].select_done)) break;
      const unsigned c = atomicAdd(&p.ctl[v].c_claim, 1u);
      if (c < __ldcg(&p.ctl[v].tca)) {
        kind = TASK_C; view = (int)v; idx = (int)c;
        return;
      }
      atomicCAS(&sched[1], v, v + 1);
    }
    if (s.pend_valid) {  // at most one deferred band per CTA
      kind = TASK_NONE;
      return;
    }
  }
  const unsigned long long total_e = (unsigned long long)p.B * p.TE;
  unsigned long long* e_next = (unsigned long long*)&sched[4];
  unsigned long long t = ld_acquire64(e_next);
  // throttle: E at most `ahead` views past the A front (racy by design: concurrent claimers
  // may overshoot; the ring guard below makes an overshoot safe).  A claim is one atomicAdd:
  // a compare-and-swap claim serialises the grid on the atomic's round trip.
  if (t < total_e && !(p.median && t / p.TE >= ld_acquire(&sched[2]) + (unsigned)p.ahead)) {
    t = atomicAdd(e_next, 1ull);
    if (t < total_e) {
      const unsigned v = (unsigned)(t / p.TE);
      const int i = (int)(t - (unsigned long long)v * p.TE);
      if (p.median && !ring_free(p, v)) {
        // view v - RING still reads ring slot v % RING: defer the band (this CTA keeps
        // running collect / apply work meanwhile, so older views always make progress)
        s.pend_view = (int)v;
        s.pend_idx = i;
        s.pend_valid = 1;
        kind = TASK_NONE;
        return;
      }
      kind = TASK_E; view = (int)v; idx = i;
      return;
    }
  }
  if (!p.median) {
    kind = t >= total_e ? TASK_END : TASK_NONE;
    return;
  }
  kind = ld_acquire(&sched[2]) >= B ? TASK_END : TASK_NONE;
}

// L2 prefetch of input rows [y_lo, y_hi) (clamped) of a band: one bulk prefetch per row,
// the rows spread over the lanes of the calling warp, with the input's evict_first policy.
template <int CH, bool F64>
__device__ void prefetch_rows(const Params& p, int v, int x0, int xw, int y_lo, int y_hi,
                              unsigned long long pol) {
  using T = typename std::conditional<F64, double, float>::type;
  const int H = (int)p.H, W = (int)p.W;
  const int xl = clamp_i(x0 - 4, 0, W - 1), xh = clamp_i(x0 + xw + 4, 1, W);
  const char* base = (const char*)p.img;
  const unsigned long long total = ((unsigned long long)p.B * p.npx * CH * sizeof(T)) & ~15ull;
  y_lo = clamp_i(y_lo, 0, H);
  y_hi = clamp_i(y_hi, 0, H);
  for (int y = y_lo + (int)(threadIdx.x & 31); y < y_hi; y += 32) {
    const unsigned long long row = (unsigned long long)v * p.npx + (unsigned long long)y * W;
    unsigned long long a = ((row + xl) * CH * sizeof(T)) & ~15ull;
    unsigned long long e = ((row + xh) * CH * sizeof(T) + 15) & ~15ull;
    if (e > total) e = total;
    if (e <= a) continue;
    asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(base + a),
                 "r"((unsigned)(e - a)), "l"(pol)
                 : "memory");
  }
}

template <int CH, bool F64>
__device__ void prefetch_band_start(const Params& p, int v, int t, unsigned long long pol) {
  const int cb = t % p.ncols, rb = t / p.ncols;
  const int x0 = cb * p.tw, xw = min(p.tw, (int)p.W - x0);
  const int ya = rb * p.band_h;
  prefetch_rows<CH, F64>(p, v, x0, xw, ya - 4, ya + SR + 4, pol);
}

// Thread 0: claim the next task into s.task_* and warm L2 with its input rows.
template <int CH, bool F64>
__device__ void claim_next(const Params& p, Smem& s, unsigned long long pol_in) {
  // called by a whole warp: lane 0 claims, the warp prefetches the first rows of a band
  if ((threadIdx.x & 31) == 0) {
    int nk = 0, nv = 0, ni = 0;
    claim_task(p, s, nk, nv, ni);
    s.task_kind = nk;
    s.task_view = nv;
    s.task_idx = ni;
  }
  __syncwarp();
  if (s.task_kind == TASK_E && p.mode == MODE_FUSED)
    prefetch_band_start<CH, F64>(p, s.task_view, s.task_idx, pol_in);
}

template <bool FAST, int CH, bool F64>
__global__ void __launch_bounds__(NT, IGS_MINB) edge_persistent_kernel(const __grid_constant__ Params p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& s = *reinterpret_cast<Smem*>(smem_raw);
  for (int i = threadIdx.x; i < NB / 2; i += NT) s.hist[i] = 0;
  if (threadIdx.x == 0) {
    for (int k = 0; k < 4; ++k) mbar_init(&s.mbar[k]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    s.mbar_seq = 0;
    s.pend_valid = 0;
  }
  const unsigned long long pol_in = policy_evict_first();
  const unsigned long long pol_mid = policy_evict_last();
  const unsigned long long pol_out = policy_evict_first();
  if (threadIdx.x == 0) {
    int kind = 0, view = 0, idx = 0;
    claim_task(p, s, kind, view, idx);
    s.task_kind = kind;
    s.task_view = view;
    s.task_idx = idx;
  }
  __syncthreads();
  TraceRec* trace = g_trace;
  for (;;) {
    const int kind = s.task_kind, v = s.task_view, idx = s.task_idx;
    __syncthreads();
    if (kind == TASK_END) break;
    const unsigned long long t_start = trace ? gtimer() : 0ull;
    // Claim the next task while this one runs: short tasks claim now; a fused band claims at
    // the start of its last sub-step, so ready C/A work is not held behind a whole band.
    const bool late_claim = kind == TASK_E && p.mode == MODE_FUSED;
    // C / A tasks: the last warp claims (the tasks' first phases use warps 0..3 most)
    if (threadIdx.x >= NT - 32 && !late_claim) claim_next<CH, F64>(p, s, pol_in);
    if (kind == TASK_E) {
      if (p.mode == MODE_FUSED) run_band<FAST, CH, F64>(p, s, v, idx, pol_in, pol_mid);
      else run_hist_chunk(p, s, v, idx);
      if (p.median) {
        flush_hist(p, s, v);
        __syncthreads();
        if (threadIdx.x == 0) {
          __threadfence();
          s.flag = (atomicAdd(&p.ctl[v].tiles_done, 1u) == (unsigned)p.TE - 1);
          if (s.flag) __threadfence();
        }
        __syncthreads();
        if (s.flag) find_median_bins(p, s, v);
      }
    } else if (kind == TASK_C) {
      run_collect(p, s, v, idx);
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        s.flag = __ldcg(&p.ctl[v].npos) &&
                 (atomicAdd(&p.ctl[v].collect_done, 1u) == __ldcg(&p.ctl[v].tca) - 1);
        if (s.flag) __threadfence();
      }
      __syncthreads();
      if (s.flag) run_select(p, s, v);
    } else if (kind == TASK_A) {
      run_apply(p, s, v, idx, pol_out);
      __syncthreads();
      if (threadIdx.x == 0) {  // every read of the ring slot by this task has landed
        __threadfence();
        atomicAdd(&p.ctl[v].a_done, 1u);
      }
    } else if (threadIdx.x == 0) {
      __nanosleep(1000);
    }
    __syncthreads();
    if (trace && threadIdx.x == 0) {
      const unsigned long long k = atomicAdd(&g_trace_n, 1ull);
      if (k < g_trace_cap) {
        unsigned sm;
        asm("mov.u32 %0, %%smid;" : "=r"(sm));
        trace[k] = TraceRec{t_start, gtimer(), kind, v, idx, (int)sm};
      }
    }
  }
}

// ------------------------------------------------------------- host side
struct Layout {
  size_t ctl, hist, hist2, slots, cand, queue, zero_bytes, total;
};

Layout layout(long long B, long long npx, bool median) {
  Layout L;
  size_t off = 0;
  L.queue = off;
  off += 256;
  L.ctl = off;
  off = align_up(off + sizeof(ViewCtl) * (size_t)B, 256);
  L.hist = off;
  off = align_up(off + sizeof(unsigned) * NB * (size_t)B, 256);
  L.hist2 = off;
  off = align_up(off + sizeof(unsigned) * 2 * NB2 * (size_t)RING, 256);
  L.zero_bytes = off;
  L.slots = off;
  off = align_up(off + sizeof(double) * 2 * NB2 * SLOTS * (size_t)RING, 256);
  L.cand = off;
  if (median)
    off = align_up(off + sizeof(double) * 3 * (size_t)((npx + 1) & ~1ll) * (size_t)(B < RING ? B : RING), 256);
  L.total = off;
  return L;
}

typedef void (*KernelFn)(Params);

template <bool FAST, int CH, bool F64>
int blocks_for() {
  static int cached = -1;
  if (cached < 0) {
    int n = 0;
    auto fn = edge_persistent_kernel<FAST, CH, F64>;
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(Smem)) != cudaSuccess)
      return 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, NT, sizeof(Smem)) != cudaSuccess)
      return 0;
    cached = n;
  }
  return cached;
}

template <bool FAST, int CH, bool F64>
void pick(KernelFn& fn, int& bps) {
  fn = edge_persistent_kernel<FAST, CH, F64>;
  bps = blocks_for<FAST, CH, F64>();
}

int launch(Params& p, void* ws, size_t ws_bytes, cudaStream_t stream) {
  const bool median = p.median != 0;
  Layout L = layout(p.B, p.npx, median);
  if (ws_bytes < L.total || ws == nullptr) return IGS_ERR_WORKSPACE;
  char* w = (char*)ws;
  p.sched = (unsigned*)(w + L.queue);
  p.ctl = (ViewCtl*)(w + L.ctl);
  p.hist = (unsigned*)(w + L.hist);
  p.hist2 = (unsigned*)(w + L.hist2);
  p.cand = (double*)(w + L.cand);
  p.slot = 3 * ((p.npx + 1) & ~1ll);  // even: every ring slot starts 16-byte aligned
  p.slots = (double*)(w + L.slots);
  IGS_CUDA_TRY(cudaMemsetAsync(w, 0, L.zero_bytes, stream));  // sched, ctl, hist, hist2
  p.kgray[0] = 0.299;
  p.kgray[1] = 0.587;
  p.kgray[2] = 0.114;
  p.ktan = 0.41421356237309503;
  p.ktol = 1e-12;
  if (p.mode == MODE_FUSED) {
    p.ncols = (int)((p.W + TWM - 1) / TWM);
    p.tw = (int)((p.W + p.ncols - 1) / p.ncols);
    // band height: 112 rows, unless the batch is too small to give the grid ~1.5 band tasks
    // per CTA, then the tallest of 96 / 64 / 48 / 32 rows that does (measured on one view:
    // 0.134 ms at 128 rows, 0.090 ms at 32; four views: 0.187 -> 0.157 ms at 48)
    int bh = BAND_H_DEFAULT;
    const long long grid_est = 3LL * sm_count();
    for (int cand : {BAND_H_DEFAULT, 96, 64, 48, 32}) {
      bh = cand;
      const long long tasks = (long long)p.ncols * ((p.H + cand - 1) / cand) * p.B;
      if (2 * tasks >= 3 * grid_est) break;
    }
    if (const char* e = getenv("IGS_BAND_H"))  // tuning override, clamped to [SR, BAND_H]
      bh = atoi(e) < SR ? SR : (atoi(e) > BAND_H ? BAND_H : atoi(e));
    const int nbands = (int)((p.H + bh - 1) / bh);
    // equal bands, rounded up to whole sub-steps (a partial sub-step costs its barriers and
    // context work for a few rows): 822 rows -> 6 x 128 + 54 instead of 7 x 118
    const int eq = (int)((p.H + nbands - 1) / nbands);
    p.band_h = ((eq + SR - 1) / SR) * SR;
    if (p.band_h > BAND_H) p.band_h = BAND_H;
    p.TE = p.ncols * (int)((p.H + p.band_h - 1) / p.band_h);
  } else {
    p.TE = (int)((p.npx + CHUNK - 1) / CHUNK);
  }
  // fused mode: survivor entries per collect / apply task (16384; small batches use shorter
  // tasks so the median passes of a few views spread over more CTAs)
  p.chunk = CHUNK;
  if (p.mode == MODE_FUSED && p.B <= 8) p.chunk = p.B == 1 ? CHUNK / 8 : CHUNK / 4;  // one
                                                // view: 2048 (0.076 -> 0.0745 ms measured)
  if (const char* e = getenv("IGS_CHUNK")) {  // tuning override: a multiple of APIECE
    const int c = atoi(e);
    if (c >= APIECE && c <= CHUNK && c % APIECE == 0) p.chunk = c;
  }
  if (p.mode != MODE_FUSED) p.chunk = CHUNK;
  p.TC = median ? (int)((p.npx + p.chunk - 1) / p.chunk) : 0;
  p.TA = p.TC;
  const bool fast = p.sym && !p.skip;
  KernelFn fn = nullptr;
  int bps = 0;
  if (p.mode == MODE_MEDIAN_ONLY) pick<true, 1, true>(fn, bps);
  else if (p.channels == 3 && p.in_f64) fast ? pick<true, 3, true>(fn, bps) : pick<false, 3, true>(fn, bps);
  else if (p.channels == 3) fast ? pick<true, 3, false>(fn, bps) : pick<false, 3, false>(fn, bps);
  else if (p.in_f64) fast ? pick<true, 1, true>(fn, bps) : pick<false, 1, true>(fn, bps);
  else fast ? pick<true, 1, false>(fn, bps) : pick<false, 1, false>(fn, bps);
  if (bps <= 0) return IGS_ERR_CUDA;
  long long grid = (long long)bps * sm_count();
  // enough E work in flight to occupy the grid, bounded by the candidate ring
  {
    // as many views in flight as the candidate ring allows: the collect / select / apply
    // latency of a view is hidden behind later views' E work (measured: more is faster)
    long long a = RING - 2;
    if (const char* e = getenv("IGS_AHEAD")) a = atoi(e);
    p.ahead = (int)(a < 2 ? 2 : (a > RING - 2 ? RING - 2 : a));
  }
  const long long total_tasks = (long long)(p.TE + p.TC + p.TA) * p.B;
  if (grid > total_tasks) grid = total_tasks;
  if (grid < 1) grid = 1;
  void* args[] = {&p};
  IGS_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)fn, dim3((unsigned)grid), dim3(NT), args,
                                           sizeof(Smem), stream));
  return IGS_OK;
}

void set_weights(Params& p, const double* w25) {
  memcpy(p.w25, w25, sizeof(p.w25));
  p.keep_mask = 0;
  for (int t = 0; t < 25; ++t)
    if (fabs(w25[t]) > 2.220446049250313e-16) p.keep_mask |= 1u << t;
  p.skip = p.keep_mask != 0x1ffffffu;
  bool sym = true;
  for (int i = 0; i < 5 && sym; ++i)
    for (int j = 0; j < 5; ++j) {
      int a = i < 2 ? 2 - i : i - 2, b = j < 2 ? 2 - j : j - 2;
      double ref = w25[(2 + a) * 5 + (2 + b)];
      // bitwise equality across the dihedral group
      if (memcmp(&ref, &w25[i * 5 + j], sizeof(double)) != 0) sym = false;
    }
  p.sym = sym;
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) p.w6[a][b] = w25[(2 + a) * 5 + (2 + b)];
}

// ---------------------------------------------------------------- stage kernels
__global__ void gray_kernel(const void* img, int in_f64, long long n, double* gray) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double r, g, b;
  if (in_f64) {
    const double* s = (const double*)img + 3 * i;
    r = s[0]; g = s[1]; b = s[2];
  } else {
    const float* s = (const float*)img + 3 * i;
    r = s[0]; g = s[1]; b = s[2];
  }
  gray[i] = np_clip01(((0.299 * r) + (0.587 * g)) + (0.114 * b));
}

struct W25 { double w[25]; unsigned keep; };

__global__ void blur_kernel(const double* in, long long B, long long H, long long W, W25 w,
                            double* out) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= B * H * W) return;
  long long v = i / (H * W), r = i - v * H * W, y = r / W, x = r - y * W;
  const double* src = in + v * H * W;
  double acc = 0.0;
  for (int a = 0; a < 5; ++a) {
    long long yy = clampi(y + a - 2, 0, H - 1);
    for (int b = 0; b < 5; ++b) {
      long long xx = clampi(x + b - 2, 0, W - 1);
      if ((w.keep >> (a * 5 + b)) & 1u) acc = acc + src[yy * W + xx] * w.w[a * 5 + b];
    }
  }
  out[i] = np_clip01(acc);
}

__global__ void sobel_kernel(const double* in, long long B, long long H, long long W,
                             double* mag, double* ori) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= B * H * W) return;
  long long v = i / (H * W), r = i - v * H * W, y = r / W, x = r - y * W;
  const double* s = in + v * H * W;
  long long ym = clampi(y - 1, 0, H - 1), yp = clampi(y + 1, 0, H - 1);
  long long xm = clampi(x - 1, 0, W - 1), xp = clampi(x + 1, 0, W - 1);
  double b00 = s[ym * W + xm], b01 = s[ym * W + x], b02 = s[ym * W + xp];
  double b10 = s[y * W + xm], b12 = s[y * W + xp];
  double b20 = s[yp * W + xm], b21 = s[yp * W + x], b22 = s[yp * W + xp];
  double gx = 0.0;
  gx = gx + b00 * -1.0;
  gx = gx + b02 * 1.0;
  gx = gx + b10 * -2.0;
  gx = gx + b12 * 2.0;
  gx = gx + b20 * -1.0;
  gx = gx + b22 * 1.0;
  double gy = 0.0;
  gy = gy + b00 * -1.0;
  gy = gy + b01 * -2.0;
  gy = gy + b02 * -1.0;
  gy = gy + b20 * 1.0;
  gy = gy + b21 * 2.0;
  gy = gy + b22 * 1.0;
  mag[i] = hypot_glibc(gx, gy);
  ori[i] = np_mod(atan2(gy, gx), 3.141592653589793);
}

__global__ void nms_kernel(const double* mag, const double* ori, long long B, long long H,
                           long long W, double* out) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= B * H * W) return;
  long long v = i / (H * W), r = i - v * H * W, y = r / W, x = r - y * W;
  const double* m = mag + v * H * W;
  int bn = np_orientation_bin(ori[i]);
  int pa = bn == 0 ? 0 : -1, pb = bn == 0 ? -1 : (bn == 1 ? -1 : (bn == 2 ? 0 : 1));
  auto at = [&](long long yy, long long xx) -> double {
    return (yy >= 0 && yy < H && xx >= 0 && xx < W) ? m[yy * W + xx] : 0.0;
  };
  double c = m[y * W + x];
  bool keep = (c > at(y + pa, x + pb)) && (c >= at(y - pa, x - pb));
  out[i] = keep ? c : 0.0;
}

}  // namespace edge
}  // namespace igs

using namespace igs;

extern "C" {

int igs_edge_workspace_bytes(int64_t batch, int64_t height, int64_t width, int flags,
                             size_t* bytes) {
  if (!bytes || batch < 0 || height < 0 || width < 0) return IGS_ERR_ARGUMENT;
  *bytes = edge::layout(batch, height * width, !(flags & IGS_EDGE_NO_MEDIAN)).total;
  return IGS_OK;
}

int igs_edge_importance(const void* image, int in_dtype, int channels, int64_t batch,
                        int64_t height, int64_t width, const double* blur_w25, int flags,
                        double* out, void* workspace, size_t workspace_bytes, void* stream) {
  if (!image || !out || !blur_w25) return IGS_ERR_ARGUMENT;
  if (channels != 1 && channels != 3) return IGS_ERR_ARGUMENT;
  if (in_dtype != IGS_F32 && in_dtype != IGS_F64) return IGS_ERR_ARGUMENT;
  if (height < 3 || width < 3 || batch < 0) return IGS_ERR_ARGUMENT;
  if (batch == 0) return IGS_OK;
  if (height * width > (1ll << 31)) return IGS_ERR_UNSUPPORTED;
  edge::Params p;
  memset(&p, 0, sizeof(p));
  p.img = image;
  p.in_f64 = in_dtype == IGS_F64;
  p.channels = channels;
  p.mode = edge::MODE_FUSED;
  p.nms = !(flags & IGS_EDGE_NO_NMS);
  p.median = !(flags & IGS_EDGE_NO_MEDIAN);
  p.B = batch;
  p.H = height;
  p.W = width;
  p.npx = height * width;
  p.out = out;
  edge::set_weights(p, blur_w25);
  return edge::launch(p, workspace, workspace_bytes, (cudaStream_t)stream);
}

// Debug: trace every task of subsequent igs_edge_importance launches into buf (device memory,
// capacity records of 32 bytes); buf == NULL disables.  Returns the records written so far
// (of the previous launches) in *written when non-NULL.
int igs_debug_edge_trace(void* buf, int64_t capacity, int64_t* written) {
  if (written) {
    unsigned long long n = 0;
    IGS_CUDA_TRY(cudaMemcpyFromSymbol(&n, edge::g_trace_n, sizeof(n)));
    *written = (int64_t)n;
  }
  edge::TraceRec* p = (edge::TraceRec*)buf;
  unsigned long long cap = buf ? (unsigned long long)capacity : 0ull, zero = 0;
  IGS_CUDA_TRY(cudaMemcpyToSymbol(edge::g_trace, &p, sizeof(p)));
  IGS_CUDA_TRY(cudaMemcpyToSymbol(edge::g_trace_cap, &cap, sizeof(cap)));
  IGS_CUDA_TRY(cudaMemcpyToSymbol(edge::g_trace_n, &zero, sizeof(zero)));
  return IGS_OK;
}

// Debug (library built with -DIGS_PHASE_PROF): per-phase nanoseconds of the band sub-steps
// summed over blocks since the last reset: gray, blur, Sobel, NMS decide, NMS finish.
int igs_debug_edge_phases(uint64_t* out8, int reset) {
#ifdef IGS_PHASE_PROF
  unsigned long long h[8];
  IGS_CUDA_TRY(cudaMemcpyFromSymbol(h, edge::g_phase_ns, sizeof(h)));
  if (out8)
    for (int i = 0; i < 8; ++i) out8[i] = h[i];
  if (reset) {
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    IGS_CUDA_TRY(cudaMemcpyToSymbol(edge::g_phase_ns, z, sizeof(z)));
  }
  return IGS_OK;
#else
  (void)out8;
  (void)reset;
  return IGS_ERR_UNSUPPORTED;
#endif
}

int igs_median_normalize(const double* in, int64_t batch, int64_t n, double* out,
                         double* medians, void* workspace, size_t workspace_bytes,
                         void* stream) {
  if (!in || !out || batch < 0 || n < 0) return IGS_ERR_ARGUMENT;
  if (batch == 0 || n == 0) return IGS_OK;
  if (n > (1ll << 31)) return IGS_ERR_UNSUPPORTED;
  edge::Params p;
  memset(&p, 0, sizeof(p));
  p.img = in;
  p.in_f64 = 1;
  p.channels = 1;
  p.mode = edge::MODE_MEDIAN_ONLY;
  p.nms = 0;
  p.median = 1;
  p.B = batch;
  p.H = 1;
  p.W = n;
  p.npx = n;
  p.out = out;
  p.medians = medians;
  return edge::launch(p, workspace, workspace_bytes, (cudaStream_t)stream);
}

int igs_to_grayscale(const void* image, int in_dtype, int64_t batch, int64_t height,
                     int64_t width, double* gray, void* stream) {
  if (!image || !gray || batch < 0 || height < 1 || width < 1) return IGS_ERR_ARGUMENT;
  long long n = batch * height * width;
  if (n == 0) return IGS_OK;
  edge::gray_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      image, in_dtype == IGS_F64, n, gray);
  IGS_LAUNCH_CHECK();
  return IGS_OK;
}

int igs_gaussian_blur_5x5(const double* gray, int64_t batch, int64_t height, int64_t width,
                          const double* blur_w25, double* out, void* stream) {
  if (!gray || !out || !blur_w25 || batch < 0 || height < 1 || width < 1) return IGS_ERR_ARGUMENT;
  long long n = batch * height * width;
  if (n == 0) return IGS_OK;
  edge::W25 w;
  memcpy(w.w, blur_w25, sizeof(w.w));
  w.keep = 0;
  for (int t = 0; t < 25; ++t)
    if (fabs(blur_w25[t]) > 2.220446049250313e-16) w.keep |= 1u << t;
  edge::blur_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      gray, batch, height, width, w, out);
  IGS_LAUNCH_CHECK();
  return IGS_OK;
}

int igs_sobel_gradients(const double* gray, int64_t batch, int64_t height, int64_t width,
                        double* magnitude, double* orientation, void* stream) {
  if (!gray || !magnitude || !orientation || batch < 0 || height < 3 || width < 3)
    return IGS_ERR_ARGUMENT;
  long long n = batch * height * width;
  if (n == 0) return IGS_OK;
  edge::sobel_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      gray, batch, height, width, magnitude, orientation);
  IGS_LAUNCH_CHECK();
  return IGS_OK;
}

int igs_nms_thin(const double* magnitude, const double* orientation, int64_t batch,
                 int64_t height, int64_t width, double* out, void* stream) {
  if (!magnitude || !orientation || !out || batch < 0 || height < 1 || width < 1)
    return IGS_ERR_ARGUMENT;
  long long n = batch * height * width;
  if (n == 0) return IGS_OK;
  edge::nms_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      magnitude, orientation, batch, height, width, out);
  IGS_LAUNCH_CHECK();
  return IGS_OK;
}

}  // extern "C"
