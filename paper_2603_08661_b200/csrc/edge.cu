// Edge-importance map on sm_100a: one persistent, task-queued launch per batch of views.
//
// Replaces splitkit.edge_pipeline.importance_pipeline and its stages
// (/root/reference/pkg/src/splitkit/edge_pipeline.py:42-135).
//
// Task kinds, handed out in queue order by an atomic counter (every task
// depends only on tasks handed out earlier, and the grid is co-resident, so
// spinning on a dependency always terminates):
//   E(v,t)  fused tile: gray -> 5x5 blur -> Sobel -> |g| + direction bin -> NMS
//           for a TH x TW output tile staged in shared memory with a 4-pixel
//           halo; writes the thinned map and merges a per-view histogram of the
//           positive survivors.  The last E task of a view locates the median
//           histogram bin(s).                                 (:42-114, :123)
//   C(v,c)  collect: gathers the values falling in the median bin(s) into a
//           candidate buffer.  The last C task radix-selects the exact order
//           statistic(s) -> median m (np.median: (a+b)/2 for an even count). (:124)
//   A(v,c)  apply: out = min(v / (2 m), 1) in place.                   (:125)
// Queue order per step s: E(s) tiles, C(s-LAG1) chunks, A(s-LAG2) chunks, so
// at most LAG2+1 views' thinned maps are live and they stay L2-resident
// between E, C and A (the final map is written back to HBM once).
//
// Arithmetic: float64 in scipy's order (see oracle/edge.py): taps summed in
// row-major order from 0.0 with separately rounded multiply and add; glibc's
// hypot; the NMS direction bin from exact comparisons against tan(pi/8) with a
// fallback to numpy's floor((mod(atan2)+pi/8)/(pi/4)) within 1e-12 rad of a
// boundary.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "igs_common.cuh"

namespace igs {
namespace edge {

constexpr int TH = 32, TW = 60;              // output tile
constexpr int MH = TH + 2, MW = TW + 2;      // gradient magnitude region (NMS halo 1)
constexpr int BH = TH + 4, BW = TW + 4;      // blurred region (Sobel halo 1)
constexpr int GH = TH + 8, GW = TW + 8;      // gray region (blur halo 2)
constexpr int NT = 256;                      // threads per block
constexpr int SB = 9;                        // blur strip height: BW x (BH/SB) = 256 strips
static_assert(BW * (BH / SB) == NT && BH % SB == 0, "blur strips must cover the block");
static_assert(MH * MW <= GH * GW, "magnitude aliases the gray buffer");

constexpr int NB = 2048;                     // median histogram: 16 bins per octave
constexpr int HIST_BASE = 14768;             // (bits>>48) of 2^-100; bins cover [2^-100, 2^28)
constexpr int CHUNK = 32768;                 // pixels per collect/apply task
constexpr int LAG1 = 2, LAG2 = 3;            // queue lags of C and A behind E
constexpr int RING = LAG2 + 3;               // candidate buffers in flight

enum Mode { MODE_FUSED = 0, MODE_MEDIAN_ONLY = 1 };

struct ViewCtl {            // per-view control block, zeroed before launch
  unsigned tiles_done;      // E tasks finished
  unsigned binfound;        // 1 once the median bins are known
  unsigned collect_done;    // C tasks finished
  unsigned select_done;     // 1 once denom is published
  unsigned cnt1, cnt2;      // candidate append counters (front / back)
  int b1, b2;               // median bins of ranks k1, k2
  unsigned long long r1, r2;// ranks within those bins
  unsigned long long npos;  // positive count
  double denom;             // 2 * median
  double median;
  unsigned pad[14];
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
  int tiles_x, tiles_y, TE, TC, TA;
  long long total_tasks;
  // workspace
  unsigned long long* queue;
  ViewCtl* ctl;
  unsigned* hist;           // (B, NB)
  double* cand;             // (RING, npx)
};

struct __align__(16) Smem {
  double g[GH * GW];        // gray, then gradient magnitude
  double b[BH * BW];        // blurred
  uint8_t bin[TH * TW];     // NMS direction bins of the output tile
  unsigned hist[NB];
  unsigned warp_sums[32];
  long long task;
  int flag;
  int ivals[4];
};

__device__ __forceinline__ int clampi(long long v, long long lo, long long hi) {
  return (int)(v < lo ? lo : (v > hi ? hi : v));
}

__device__ __forceinline__ int hist_bin(double v) {
  long long hb = (long long)((unsigned long long)__double_as_longlong(v) >> 48) - HIST_BASE;
  return hb < 0 ? 0 : (hb >= NB ? NB - 1 : (int)hb);
}

__device__ __forceinline__ double load_px(const Params& p, long long idx) {
  return p.in_f64 ? __ldg((const double*)p.img + idx) : (double)__ldg((const float*)p.img + idx);
}

// ---------------------------------------------------------------- E: fused tile
template <bool FAST>
__device__ void run_tile(const Params& p, Smem& s, int v, int t) {
  const int tid = threadIdx.x;
  const long long H = p.H, W = p.W;
  const int ty = t / p.tiles_x, tx = t - ty * p.tiles_x;
  const long long y0 = (long long)ty * TH, x0 = (long long)tx * TW;
  const long long vbase = (long long)v * p.npx;

  // Phase A: gray over the GH x GW region, stored at clamped coordinates (mode="nearest").
  for (int i = tid; i < GH * GW; i += NT) {
    int u = i / GW, c = i - u * GW;
    int y = clampi(y0 - 4 + u, 0, H - 1), x = clampi(x0 - 4 + c, 0, W - 1);
    long long pix = vbase + (long long)y * W + x;
    double g;
    if (p.channels == 3) {
      double r = load_px(p, pix * 3), gg = load_px(p, pix * 3 + 1), bb = load_px(p, pix * 3 + 2);
      g = np_clip01(((0.299 * r) + (0.587 * gg)) + (0.114 * bb));
    } else {
      g = load_px(p, pix);
    }
    s.g[i] = g;
  }
  __syncthreads();

  // Phase B: 5x5 blur in vertical strips of SB outputs per thread.  Input rows stream
  // top to bottom, so every output still accumulates its taps in row-major order.  With
  // dihedrally symmetric weights (FAST) rows r-o and r-(4-o) share one product.
  {
    const int c = tid % BW, u0 = (tid / BW) * SB;
    double acc[SB];
#pragma unroll
    for (int o = 0; o < SB; ++o) acc[o] = 0.0;
#pragma unroll
    for (int r = 0; r < SB + 4; ++r) {
      double xv[5];
#pragma unroll
      for (int dj = 0; dj < 5; ++dj) xv[dj] = s.g[(u0 + r) * GW + c + dj];
#pragma unroll
      for (int o = 0; o < SB; ++o) {
        const int di = r - o;
        if (di < 0 || di > 4) continue;
#pragma unroll
        for (int dj = 0; dj < 5; ++dj) {
          const int t25 = di * 5 + dj;
          if (FAST) {
            acc[o] = acc[o] + xv[dj] * p.w6[di < 2 ? 2 - di : di - 2][dj < 2 ? 2 - dj : dj - 2];
          } else if ((p.keep_mask >> t25) & 1u) {
            acc[o] = acc[o] + xv[dj] * p.w25[t25];
          }
        }
      }
    }
#pragma unroll
    for (int o = 0; o < SB; ++o) s.b[(u0 + o) * BW + c] = np_clip01(acc[o]);
  }
  __syncthreads();
  // Border tiles: out-of-image blurred cells take the value of the clamped in-image cell.
  if (y0 < 2 || x0 < 2 || y0 + TH + 2 > H || x0 + TW + 2 > W) {
    constexpr int FIX = BH * BW / NT;
    static_assert(BH * BW % NT == 0, "fix-up covers the blurred region exactly");
    double val[FIX];
    bool fix[FIX];
#pragma unroll
    for (int k = 0; k < FIX; ++k) {
      int i = tid + k * NT, u = i / BW, c = i - u * BW;
      long long y = y0 - 2 + u, x = x0 - 2 + c;
      long long cy = y < 0 ? 0 : (y >= H ? H - 1 : y), cx = x < 0 ? 0 : (x >= W ? W - 1 : x);
      fix[k] = (cy != y) || (cx != x);
      val[k] = fix[k] ? s.b[(int)(cy - (y0 - 2)) * BW + (int)(cx - (x0 - 2))] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < FIX; ++k)
      if (fix[k]) s.b[tid + k * NT] = val[k];
    __syncthreads();
  }

  // Phase C: Sobel (NI_Correlate tap order, zero taps skipped), glibc hypot, direction bin.
  for (int i = tid; i < MH * MW; i += NT) {
    int u = i / MW, c = i - u * MW;
    long long y = y0 - 1 + u, x = x0 - 1 + c;
    double m = 0.0;  // out-of-image neighbours count as 0 for NMS (edge_pipeline.py:97)
    if (y >= 0 && y < H && x >= 0 && x < W) {
      const double* b = &s.b[u * BW + c];
      double b00 = b[0], b01 = b[1], b02 = b[2];
      double b10 = b[BW], b12 = b[BW + 2];
      double b20 = b[2 * BW], b21 = b[2 * BW + 1], b22 = b[2 * BW + 2];
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
      m = hypot_glibc(gx, gy);
      if (p.nms && u >= 1 && u <= TH && c >= 1 && c <= TW)
        s.bin[(u - 1) * TW + (c - 1)] = (uint8_t)gradient_bin(gx, gy);
    }
    s.g[i] = m;  // gray is dead after phase B
  }
  __syncthreads();

  // Phase D: NMS (keep iff m > prev and m >= next), store, histogram the survivors.
  for (int i = tid; i < TH * TW; i += NT) {
    int a = i / TW, c = i - a * TW;
    long long y = y0 + a, x = x0 + c;
    if (y >= H || x >= W) continue;
    const double* mp = &s.g[(a + 1) * MW + (c + 1)];
    double m = *mp, outv = m;
    if (p.nms) {
      int bn = s.bin[i];
      int po = bn == 0 ? -1 : (bn == 1 ? -MW - 1 : (bn == 2 ? -MW : -MW + 1));
      bool keep = (m > mp[po]) && (m >= mp[-po]);
      outv = keep ? m : 0.0;
    }
    p.out[vbase + y * W + x] = outv;
    if (p.median && outv > 0.0) atomicAdd(&s.hist[hist_bin(outv)], 1u);
  }
}

// ------------------------------------------------ histogram-only tile (median-only mode)
__device__ void run_hist_chunk(const Params& p, Smem& s, int v, int c) {
  const long long lo = (long long)c * CHUNK, hi = min(lo + (long long)CHUNK, p.npx);
  const double* src = (const double*)p.img + (long long)v * p.npx;
  for (long long i = lo + threadIdx.x; i < hi; i += NT) {
    double x = __ldg(src + i);
    if (x > 0.0) atomicAdd(&s.hist[hist_bin(x)], 1u);
  }
}

// Flush the block histogram into the view's global histogram and clear it.
__device__ void flush_hist(const Params& p, Smem& s, int v) {
  __syncthreads();
  unsigned* gh = p.hist + (long long)v * NB;
  for (int i = threadIdx.x; i < NB; i += NT) {
    unsigned h = s.hist[i];
    if (h) {
      atomicAdd(&gh[i], h);
      s.hist[i] = 0;
    }
  }
}

// Last E task of a view: locate the bins holding ranks k1 = (n-1)/2 and k2 = n/2.
__device__ void find_median_bins(const Params& p, Smem& s, int v) {
  const unsigned* gh = p.hist + (long long)v * NB;
  constexpr int PER = NB / NT;
  unsigned h[PER], local = 0;
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    h[k] = __ldcg(&gh[threadIdx.x * PER + k]);
    local += h[k];
  }
  unsigned total;
  unsigned before = block_exclusive_scan(local, s.warp_sums, &total);
  ViewCtl& ctl = p.ctl[v];
  if (total == 0) {
    if (threadIdx.x == 0) {
      ctl.npos = 0;
      ctl.median = 1.0;
      ctl.denom = 2.0 * 1.0;
      if (p.medians) p.medians[v] = 1.0;
    }
  } else {
    const unsigned long long k1 = (total - 1) / 2, k2 = total / 2;
    unsigned long long cum = before;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const unsigned long long nxt = cum + h[k];
      if (h[k] && k1 >= cum && k1 < nxt) {
        ctl.b1 = threadIdx.x * PER + k;
        ctl.r1 = k1 - cum;
      }
      if (h[k] && k2 >= cum && k2 < nxt) {
        ctl.b2 = threadIdx.x * PER + k;
        ctl.r2 = k2 - cum;
      }
      cum = nxt;
    }
    if (threadIdx.x == 0) ctl.npos = total;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    if (total == 0) atomicExch(&ctl.select_done, 1u);
    atomicExch(&ctl.binfound, 1u);
  }
}

// ------------------------------------------------------------- C: collect candidates
__device__ void run_collect(const Params& p, Smem& s, int v, int c) {
  ViewCtl& ctl = p.ctl[v];
  if (threadIdx.x == 0) {
    spin_until_geq(&ctl.binfound, 1u);
    if (v >= RING) spin_until_geq(&p.ctl[v - RING].select_done, 1u);  // ring slot free
    s.ivals[0] = __ldcg(&ctl.npos) ? 1 : 0;
    s.ivals[1] = __ldcg(&ctl.b1);
    s.ivals[2] = __ldcg(&ctl.b2);
  }
  __syncthreads();
  if (s.ivals[0]) {
    const int b1 = s.ivals[1], b2 = s.ivals[2];
    const double* src = (p.mode == MODE_FUSED) ? p.out + (long long)v * p.npx
                                               : (const double*)p.img + (long long)v * p.npx;
    double* cand = p.cand + (long long)(v % RING) * p.npx;
    const long long lo = (long long)c * CHUNK, hi = min(lo + (long long)CHUNK, p.npx);
    for (long long base = lo; base < hi; base += NT) {
      long long i = base + threadIdx.x;
      double x = 0.0;
      if (i < hi) x = __ldcg(src + i);
      int hb = x > 0.0 ? hist_bin(x) : -1;
      bool f1 = hb == b1, f2 = (hb == b2) && (b2 != b1);
      unsigned m1 = __ballot_sync(0xffffffffu, f1), m2 = __ballot_sync(0xffffffffu, f2);
      if (m1) {
        unsigned slot = 0;
        int leader = __ffs(m1) - 1;
        if ((int)lane_id() == leader) slot = atomicAdd(&ctl.cnt1, __popc(m1));
        slot = __shfl_sync(0xffffffffu, slot, leader);
        if (f1) cand[slot + __popc(m1 & lanemask_lt())] = x;
      }
      if (m2) {
        unsigned slot = 0;
        int leader = __ffs(m2) - 1;
        if ((int)lane_id() == leader) slot = atomicAdd(&ctl.cnt2, __popc(m2));
        slot = __shfl_sync(0xffffffffu, slot, leader);
        if (f2) cand[p.npx - 1 - (slot + __popc(m2 & lanemask_lt()))] = x;
      }
    }
  }
}

// Block-wide radix select: bits of the rank-th smallest among cand[0..n) (positive doubles,
// so unsigned bit order == value order).  `dir` -1 reads the array backwards from `cand`.
__device__ unsigned long long block_radix_select(Smem& s, const double* cand, long long n,
                                                 int dir, unsigned long long rank) {
  unsigned long long prefix = 0, pmask = 0;
  unsigned* h = s.hist;  // reuse (cleared on entry and exit)
  for (int pass = 0; pass < 6; ++pass) {
    const int shift = pass < 5 ? 53 - 11 * pass : 0;
    const unsigned dmask = pass < 5 ? 2047u : 511u;
    const int nb = 2048;
    for (int i = threadIdx.x; i < nb; i += NT) h[i] = 0;
    __syncthreads();
    for (long long i = threadIdx.x; i < n; i += NT) {
      unsigned long long bits = (unsigned long long)__double_as_longlong(__ldcg(cand + dir * i));
      if ((bits & pmask) == prefix) atomicAdd(&h[(bits >> shift) & dmask], 1u);
    }
    __syncthreads();
    // find the digit: thread k owns bins [8k, 8k+8)
    unsigned loc[8], sum = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      loc[k] = h[threadIdx.x * 8 + k];
      sum += loc[k];
    }
    unsigned total;
    unsigned before = block_exclusive_scan(sum, s.warp_sums, &total);
    unsigned long long cum = before;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (loc[k] && rank >= cum && rank < cum + loc[k]) {
        s.ivals[0] = threadIdx.x * 8 + k;
        s.ivals[1] = (int)(rank - cum);
      }
      cum += loc[k];
    }
    __syncthreads();
    const unsigned long long d = (unsigned)s.ivals[0];
    rank = (unsigned)s.ivals[1];
    prefix |= d << shift;
    pmask |= (unsigned long long)dmask << shift;
    __syncthreads();
  }
  for (int i = threadIdx.x; i < NB; i += NT) s.hist[i] = 0;
  __syncthreads();
  return prefix;
}

__device__ void run_select(const Params& p, Smem& s, int v) {
  ViewCtl& ctl = p.ctl[v];
  const double* cand = p.cand + (long long)(v % RING) * p.npx;
  const unsigned n1 = __ldcg(&ctl.cnt1), n2 = __ldcg(&ctl.cnt2);
  const unsigned long long r1 = __ldcg(&ctl.r1), r2 = __ldcg(&ctl.r2);
  const int b1 = __ldcg(&ctl.b1), b2 = __ldcg(&ctl.b2);
  double a = __longlong_as_double(block_radix_select(s, cand, n1, 1, r1));
  double m = a;
  const unsigned long long npos = __ldcg(&ctl.npos);
  if ((npos & 1ull) == 0) {
    double b = (b2 == b1) ? __longlong_as_double(block_radix_select(s, cand, n1, 1, r2))
                          : __longlong_as_double(
                                block_radix_select(s, cand + p.npx - 1, n2, -1, r2));
    m = (a + b) / 2.0;
  }
  if (threadIdx.x == 0) {
    ctl.median = m;
    ctl.denom = 2.0 * m;
    if (p.medians) p.medians[v] = m;
    __threadfence();
    atomicExch(&ctl.select_done, 1u);
  }
  __syncthreads();
}

// ------------------------------------------------------------------ A: apply
__device__ void run_apply(const Params& p, Smem& s, int v, int c) {
  ViewCtl& ctl = p.ctl[v];
  if (threadIdx.x == 0) {
    spin_until_geq(&ctl.select_done, 1u);
    s.ivals[0] = 0;
  }
  __syncthreads();
  const double denom = __ldcg(&ctl.denom);
  const double* src = (p.mode == MODE_FUSED) ? p.out + (long long)v * p.npx
                                             : (const double*)p.img + (long long)v * p.npx;
  double* dst = p.out + (long long)v * p.npx;
  const long long lo = (long long)c * CHUNK, hi = min(lo + (long long)CHUNK, p.npx);
  for (long long i = lo + threadIdx.x; i < hi; i += NT) {
    double x = __ldcg(src + i);
    __stcs(dst + i, np_min1(x / denom));
  }
}

// ------------------------------------------------------------- scheduler
__device__ __forceinline__ long long clampll(long long v, long long lo, long long hi) {
  return v < lo ? lo : (v > hi ? hi : v);
}
__device__ __forceinline__ long long step_start(const Params& p, long long st) {
  return (long long)p.TE * clampll(st, 0, p.B) + (long long)p.TC * clampll(st - LAG1, 0, p.B) +
         (long long)p.TA * clampll(st - LAG2, 0, p.B);
}

template <bool FAST>
__global__ void __launch_bounds__(NT) edge_persistent_kernel(Params p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& s = *reinterpret_cast<Smem*>(smem_raw);
  for (int i = threadIdx.x; i < NB; i += NT) s.hist[i] = 0;
  __syncthreads();
  const long long nsteps = p.B + (p.median ? LAG2 : 0);
  for (;;) {
    if (threadIdx.x == 0) s.task = (long long)atomicAdd(p.queue, 1ull);
    __syncthreads();
    const long long t = s.task;
    __syncthreads();
    if (t >= p.total_tasks) break;
    // locate the step: largest st with step_start(st) <= t
    long long lo = 0, hi = nsteps;  // step_start(hi) > t
    while (hi - lo > 1) {
      long long mid = (lo + hi) >> 1;
      if (step_start(p, mid) <= t) lo = mid; else hi = mid;
    }
    long long off = t - step_start(p, lo);
    const long long st = lo;
    if (st < p.B) {
      if (off < p.TE) {
        const int v = (int)st;
        if (p.mode == MODE_FUSED) run_tile<FAST>(p, s, v, (int)off);
        else run_hist_chunk(p, s, v, (int)off);
        if (p.median) {
          flush_hist(p, s, v);
          __threadfence();
          __syncthreads();
          if (threadIdx.x == 0) s.flag = (atomicAdd(&p.ctl[v].tiles_done, 1u) == (unsigned)p.TE - 1);
          __syncthreads();
          if (s.flag) {
            __threadfence();
            find_median_bins(p, s, v);
          }
        }
        __syncthreads();
        continue;
      }
      off -= p.TE;
    }
    if (st >= LAG1 && st < p.B + LAG1) {
      if (off < p.TC) {
        const int v = (int)(st - LAG1);
        run_collect(p, s, v, (int)off);
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0)
          s.flag = __ldcg(&p.ctl[v].npos) && (atomicAdd(&p.ctl[v].collect_done, 1u) == (unsigned)p.TC - 1);
        __syncthreads();
        if (s.flag) {
          __threadfence();
          run_select(p, s, v);
        }
        __syncthreads();
        continue;
      }
      off -= p.TC;
    }
    run_apply(p, s, (int)(st - LAG2), (int)off);
    __syncthreads();
  }
}

// ------------------------------------------------------------- host side
struct Layout {
  size_t ctl, hist, cand, queue, total;
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
  L.cand = off;
  if (median) off = align_up(off + sizeof(double) * (size_t)npx * (size_t)(B < RING ? B : RING), 256);
  L.total = off;
  return L;
}

template <bool FAST>
int blocks_per_sm() {
  static int cached = -1;
  if (cached < 0) {
    int n = 0;
    if (cudaFuncSetAttribute(edge_persistent_kernel<FAST>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(Smem)) != cudaSuccess)
      return 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, edge_persistent_kernel<FAST>, NT,
                                                      sizeof(Smem)) != cudaSuccess)
      return 0;
    cached = n;
  }
  return cached;
}

int launch(Params& p, void* ws, size_t ws_bytes, cudaStream_t stream) {
  const bool median = p.median != 0;
  Layout L = layout(p.B, p.npx, median);
  if (ws_bytes < L.total || ws == nullptr) return IGS_ERR_WORKSPACE;
  char* w = (char*)ws;
  p.queue = (unsigned long long*)(w + L.queue);
  p.ctl = (ViewCtl*)(w + L.ctl);
  p.hist = (unsigned*)(w + L.hist);
  p.cand = (double*)(w + L.cand);
  IGS_CUDA_TRY(cudaMemsetAsync(w, 0, L.cand, stream));  // queue, ctl, hist
  if (p.mode == MODE_FUSED) {
    p.tiles_x = (int)((p.W + TW - 1) / TW);
    p.tiles_y = (int)((p.H + TH - 1) / TH);
    p.TE = p.tiles_x * p.tiles_y;
  } else {
    p.TE = (int)((p.npx + CHUNK - 1) / CHUNK);
  }
  p.TC = median ? (int)((p.npx + CHUNK - 1) / CHUNK) : 0;
  p.TA = p.TC;
  p.total_tasks = (long long)(p.TE + p.TC + p.TA) * p.B;
  const bool fast = p.sym && !p.skip;
  int bps = fast ? blocks_per_sm<true>() : blocks_per_sm<false>();
  if (bps <= 0) return IGS_ERR_CUDA;
  long long grid = (long long)bps * sm_count();
  if (grid > p.total_tasks) grid = p.total_tasks;
  if (grid < 1) grid = 1;
  void* args[] = {&p};
  const void* fn = fast ? (const void*)edge_persistent_kernel<true>
                        : (const void*)edge_persistent_kernel<false>;
  IGS_CUDA_TRY(cudaLaunchCooperativeKernel(fn, dim3((unsigned)grid), dim3(NT), args, sizeof(Smem),
                                           stream));
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
