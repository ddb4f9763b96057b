// sgns_kernels.cu -- kernels and C ABI of the B200-native pSGNScc hot path.
//
// Kernels:
//   update_windows_kernel  packed windows (process_batch / microbench), one warp per window
//   drive_kernel           the fused, resumable epoch driver: one warp = one worker that
//                          walks its contiguous sentence range (trainer.py:217-311)
//   init_model_kernel      init_model (model.py:64-74), bit-identical
//   expand_slots_kernel    the reference's negative slot table (corpus.py:139-155)
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../../include/sgns_b200.h"
#include "sgns_device.cuh"
#include "sgns_fast.cuh"

// The library is built from this one file as five translation units compiled in parallel
// (SGNS_PART 0: C ABI + init/slot kernels, 1: update_windows, 2: static driver, 3: fast
// driver, 4: fast driver in warp pairs; see __graft_entry__.build_lib).  Without SGNS_PART it is a single unit.
// SGNS_ONLY_NS=n (experiment builds, tools/build_variant.py) instantiates the dynamic
// driver for one row width only.
#ifdef SGNS_PART
#define SGNS_HAS(n) (SGNS_PART == (n))
#else
#define SGNS_HAS(n) 1
#endif

namespace sgns {

constexpr int kMaxSentence = 1024;
constexpr int kMaxK1 = 32;

// slab pieces start on 32-byte boundaries: a 16-byte cp.async whose shared destination and
// global source differ in their offset within a 32-byte sector fetches one sector per lane
// (tools/probes/ldgsts_probe.cu), so staged rows keep the sector phase of the model rows
// whenever ld is a multiple of 32 bytes (model.py padded_ld)
__host__ __device__ inline int64_t round32(int64_t b) { return (b + 31) & ~int64_t(31); }

// shared-memory slab of one warp
struct Slab {
  int64_t rows, e, ids, roff, kept, off, hot, total;
};
// MODE_F2: float32 fast path (only the m input rows are staged); MODE_SMEM: all rows staged
// MODE_F2S: float32 8 < k1 <= 16, all rows staged; MODE_F2G: the same k1 in two register groups
// MODE_F2W: float32 8 < k1 <= 16 at d <= 128, one register group of up to 16 output rows
enum { MODE_SMEM = 0, MODE_F2 = 1, MODE_F2S = 2, MODE_F2G = 3, MODE_F2W = 4 };
// hot_rows: shared-memory hot-row sink rows of update_windows (H_in + H_out rows, see HotSink)
// ld: stride of the staged rows (ModelView::lds); hot_ld: of the hot-row sinks (the HBM stride)
__host__ __device__ inline Slab slab_layout(int mode, int64_t elem, int64_t ld, int mcap, int k1,
                                            int kept_cap, int hot_rows = 0, int64_t hot_ld = 0) {
  Slab s;
  s.rows = 0;
  const bool a_only = mode == MODE_F2 || mode == MODE_F2G || mode == MODE_F2W;  // only the input rows are staged
  s.e = round32((int64_t)(a_only ? mcap : mcap + k1) * ld * elem);
  // error rows: padded to 8 floats (F2, F2G per group), 16 (F2S), k1 (generic)
  const int erow = (mode == MODE_F2S || mode == MODE_F2W) ? 16 : mode == MODE_F2G ? 8 : (k1 > 8 ? k1 : 8);
  // F2 / F2G keep only the scaled errors; the other bodies keep raw and scaled
  s.ids = s.e + round32((int64_t)(a_only ? 1 : 2) * mcap * erow * elem);
  s.roff = s.ids + round32((int64_t)(mcap + k1) * 4);
  s.kept = s.roff + round32((int64_t)(mcap + k1) * 4);
  s.off = s.kept + round32((int64_t)kept_cap * 4);
  s.hot = s.off + round32((int64_t)kept_cap * 4);
  s.total = s.hot + round32((int64_t)hot_rows * hot_ld * elem);
  return s;
}
__host__ __device__ inline int64_t table_bytes(int64_t elem) { return round32(kSigBins * elem); }

template <typename T>
__device__ __forceinline__ void load_table(T *sig_s, const T *sig_g) {
  for (int i = threadIdx.x; i < kSigBins; i += blockDim.x) sig_s[i] = sig_g[i];
  __syncthreads();
}

template <typename T>
__device__ __forceinline__ void flush_loss(double loss, long long cells, double *dst_loss,
                                           int64_t *dst_cells, bool atomic, int lane) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    loss += __shfl_xor_sync(0xffffffffu, loss, o);
    cells += __shfl_xor_sync(0xffffffffu, cells, o);
  }
  if (lane == 0 && (cells != 0 || loss != 0.0)) {
    if (atomic) {
      atomicAdd(dst_loss, loss);
      atomicAdd(reinterpret_cast<unsigned long long *>(dst_cells), (unsigned long long)cells);
    } else {
      *dst_loss += loss;
      *dst_cells += cells;
    }
  }
}

// K1R == 6 is instantiated for k1 == 6 exactly (K = 5, the north-star shape); K1R == 8
// covers k1 <= 8 with predicates.
// HOT: see HotSink (sgns_device.cuh; float32 k1 <= 16 paths, snapshot mode); `hot` is
// the warp's sink, unused otherwise.
__host__ __device__ constexpr int hot_slots(int ns) { return ns > 0 ? ns : 1; }
template <typename T, int MODE, int NS, int NCH, int K1R, bool HOT = false>
__device__ __forceinline__ void run_window(const ModelView<T> &mv, const int *ids_s, uint32_t *roff_s,
                                           int m, int k1, T alpha, bool exact, const T *sig_s,
                                           bool want, double &loss, long long &cells, T *rows_s,
                                           T *e_s, int lane, HotSink<hot_slots(NS)> &hot) {
  if constexpr (MODE == MODE_F2) {
    for (int r = lane; r < m + k1; r += 32) roff_s[r] = (uint32_t)ids_s[r] * (uint32_t)mv.ld;
    __syncwarp();
    window_update_f2<NS, NCH, K1R, K1R == 6, HOT>(mv, roff_s, m, k1, alpha, exact, sig_s, want, loss,
                                                  cells, rows_s, e_s, lane, hot);
  } else if constexpr (MODE == MODE_F2G) {
    for (int r = lane; r < m + k1; r += 32) roff_s[r] = (uint32_t)ids_s[r] * (uint32_t)mv.ld;
    __syncwarp();
    window_update_f2g<NS, NCH, K1R, HOT>(mv, roff_s, m, k1, alpha, exact, sig_s, want, loss, cells,
                                         rows_s, e_s, lane, hot);
  } else if constexpr (MODE == MODE_F2W) {
    for (int r = lane; r < m + k1; r += 32) roff_s[r] = (uint32_t)ids_s[r] * (uint32_t)mv.ld;
    __syncwarp();
    window_update_f2w<NS, NCH, K1R, HOT>(mv, roff_s, m, k1, alpha, exact, sig_s, want, loss, cells,
                                         rows_s, e_s, lane, hot);
  } else if constexpr (MODE == MODE_F2S) {
    for (int r = lane; r < m + k1; r += 32) roff_s[r] = (uint32_t)ids_s[r] * (uint32_t)mv.ld;
    __syncwarp();
    window_update_f2s<NS, NCH, HOT>(mv, roff_s, m, k1, alpha, exact, sig_s, want, loss, cells,
                                    rows_s, e_s, lane, hot);
  } else {
    window_update<T, NCH>(mv, ids_s, m, k1, alpha, exact, sig_s, want, loss, cells,
                                    rows_s, e_s, lane);
  }
}

// ------------------------------------------------------- update_windows ----
template <typename T> struct UpdateArgs {
  ModelView<T> mv;
  int64_t vocab;
  const int32_t *in_off, *in_ids, *out_ids;
  int n_win, k1, mcap;
  const T *alpha, *sig;
  int exact, loss_every;
  double *loss_sum;
  int64_t *loss_cells;
  int32_t *error;
  int wpb;
  int hot_in, hot_out;  // shared-memory hot-row sink rows (HOT launches; hot_in 0: register sink)
  int mstage;           // input rows staged at once (= mcap; less: snapshot windows run in chunks)
};

// Register budget of update_windows_kernel: 128 (16 warps per SM) for the register-row
// float32 bodies, except 7-8 output rows of >= 5 slots (d > 256) -- F2G's first group always
// has 8 -- which get up to 168 (12-13 warps) instead of spilling, as the fast driver does;
// the all-staged generic body 255.
// d <= 128 with K + 1 <= 6 needs 87-103 registers depending on unrelated code around the body;
// capped at 96 it keeps 20 resident warps (configs[1] d = 100, K = 5: 0.51-0.56 at 16 warps ->
// 0.57-0.62 at 20), without spills.
template <int MODE, int NS, int K1R, bool DRIVER = false> struct UpdRegs {
  static constexpr int v = MODE == MODE_SMEM ? 255
                           : ((MODE == MODE_F2 && K1R >= 7) || MODE == MODE_F2G) && NS >= 5
                               ? SGNS_FAST_MAXNREG_WIDE
                               : (!DRIVER && MODE == MODE_F2 && NS <= 2 && K1R <= 6) ? 96 : 128;
};
template <typename T, int MODE, int NS, int NCH, int K1R, bool HOT>
__global__ void __maxnreg__((UpdRegs<MODE, NS, K1R>::v)) update_windows_kernel(UpdateArgs<T> p) {
  extern __shared__ __align__(128) unsigned char smem[];
  T *sig_s = reinterpret_cast<T *>(smem);
  load_table(sig_s, p.sig);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const Slab L = slab_layout(MODE, sizeof(T), p.mv.lds, p.mstage, p.k1, 0, HOT ? p.hot_in + p.hot_out : 0, p.mv.ld);
  unsigned char *base = smem + table_bytes(sizeof(T)) + (int64_t)warp * L.total;
  T *rows_s = reinterpret_cast<T *>(base + L.rows);
  T *e_s = reinterpret_cast<T *>(base + L.e);
  int *ids_s = reinterpret_cast<int *>(base + L.ids);
  uint32_t *roff_s = reinterpret_cast<uint32_t *>(base + L.roff);
  double loss = 0.0;
  long long cells = 0;
  HotSink<hot_slots(NS)> hot;
#pragma unroll
  for (int j = 0; j < hot_slots(NS); ++j) hot.reg[j] = make_float2(0.f, 0.f);
  hot.in_s = hot.out_s = nullptr;
  hot.in_lim = 1;  // register sink: row 0 of M_in
  hot.out_lim = 0;
  if constexpr (HOT) {
    float *hs = reinterpret_cast<float *>(base + L.hot);
    if (p.hot_in > 0) {
      hot.in_s = hs;
      hot.in_lim = (uint32_t)(p.hot_in * p.mv.ld);
    }
    if (p.hot_out > 0) {
      hot.out_s = hs + (int64_t)p.hot_in * p.mv.ld;
      hot.out_lim = (uint32_t)(p.hot_out * p.mv.ld);
    }
    for (int64_t q = lane; q < (int64_t)(p.hot_in + p.hot_out) * p.mv.ld; q += 32) hs[q] = 0.f;
    __syncwarp();
  }
  const int step = gridDim.x * p.wpb;
  for (int w = blockIdx.x * p.wpb + warp; w < p.n_win; w += step) {
    const int lo = p.in_off[w], hi = p.in_off[w + 1];
    const int m = hi - lo;
    if (m < 1 || m > p.mcap) {
      if (lane == 0 && p.error) atomicExch(p.error, 1);
      continue;
    }
    const bool want = p.loss_every > 0 && (w % p.loss_every) == 0;
    // mstage < mcap (snapshot mode only, see launch_update_t): the window runs as chunks of
    // its inputs against the same outputs -- every gradient comes from the snapshot, so the
    // chunks are independent and their dC parts add up
    for (int c0 = 0; c0 < m; c0 += p.mstage) {
      const int mc = min(p.mstage, m - c0);
      for (int r = lane; r < mc + p.k1; r += 32)
        ids_s[r] = r < mc ? p.in_ids[lo + c0 + r] : p.out_ids[(int64_t)w * p.k1 + (r - mc)];
      __syncwarp();
      run_window<T, MODE, NS, NCH, K1R, HOT>(p.mv, ids_s, roff_s, mc, p.k1, p.alpha[w], p.exact != 0,
                                             sig_s, want, loss, cells, rows_s, e_s, lane, hot);
      __syncwarp();
    }
  }

  if constexpr (HOT && (MODE == MODE_F2 || MODE == MODE_F2S || MODE == MODE_F2G || MODE == MODE_F2W)) {
    // the warp's sums: one scatter per hot row, none for a row it never updated
    auto flush = [&](const float2 (&v)[NS], float *row) {
      bool any = false;
#pragma unroll
      for (int j = 0; j < NS; ++j) any |= v[j].x != 0.f || v[j].y != 0.f;
      if (__any_sync(0xffffffffu, any)) {
#pragma unroll
        for (int j = 0; j < NS; ++j)
          if (j < NS - 1 || lane + 32 * j < 2 * p.mv.nvec)
            atomicAdd(reinterpret_cast<float2 *>(row + 2 * lane + 64 * j), v[j]);
      }
    };
    __syncwarp();
    if (!hot.in_s) flush(hot.reg, reinterpret_cast<float *>(p.mv.in_dst));
    const float *hs = reinterpret_cast<const float *>(base + L.hot);
    for (int r = 0; r < p.hot_in + p.hot_out; ++r) {
      const float *src = hs + (int64_t)r * p.mv.ld + 2 * lane;
      float2 v[NS];
#pragma unroll
      for (int j = 0; j < NS; ++j)
        v[j] = (j < NS - 1 || lane + 32 * j < 2 * p.mv.nvec)
                   ? *reinterpret_cast<const float2 *>(src + 64 * j) : make_float2(0.f, 0.f);
      float *dst = r < p.hot_in ? reinterpret_cast<float *>(p.mv.in_dst) + (int64_t)r * p.mv.ld
                                : reinterpret_cast<float *>(p.mv.out_dst) + (int64_t)(r - p.hot_in) * p.mv.ld;
      flush(v, dst);
    }
  }
  if (p.loss_every > 0) flush_loss<T>(loss, cells, p.loss_sum, p.loss_cells, true, lane);
}

// ---------------------------------------------------------------- driver ----
template <typename T> struct DriveArgs {
  ModelView<T> mv;
  const int32_t *ids;
  const int64_t *offsets;
  const double *keep;
  const int32_t *slots;
  uint64_t n_slots;
  const uint32_t *alias_thr;
  const int32_t *alias_idx;
  uint32_t vocab;
  uint32_t key0, key1;
  int window, dynamic, k_neg, cap, exact;
  const T *sig;
  double alpha0, floor_frac, total_x_epochs;
  int64_t refresh;
  unsigned long long *shared;
  int epochs, loss_every;
  sgns_worker *workers;
  int n_workers;
  int64_t budget;
  double *loss_by_epoch;
  int64_t *cells_by_epoch;
  int update;
  int kept_cap;
  int64_t trace_cap;
  int32_t *trace;
  double *trace_alpha;
  int64_t *trace_count;
  int32_t *error;
  int wpb;
  int64_t token_base;
  uint32_t epoch_base;
  uint8_t *dirty;  // optional touched-row map [2 * vocab]
};

// Splitmix stream window: 32 consecutive draws evaluated by the 32 lanes.
struct SmBatch {
  uint64_t base;  // stream state before draw 0 of this batch
  uint64_t z;     // this lane's draw
  int used;       // draws consumed so far (uniform)
  __device__ __forceinline__ void refill(uint64_t st, int lane) {
    base = st;
    z = sm_mix(st + (uint64_t)(lane + 1) * kGolden);
    used = 0;
  }
  __device__ __forceinline__ uint64_t state_after() const { return base + (uint64_t)used * kGolden; }
};

template <typename T, int MODE, int NS, int NCH, int K1R, int RNG>
__global__ void __maxnreg__((UpdRegs<MODE, NS, K1R, true>::v)) drive_kernel(DriveArgs<T> p) {
  extern __shared__ __align__(128) unsigned char smem[];
  T *sig_s = reinterpret_cast<T *>(smem);
  load_table(sig_s, p.sig);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wid = blockIdx.x * p.wpb + warp;
  if (wid >= p.n_workers) return;
  const int k1 = p.k_neg + 1;
  const int mcap = min(p.cap, 2 * p.window);
  const Slab L = slab_layout(MODE, sizeof(T), p.mv.lds, mcap, k1, p.kept_cap);
  unsigned char *base = smem + table_bytes(sizeof(T)) + (int64_t)warp * L.total;
  T *rows_s = reinterpret_cast<T *>(base + L.rows);
  T *e_s = reinterpret_cast<T *>(base + L.e);
  int *ids_s = reinterpret_cast<int *>(base + L.ids);
  uint32_t *roff_s = reinterpret_cast<uint32_t *>(base + L.roff);
  int *kept_s = reinterpret_cast<int *>(base + L.kept);
  int *koff_s = reinterpret_cast<int *>(base + L.off);
  const unsigned lt_mask = (1u << lane) - 1u;

  sgns_worker S = p.workers[wid];
  if (S.done) return;
  double alpha = S.alpha, read_local = S.read_local, trained_local = S.trained_local;
  T alpha_t = (T)alpha;
  uint64_t rng = S.rng;
  int64_t s = S.next_sent, budget_used = 0, trained = 0, kc = S.kernel_counter, inputs = 0;
  int epoch = S.epoch;
  int done = 0;
  double loss = 0.0;
  long long cells = 0;
  const int rec_len = 4 + p.cap + k1;

  auto close_epoch = [&]() {
    flush_loss<T>(loss, cells, p.loss_by_epoch + (int64_t)wid * p.epochs + epoch,
                  p.cells_by_epoch + (int64_t)wid * p.epochs + epoch, false, lane);
    loss = 0.0;
    cells = 0;
    epoch += 1;
    s = S.lo;
    if (epoch >= p.epochs) {
      done = 1;
      if (lane == 0) {  // ThreadRun.flush_counters (trainer.py:448-453)
        atomicAdd(p.shared, (unsigned long long)(int64_t)read_local);
        atomicAdd(p.shared + 1, (unsigned long long)(int64_t)trained_local);
      }
      read_local = trained_local = 0.0;
    }
  };

  while (!done && budget_used < p.budget) {
    if (s >= S.hi) {
      close_epoch();
      continue;
    }
    const int64_t lo_t = p.offsets[s], hi_t = p.offsets[s + 1];
    const int n = (int)(hi_t - lo_t);
    if (n > p.kept_cap) {
      if (lane == 0 && p.error) atomicExch(p.error, 2);
      done = 1;
      break;
    }
    read_local += (double)n;
    budget_used += n;
    if (read_local >= (double)p.refresh) {  // alpha refresh (trainer.py:243-252)
      unsigned long long before = 0;
      if (lane == 0) {
        before = atomicAdd(p.shared, (unsigned long long)(int64_t)read_local);
        atomicAdd(p.shared + 1, (unsigned long long)(int64_t)trained_local);
      }
      before = __shfl_sync(0xffffffffu, before, 0);
      const double now = (double)(int64_t)(before + (unsigned long long)(int64_t)read_local);
      read_local = trained_local = 0.0;
      double frac = 1.0 - now / (p.total_x_epochs + 1.0);
      if (frac < p.floor_frac) frac = p.floor_frac;
      alpha = p.alpha0 * frac;
      alpha_t = (T)alpha;
    }
    // subsample (corpus.py:168-181): one uniform per token, survivors compacted in order
    int nk = 0;
    for (int b0 = 0; b0 < n; b0 += 32) {
      const int i = b0 + lane;
      const bool valid = i < n;
      const int w = valid ? p.ids[lo_t + i] : 0;
      bool keep = valid;
      if (p.keep != nullptr && valid) {
        double u;
        if (RNG == SGNS_RNG_SPLITMIX) {
          u = u53(sm_mix(rng + (uint64_t)(i + 1) * kGolden));
        } else {
          const uint4 o = philox_tok((uint64_t)(p.token_base + lo_t + i), p.epoch_base + (uint32_t)epoch,
                                     kTagSub, p.key0, p.key1);
          u = u53((uint64_t)o.x | ((uint64_t)o.y << 32));
        }
        keep = u < p.keep[w];
      }
      const unsigned mask = __ballot_sync(0xffffffffu, keep);
      if (keep) {
        const int pos = nk + __popc(mask & lt_mask);
        kept_s[pos] = w;
        koff_s[pos] = i;
      }
      nk += __popc(mask);
    }
    if (RNG == SGNS_RNG_SPLITMIX && p.keep != nullptr) rng += (uint64_t)n * kGolden;
    __syncwarp();

    SmBatch sb;
    for (int pos = 0; pos < nk; ++pos) {
      int b = p.window;
      if (RNG == SGNS_RNG_SPLITMIX) {
        sb.refill(rng, lane);
        if (p.dynamic) {
          const uint64_t bz = __shfl_sync(0xffffffffu, sb.z, 0);
          b = 1 + (int)(bz % (uint64_t)p.window);
          sb.used = 1;
        }
      } else if (p.dynamic) {
        const uint4 o = philox_tok((uint64_t)(p.token_base + lo_t + koff_s[pos]),
                                   p.epoch_base + (uint32_t)epoch, kTagWin, p.key0, p.key1);
        b = 1 + (int)(((uint64_t)o.x * (uint64_t)p.window) >> 32);
      }
      const int wlo = max(pos - b, 0);
      const int whi = min(pos + b + 1, nk);
      const int m = whi - wlo - 1;
      if (m <= 0) {
        if (RNG == SGNS_RNG_SPLITMIX) rng = sb.state_after();
        continue;
      }
      const int target = kept_s[pos];
      const int left = pos - wlo;
      uint32_t attempt = 0;  // philox attempt counter within the chunk
      int chunk = 0;
      for (int start = 0; start < m; start += p.cap, ++chunk) {
        const int mc = min(p.cap, m - start);
        for (int r = lane; r < mc; r += 32) {
          const int q = start + r;
          ids_s[r] = q < left ? kept_s[wlo + q] : kept_s[pos + 1 + (q - left)];
        }
        if (lane == 0) ids_s[mc] = target;
        // K shared negatives, rejecting the target (kernel_batched.py:57-66)
        int need = p.k_neg;
        attempt = 0;
        while (need > 0) {
          bool ok = false;
          int word = -1;
          int span;
          if (RNG == SGNS_RNG_SPLITMIX) {
            if (sb.used >= 32) sb.refill(sb.state_after(), lane);
            span = min(32 - sb.used, need + 2);
            if (lane >= sb.used && lane < sb.used + span) {
              word = p.slots[sb.z % p.n_slots];
              ok = word != target;
            }
          } else {
            span = min(32, need + 2);
            if (lane < span) {
              const uint32_t a = attempt + (uint32_t)lane;
              const uint4 o = philox_tok((uint64_t)(p.token_base + lo_t + koff_s[pos]),
                                         p.epoch_base + (uint32_t)epoch,
                                         kTagNeg | ((uint32_t)(chunk & 0xFF) << 16) | ((a >> 1) & 0xFFFFu),
                                         p.key0, p.key1);
              const uint32_t bw = (a & 1) ? o.z : o.x, coin = (a & 1) ? o.w : o.y;
              const uint32_t bucket = (uint32_t)(((uint64_t)bw * (uint64_t)p.vocab) >> 32);
              word = coin < p.alias_thr[bucket] ? (int)bucket : p.alias_idx[bucket];
              ok = word != target;
            }
          }
          const unsigned mask = __ballot_sync(0xffffffffu, ok);
          const int avail = __popc(mask);
          const int take = min(avail, need);
          const int rank = __popc(mask & lt_mask);
          if (ok && rank < take) ids_s[mc + 1 + (p.k_neg - need) + rank] = word;
          int consumed_to;  // lane index one past the last consumed draw
          if (take == need && take > 0) {
            unsigned mm = mask;
            for (int t = 1; t < take; ++t) mm &= mm - 1;  // drop take-1 lowest set bits
            consumed_to = __ffs(mm);                      // 1-based lane of the take-th accept
          } else {
            consumed_to = (RNG == SGNS_RNG_SPLITMIX ? sb.used : 0) + span;
          }
          if (RNG == SGNS_RNG_SPLITMIX) sb.used = consumed_to;
          else attempt += (uint32_t)consumed_to;
          need -= take;
          if (RNG != SGNS_RNG_SPLITMIX && need > 0 && attempt >= kMaxNegAttempts) {
            // 17 attempt bits in the Philox counter: flag instead of cycling forever
            if (lane == 0 && p.error) atomicExch(p.error, 3);
            for (int r = lane; r < need; r += 32)
              ids_s[mc + 1 + (p.k_neg - need) + r] = (target + 1 + r) % (int)p.vocab;
            need = 0;
          }
        }
        __syncwarp();
        kc += 1;
        inputs += mc;
        if (p.dirty != nullptr) {  // touched rows (data-parallel touched-row averaging)
          for (int r = lane; r < mc + k1; r += 32) p.dirty[(r < mc ? 0u : p.vocab) + (uint32_t)ids_s[r]] = 1;
        }
        const bool want = p.loss_every > 0 && (kc % p.loss_every) == 0;
        if (p.trace_cap > 0) {
          int64_t idx = p.trace_count[wid];
          if (idx < p.trace_cap) {
            int32_t *rec = p.trace + ((int64_t)wid * p.trace_cap + idx) * rec_len;
            for (int r = lane; r < rec_len; r += 32) {
              int v;
              if (r == 0) v = target;
              else if (r == 1) v = mc;
              else if (r == 2) v = (int)s;
              else if (r == 3) v = epoch;
              else if (r < 4 + p.cap) v = (r - 4) < mc ? ids_s[r - 4] : -1;
              else v = ids_s[mc + (r - 4 - p.cap)];
              rec[r] = v;
            }
            if (lane == 0) p.trace_alpha[(int64_t)wid * p.trace_cap + idx] = (double)alpha_t;
          }
          __syncwarp();
          if (lane == 0) p.trace_count[wid] = idx + 1;
        }
        if (p.update) {
          HotSink<hot_slots(NS)> no_hot;  // in-place training: no deferred rows (HOT = false)
          run_window<T, MODE, NS, NCH, K1R>(p.mv, ids_s, roff_s, mc, k1, alpha_t, p.exact != 0, sig_s,
                                            want, loss, cells, rows_s, e_s, lane, no_hot);
        }
        __syncwarp();
      }
      if (RNG == SGNS_RNG_SPLITMIX) rng = sb.state_after();
    }
    trained += nk;
    trained_local += (double)nk;
    s += 1;
  }
  if (!done && s >= S.hi) close_epoch();  // ThreadRun.advance :435-441
  if (!done || epoch < p.epochs) {
    flush_loss<T>(loss, cells, p.loss_by_epoch + (int64_t)wid * p.epochs + min(epoch, p.epochs - 1),
                  p.cells_by_epoch + (int64_t)wid * p.epochs + min(epoch, p.epochs - 1), false, lane);
  }
  if (lane == 0) {
    sgns_worker &o = p.workers[wid];
    o.next_sent = s;
    o.epoch = epoch;
    o.done = done;
    o.rng = rng;
    o.alpha = alpha;
    o.read_local = read_local;
    o.trained_local = trained_local;
    o.kernel_counter = kc;
    o.words_read = S.words_read + budget_used;
    o.words_trained = S.words_trained + trained;
    o.inputs = S.inputs + inputs;
  }
}

#if SGNS_HAS(0)
// ------------------------------------------------------------------ init ----
template <typename T>
__global__ void init_model_kernel(T *m_in, T *m_out, int64_t V, int dim, int64_t ld, uint64_t s0) {
  const double bound = 0.5 / dim;
  const int64_t total = V * ld;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = e / ld;
    const int col = (int)(e - row * ld);
    T v = T(0);
    if (col < dim) {
      const uint64_t n = (uint64_t)(row * dim + col);  // draw index in model.py's row-major fill
      const double u = u53(sm_mix(s0 + (n + 1) * kGolden));
      v = (T)((u * 2.0 - 1.0) * bound);
    }
    m_in[e] = v;
    m_out[e] = T(0);
  }
}

__global__ void expand_slots_kernel(const int64_t *bounds, int64_t V, int32_t *slots, int64_t n) {
  for (int64_t sidx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; sidx < n;
       sidx += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = V - 1;  // first w with bounds[w] > sidx
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (bounds[mid] > sidx) hi = mid;
      else lo = mid + 1;
    }
    slots[sidx] = (int32_t)lo;
  }
}

#endif  // SGNS_HAS(0)

// ----------------------------------------------------------- dispatching ----
static int nch_for(int nvec) {
  const int need = (nvec + 31) / 32;
  if (need <= 1) return 1;
  if (need <= 2) return 2;
  if (need <= 3) return 3;
  if (need <= 4) return 4;
  if (need <= 8) return 8;
  return -1;
}

static int g_num_sms = 0;
static int num_sms() {
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

template <typename K>
static int prepare(K kernel, int64_t smem_bytes) {
  if (smem_bytes > 227 * 1024) return SGNS_E_SMEM;
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem_bytes);
  return e == cudaSuccess ? 0 : (int)e;
}

// Choose warps per block maximising resident warps for a given per-warp slab.
template <typename K>
static int choose_wpb(K kernel, int64_t table, int64_t slab, int *wpb_out, int *blocks_per_sm) {
  int best = -1, best_w = 1, best_b = 1;
  for (int w : {1, 2, 4, 8}) {
    const int64_t bytes = table + (int64_t)w * slab;
    if (bytes > 227 * 1024) break;
    if (prepare(kernel, bytes) != 0) break;
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, w * 32, (size_t)bytes) != cudaSuccess)
      break;
    if (nb * w > best) {
      best = nb * w;
      best_w = w;
      best_b = nb;
    }
  }
  if (best <= 0) return SGNS_E_SMEM;
  *wpb_out = best_w;
  *blocks_per_sm = best_b;
  return 0;
}

// entry points of the parts (defined in parts 1, 2, 3)
int update_f32(UpdateArgs<float> a, cudaStream_t st);
int update_f64(UpdateArgs<double> a, cudaStream_t st);
int drive_static(const sgns_drive_params *p, cudaStream_t st, int *resident);
int fast_dispatch(const sgns_drive_params *p, cudaStream_t st, int *resident);

static int ns_for(int64_t ld_elems_f32) { return (int)((ld_elems_f32 / 2 + 31) / 32); }
static bool offsets32_ok(int64_t vocab, int64_t ld) { return vocab * ld < (int64_t(1) << 32); }

// 8 < k1 <= 16: F2S (all rows staged in shared memory, dA scattered once) while shared
// memory still allows it as many resident warps as F2G (output rows in two register
// groups, dA scattered per group); F2G otherwise (configs[1] d = 300, K = 15: 7 vs 16 warps
// per SM, 0.35 -> 0.50 of the HBM peak).
template <typename KS, typename KG>
static bool prefer_staged(KS ks, KG kg, int64_t slab_staged, int64_t slab_groups) {
  int ws = 0, bs = 0, wg = 0, bg = 0;
  if (choose_wpb(ks, table_bytes(4), slab_staged, &ws, &bs)) return false;
  if (choose_wpb(kg, table_bytes(4), slab_groups, &wg, &bg)) return true;
  return ws * bs >= wg * bg;
}

#if SGNS_HAS(1)
// Both matrices gathered from a separate source (snapshot mode): the hot-row sinks may
// defer the hottest rows' updates to the end of the launch (see HotSink).
static bool snapshot_mode(const ModelView<float> &mv) {
  return static_cast<const float *>(mv.in_dst) != mv.in_src &&
         static_cast<const float *>(mv.out_dst) != mv.out_src;
}

template <typename T, int MODE, int NS, int NCH, int K1R, bool HOT = false>
static int launch_update_t(UpdateArgs<T> a, cudaStream_t st) {
  auto kern = update_windows_kernel<T, MODE, NS, NCH, K1R, HOT>;
  a.mstage = a.mcap;
  Slab L = slab_layout(MODE, sizeof(T), a.mv.lds, a.mstage, a.k1, 0);
  int wpb = 0, bps = 0;
  int rc = choose_wpb(kern, table_bytes(sizeof(T)), L.total, &wpb, &bps);
  if (rc) return rc;
  a.hot_in = a.hot_out = 0;
  if constexpr (HOT) {
    // Snapshot mode, long windows (w = 10: 20 input rows, 24 KB per warp at d = 300) whose
    // staging leaves fewer than 16 resident warps: stage half the inputs at a time (kernel:
    // chunks) if that raises the warp count.  The output rows are loaded and their dC
    // scattered once per chunk, which costs less than the warps and the larger sink they
    // leave room for (configs[1] w = 10, K = 5 / 10 / 15: d = 300 0.68 / 0.46 / 0.44 ->
    // 0.86 / 0.56 / 0.49 at 12 instead of 8 warps; d = 200 0.65 / 0.43 / 0.40 -> 0.77 /
    // 0.48 / 0.43 at 16 instead of 12; d = 100 keeps 16 warps either way and loses 2-7%,
    // so it is not split; profiles/round2_microbench_split.jsonl).  SGNS_UPDATE_SPLIT=0/1
    // forces it off / on (experiments).
    const char *sp = std::getenv("SGNS_UPDATE_SPLIT");
    const bool split = sp ? sp[0] == '1' : (a.mcap > 12 && wpb * bps < 16);
    if (split && a.mcap > 1) {
      const int half = (a.mcap + 1) / 2;
      const Slab Ls = slab_layout(MODE, sizeof(T), a.mv.lds, half, a.k1, 0);
      int ws = 0, bs = 0;
      if (choose_wpb(kern, table_bytes(sizeof(T)), Ls.total, &ws, &bs) == 0 && (ws * bs > wpb * bps || sp)) {
        a.mstage = half;
        L = Ls;
        wpb = ws;
        bps = bs;
      }
    }
  }
  if constexpr (HOT && (MODE == MODE_F2 || MODE == MODE_F2G || MODE == MODE_F2W)) {
    // shared-memory hot-row sinks: rows [0, H) of both matrices (H <= 8), else M_out's row 0
    // beside the register sink for M_in's row 0
    const int cand[5][2] = {{8, 8}, {4, 4}, {2, 2}, {1, 1}, {0, 1}};
    // Per-warp sink rows vs resident warps (measured over the configs[1] grid with every
    // sink forced, profiles/round2_microbench_sinks.jsonl): the step from row 0 alone to rows
    // [0, 2) of both matrices is worth a quarter of the resident warps while >= 12 stay
    // (d = 300, w = 5, K = 5: 0.78 -> 0.96 of the copy peak at 12 instead of 16 warps); larger
    // sinks only pay when they cost no further warp.  So: the largest sink that keeps every
    // warp; if that is below 2 + 2 rows, a launch with at least 4 windows per resident warp
    // (d = 300, K = 5: 16,384 windows 0.62 -> 0.76, 4,096 windows 0.43 -> 0.40) may drop to >= max(12, 3/4) of the warps to reach 2 + 2; then the largest sink at that
    // warp count.  SGNS_UPDATE_HOT=hin,hout forces one candidate (experiments).
    int forced[2] = {-1, -1};
    if (const char *fh = std::getenv("SGNS_UPDATE_HOT")) std::sscanf(fh, "%d,%d", &forced[0], &forced[1]);
    int cw[5], cb[5];
    Slab cl[5];
    for (int c = 0; c < 5; ++c) {
      cl[c] = slab_layout(MODE, sizeof(T), a.mv.lds, a.mstage, a.k1, 0, cand[c][0] + cand[c][1], a.mv.ld);
      if (choose_wpb(kern, table_bytes(sizeof(T)), cl[c].total, &cw[c], &cb[c]) != 0) cw[c] = cb[c] = 0;
    }
    const int wmax = wpb * bps;
    int need = wmax, pick = -1;
    for (int c = 0; c < 5 && pick < 0; ++c)
      if (cw[c] * cb[c] >= need) pick = c;
    if ((pick < 0 || cand[pick][0] < 2) && cw[2] * cb[2] >= std::max(12, (3 * wmax + 3) / 4) &&
        (int64_t)a.n_win >= (int64_t)4 * wmax * num_sms()) {
      need = cw[2] * cb[2];
      pick = -1;
      for (int c = 0; c < 5 && pick < 0; ++c)
        if (cw[c] * cb[c] >= need) pick = c;
    }
    if (forced[0] >= 0) {
      pick = -1;
      for (int c = 0; c < 5; ++c)
        if (cand[c][0] == forced[0] && cand[c][1] == forced[1] && cw[c] > 0) pick = c;
    }
    if (pick >= 0) {
      a.hot_in = cand[pick][0];
      a.hot_out = cand[pick][1];
      L = cl[pick];
      wpb = cw[pick];
      bps = cb[pick];
    }
  }
  a.wpb = wpb;
  const int64_t bytes = table_bytes(sizeof(T)) + (int64_t)wpb * L.total;
  if ((rc = prepare(kern, bytes))) return rc;
  if (std::getenv("SGNS_UPDATE_DEBUG"))
    std::fprintf(stderr, "update_windows: mode %d NS %d K1R %d hot %d | mcap %d k1 %d | sink %d+%d rows, %d warps x %d blocks per SM, %lld B, stage %d\n",
                 MODE, NS, K1R, (int)HOT, a.mcap, a.k1, a.hot_in, a.hot_out, wpb, bps, (long long)bytes, a.mstage);
  const int64_t blocks_needed = (a.n_win + wpb - 1) / wpb;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(blocks_needed, (int64_t)num_sms() * bps));
  kern<<<grid, wpb * 32, bytes, st>>>(a);
  return (int)cudaGetLastError();
}

#endif  // SGNS_HAS(1)

#if SGNS_HAS(2)
template <typename T, int MODE, int NS, int NCH, int K1R, int RNG>
static int launch_drive_t(DriveArgs<T> a, int wpb_req, cudaStream_t st, int *resident = nullptr) {
  auto kern = drive_kernel<T, MODE, NS, NCH, K1R, RNG>;
  const int k1 = a.k_neg + 1;
  const Slab L = slab_layout(MODE, sizeof(T), a.mv.lds, std::min(a.cap, 2 * a.window), k1, a.kept_cap);
  int wpb = 0, bps = 0;
  int rc = choose_wpb(kern, table_bytes(sizeof(T)), L.total, &wpb, &bps);
  if (rc) return rc;
  if (resident) {  // occupancy query only
    *resident = wpb * bps * num_sms();
    return 0;
  }
  if (wpb_req > 0) wpb = wpb_req;
  a.wpb = wpb;
  const int64_t bytes = table_bytes(sizeof(T)) + (int64_t)wpb * L.total;
  if ((rc = prepare(kern, bytes))) return rc;
  const int grid = (a.n_workers + wpb - 1) / wpb;
  kern<<<grid, wpb * 32, bytes, st>>>(a);
  return (int)cudaGetLastError();
}

// float32 fast path: k1 <= 8, d <= 512 (NS = float2 slots per lane), V * ld < 2^32

template <int NS, int RNG>
static int drive_f2(DriveArgs<float> a, int wpb, cudaStream_t st, int *res) {
  constexpr int NCH = (NS + 1) / 2;
  if (a.k_neg + 1 == 6) return launch_drive_t<float, MODE_F2, NS, NCH, 6, RNG>(a, wpb, st, res);
  return launch_drive_t<float, MODE_F2, NS, NCH, 8, RNG>(a, wpb, st, res);
}

template <int NS, int RNG>
static int drive_f2s(DriveArgs<float> a, int wpb, cudaStream_t st, int *res) {
  constexpr int NCH = (NS + 1) / 2;
  const int k1 = a.k_neg + 1, mcap = std::min(a.cap, 2 * a.window);
  if (prefer_staged(drive_kernel<float, MODE_F2S, NS, NCH, 16, RNG>,
                    drive_kernel<float, MODE_F2G, NS, NCH, 8, RNG>,
                    slab_layout(MODE_F2S, 4, a.mv.lds, mcap, k1, a.kept_cap).total,
                    slab_layout(MODE_F2G, 4, a.mv.lds, mcap, k1, a.kept_cap).total))
    return launch_drive_t<float, MODE_F2S, NS, NCH, 16, RNG>(a, wpb, st, res);
  // F2G's K1R: rows of its second output group
  if (k1 <= 12) return launch_drive_t<float, MODE_F2G, NS, NCH, 4, RNG>(a, wpb, st, res);
  return launch_drive_t<float, MODE_F2G, NS, NCH, 8, RNG>(a, wpb, st, res);
}

template <int RNG>
static int drive_f32(DriveArgs<float> a, int wpb, cudaStream_t st, int *res) {
  const int ns = ns_for(4 * a.mv.nvec);
  if (a.k_neg + 1 > 8 && a.k_neg + 1 <= 16 && offsets32_ok(a.vocab, a.mv.ld)) {
    switch (ns) {
      case 1: return drive_f2s<1, RNG>(a, wpb, st, res);
      case 2: return drive_f2s<2, RNG>(a, wpb, st, res);
      case 3: return drive_f2s<3, RNG>(a, wpb, st, res);
      case 4: return drive_f2s<4, RNG>(a, wpb, st, res);
      case 5: return drive_f2s<5, RNG>(a, wpb, st, res);
      case 6: return drive_f2s<6, RNG>(a, wpb, st, res);
      case 7: return drive_f2s<7, RNG>(a, wpb, st, res);
      case 8: return drive_f2s<8, RNG>(a, wpb, st, res);
    }
  }
  if (a.k_neg + 1 <= 8 && offsets32_ok(a.vocab, a.mv.ld)) {
    switch (ns) {
      case 1: return drive_f2<1, RNG>(a, wpb, st, res);
      case 2: return drive_f2<2, RNG>(a, wpb, st, res);
      case 3: return drive_f2<3, RNG>(a, wpb, st, res);
      case 4: return drive_f2<4, RNG>(a, wpb, st, res);
      case 5: return drive_f2<5, RNG>(a, wpb, st, res);
      case 6: return drive_f2<6, RNG>(a, wpb, st, res);
      case 7: return drive_f2<7, RNG>(a, wpb, st, res);
      case 8: return drive_f2<8, RNG>(a, wpb, st, res);
    }
  }
  switch (nch_for(a.mv.nvec)) {
    case 1: return launch_drive_t<float, MODE_SMEM, 0, 1, 0, RNG>(a, wpb, st, res);
    case 2: return launch_drive_t<float, MODE_SMEM, 0, 2, 0, RNG>(a, wpb, st, res);
    case 3: return launch_drive_t<float, MODE_SMEM, 0, 3, 0, RNG>(a, wpb, st, res);
    case 4: return launch_drive_t<float, MODE_SMEM, 0, 4, 0, RNG>(a, wpb, st, res);
    case 8: return launch_drive_t<float, MODE_SMEM, 0, 8, 0, RNG>(a, wpb, st, res);
  }
  return SGNS_E_SHAPE;
}

template <int RNG>
static int drive_f64(DriveArgs<double> a, int wpb, cudaStream_t st, int *res) {
  switch (nch_for(a.mv.nvec)) {
    case 1: return launch_drive_t<double, MODE_SMEM, 0, 1, 0, RNG>(a, wpb, st, res);
    case 2: return launch_drive_t<double, MODE_SMEM, 0, 2, 0, RNG>(a, wpb, st, res);
    case 3: return launch_drive_t<double, MODE_SMEM, 0, 3, 0, RNG>(a, wpb, st, res);
    case 4: return launch_drive_t<double, MODE_SMEM, 0, 4, 0, RNG>(a, wpb, st, res);
    case 8: return launch_drive_t<double, MODE_SMEM, 0, 8, 0, RNG>(a, wpb, st, res);
  }
  return SGNS_E_SHAPE;
}

#endif  // SGNS_HAS(2)

#if SGNS_HAS(1)
template <int NS>
static int update_f2(UpdateArgs<float> a, cudaStream_t st) {
  constexpr int NCH = (NS + 1) / 2;
  const bool hot = snapshot_mode(a.mv);
  if (a.k1 == 6)
    return hot ? launch_update_t<float, MODE_F2, NS, NCH, 6, true>(a, st)
               : launch_update_t<float, MODE_F2, NS, NCH, 6, false>(a, st);
  return hot ? launch_update_t<float, MODE_F2, NS, NCH, 8, true>(a, st)
             : launch_update_t<float, MODE_F2, NS, NCH, 8, false>(a, st);
}

template <int NS>
static int update_f2s(UpdateArgs<float> a, cudaStream_t st) {
  constexpr int NCH = (NS + 1) / 2;
  const bool hot = snapshot_mode(a.mv);
  const char *force = std::getenv("SGNS_UPDATE_BODY");  // experiments: "g" / "s" force F2G / F2S
  // The two-group body is never slower than the all-staged one on the configs[1] grid
  // (18 shapes with K = 10 / 15, profiles/round2_microbench_bodies_grid.jsonl: equal where
  // both keep 16 warps per SM at d = 300, +4..12% at d = 100 / 200 with w <= 5, 1.3-1.9x
  // where staging the output rows costs resident warps), so it is the choice; "s" forces F2S.
  const bool staged = force && force[0] == 's';
  if constexpr (NS <= 2) {
    // d <= 128: all k1 output rows fit one register group (the wide body: configs[1] d = 100,
    // K = 10: +6..13% over F2G, K = 15: +2.4% at w <= 5, -6% at w = 10, which stays on F2G);
    // "g" forces F2G, "w" the wide body
    if (force ? force[0] == 'w' : !(a.k1 > 12 && a.mcap > 12)) {
      if (a.k1 <= 12)
        return hot ? launch_update_t<float, MODE_F2W, NS, NCH, 12, true>(a, st)
                   : launch_update_t<float, MODE_F2W, NS, NCH, 12, false>(a, st);
      return hot ? launch_update_t<float, MODE_F2W, NS, NCH, 16, true>(a, st)
                 : launch_update_t<float, MODE_F2W, NS, NCH, 16, false>(a, st);
    }
  }
  if (staged)
    return hot ? launch_update_t<float, MODE_F2S, NS, NCH, 16, true>(a, st)
               : launch_update_t<float, MODE_F2S, NS, NCH, 16, false>(a, st);
  // F2G's K1R: rows of its second output group
  if (a.k1 <= 12)
    return hot ? launch_update_t<float, MODE_F2G, NS, NCH, 4, true>(a, st)
               : launch_update_t<float, MODE_F2G, NS, NCH, 4, false>(a, st);
  return hot ? launch_update_t<float, MODE_F2G, NS, NCH, 8, true>(a, st)
             : launch_update_t<float, MODE_F2G, NS, NCH, 8, false>(a, st);
}

int update_f32(UpdateArgs<float> a, cudaStream_t st) {
  const int ns = ns_for(4 * a.mv.nvec);
  if (a.k1 > 8 && a.k1 <= 16 && offsets32_ok(a.vocab, a.mv.ld)) {
    switch (ns) {
      case 1: return update_f2s<1>(a, st);
      case 2: return update_f2s<2>(a, st);
      case 3: return update_f2s<3>(a, st);
      case 4: return update_f2s<4>(a, st);
      case 5: return update_f2s<5>(a, st);
      case 6: return update_f2s<6>(a, st);
      case 7: return update_f2s<7>(a, st);
      case 8: return update_f2s<8>(a, st);
    }
  }
  if (a.k1 <= 8 && offsets32_ok(a.vocab, a.mv.ld)) {
    switch (ns) {
      case 1: return update_f2<1>(a, st);
      case 2: return update_f2<2>(a, st);
      case 3: return update_f2<3>(a, st);
      case 4: return update_f2<4>(a, st);
      case 5: return update_f2<5>(a, st);
      case 6: return update_f2<6>(a, st);
      case 7: return update_f2<7>(a, st);
      case 8: return update_f2<8>(a, st);
    }
  }
  switch (nch_for(a.mv.nvec)) {
    case 1: return launch_update_t<float, MODE_SMEM, 0, 1, 0>(a, st);
    case 2: return launch_update_t<float, MODE_SMEM, 0, 2, 0>(a, st);
    case 3: return launch_update_t<float, MODE_SMEM, 0, 3, 0>(a, st);
    case 4: return launch_update_t<float, MODE_SMEM, 0, 4, 0>(a, st);
    case 8: return launch_update_t<float, MODE_SMEM, 0, 8, 0>(a, st);
  }
  return SGNS_E_SHAPE;
}

int update_f64(UpdateArgs<double> a, cudaStream_t st) {
  switch (nch_for(a.mv.nvec)) {
    case 1: return launch_update_t<double, MODE_SMEM, 0, 1, 0>(a, st);
    case 2: return launch_update_t<double, MODE_SMEM, 0, 2, 0>(a, st);
    case 3: return launch_update_t<double, MODE_SMEM, 0, 3, 0>(a, st);
    case 4: return launch_update_t<double, MODE_SMEM, 0, 4, 0>(a, st);
    case 8: return launch_update_t<double, MODE_SMEM, 0, 8, 0>(a, st);
  }
  return SGNS_E_SHAPE;
}

#endif  // SGNS_HAS(1)

#if SGNS_HAS(2)
template <typename T>
static void fill_drive_args(DriveArgs<T> &a, const sgns_drive_params *p) {
  std::memset(&a, 0, sizeof(a));
  T *mi = static_cast<T *>(p->d_m_in), *mo = static_cast<T *>(p->d_m_out);
  a.mv = make_view<T>(mi, mo, mi, mo, p->ld, p->dim);
  a.ids = p->d_ids;
  a.offsets = p->d_offsets;
  a.keep = p->d_keep_probs;
  a.slots = p->d_slots;
  a.n_slots = (uint64_t)p->n_slots;
  a.alias_thr = p->d_alias_thr;
  a.alias_idx = p->d_alias_idx;
  a.vocab = (uint32_t)p->vocab;
  a.key0 = (uint32_t)p->seed;
  a.key1 = (uint32_t)(p->seed >> 32);
  a.window = p->window;
  a.dynamic = p->dynamic;
  a.k_neg = p->k_neg;
  a.cap = p->batch_cap;
  a.exact = p->sigmoid_mode == SGNS_SIGMOID_EXACT;
  a.sig = static_cast<const T *>(p->d_sig_table);
  a.alpha0 = p->alpha0;
  a.floor_frac = p->floor_frac;
  a.total_x_epochs = p->total_x_epochs;
  a.refresh = p->refresh_words;
  a.shared = reinterpret_cast<unsigned long long *>(p->d_shared);
  a.epochs = p->epochs;
  a.loss_every = p->loss_every;
  a.workers = p->d_workers;
  a.n_workers = p->n_workers;
  a.budget = p->word_budget;
  a.loss_by_epoch = p->d_loss_by_epoch;
  a.cells_by_epoch = p->d_cells_by_epoch;
  a.update = p->update;
  a.kept_cap = ((std::max(p->max_sentence, 1) + 31) / 32) * 32;
  a.trace_cap = p->trace_cap;
  a.trace = p->d_trace;
  a.trace_alpha = p->d_trace_alpha;
  a.trace_count = p->d_trace_count;
  a.error = p->d_error;
  a.token_base = p->token_base;
  a.epoch_base = (uint32_t)p->epoch_base;
  a.dirty = p->d_dirty;
}

int drive_static(const sgns_drive_params *p, cudaStream_t st, int *resident) {
  const int wpb = p->warps_per_block;
  if (p->dtype == SGNS_F32) {
    DriveArgs<float> a;
    fill_drive_args(a, p);
    if (nch_for(a.mv.nvec) < 0) return SGNS_E_SHAPE;
    return p->rng_mode == SGNS_RNG_SPLITMIX ? drive_f32<SGNS_RNG_SPLITMIX>(a, wpb, st, resident)
                                            : drive_f32<SGNS_RNG_PHILOX>(a, wpb, st, resident);
  }
  DriveArgs<double> a;
  fill_drive_args(a, p);
  if (nch_for(a.mv.nvec) < 0) return SGNS_E_SHAPE;
  return p->rng_mode == SGNS_RNG_SPLITMIX ? drive_f64<SGNS_RNG_SPLITMIX>(a, wpb, st, resident)
                                          : drive_f64<SGNS_RNG_PHILOX>(a, wpb, st, resident);
}
#endif  // SGNS_HAS(2)

#if SGNS_HAS(3)
// ------------------------------------------------------------ fast path ----
template <int NS, int K1R, bool EXACT, bool FULL>
static int launch_fast_t(FastArgs a, int wpb_req, cudaStream_t st, int *resident) {
  constexpr int NCH = (NS + 1) / 2;
  auto kern = drive_fast_kernel<NS, NCH, K1R, EXACT, FULL>;
  const FastSlab L = fast_slab(fast_lds(a.mv.nvec), std::min(a.cap, 2 * a.window), K1R, a.kept_cap);
  int wpb = 0, bps = 0;
  int rc = choose_wpb(kern, table_bytes(4), L.total, &wpb, &bps);
  if (rc) return rc;
  if (resident) {
    *resident = wpb * bps * num_sms();
    return 0;
  }
  if (wpb_req > 0) wpb = wpb_req;
  a.wpb = wpb;
  const int64_t bytes = table_bytes(4) + (int64_t)wpb * L.total;
  if ((rc = prepare(kern, bytes))) return rc;
  const int grid = (a.n_workers + wpb - 1) / wpb;
  kern<<<grid, wpb * 32, bytes, st>>>(a);
  return (int)cudaGetLastError();
}

template <int NS>
static int fast_ns(FastArgs a, int wpb, cudaStream_t st, int *res) {
  const bool full = 4 * a.mv.nvec == 64 * NS;  // 32 lanes x NS float2 slots exactly
  // exact-K instantiations for K + 1 = 4..8 (no per-output predicates); K + 1 < 4 pads to 6
  switch (a.k_neg + 1) {
    case 4: return full ? launch_fast_t<NS, 4, true, true>(a, wpb, st, res)
                        : launch_fast_t<NS, 4, true, false>(a, wpb, st, res);
    case 5: return full ? launch_fast_t<NS, 5, true, true>(a, wpb, st, res)
                        : launch_fast_t<NS, 5, true, false>(a, wpb, st, res);
    case 6: return full ? launch_fast_t<NS, 6, true, true>(a, wpb, st, res)
                        : launch_fast_t<NS, 6, true, false>(a, wpb, st, res);
    case 7: return full ? launch_fast_t<NS, 7, true, true>(a, wpb, st, res)
                        : launch_fast_t<NS, 7, true, false>(a, wpb, st, res);
    case 8: return full ? launch_fast_t<NS, 8, true, true>(a, wpb, st, res)
                        : launch_fast_t<NS, 8, true, false>(a, wpb, st, res);
  }
  return full ? launch_fast_t<NS, 6, false, true>(a, wpb, st, res)
              : launch_fast_t<NS, 6, false, false>(a, wpb, st, res);
}

int pair_dispatch(const FastArgs &a, int64_t ld, int wpb, cudaStream_t st, int *resident);

int fast_dispatch(const sgns_drive_params *p, cudaStream_t st, int *resident) {
  FastArgs a;
  std::memset(&a, 0, sizeof(a));
  float *mi = static_cast<float *>(p->d_m_in), *mo = static_cast<float *>(p->d_m_out);
  a.mv = make_view<float>(mi, mo, mi, mo, p->ld, p->dim);
  a.ids = p->d_ids;
  a.offsets = p->d_offsets;
  a.keep = p->d_keep_probs;
  a.alias_thr = p->d_alias_thr;
  a.alias_idx = p->d_alias_idx;
  a.vocab = (uint32_t)p->vocab;
  a.key0 = (uint32_t)p->seed;
  a.key1 = (uint32_t)(p->seed >> 32);
  a.window = p->window;
  a.dynamic = p->dynamic;
  a.k_neg = p->k_neg;
  a.cap = p->batch_cap;
  a.sig = static_cast<const float *>(p->d_sig_table);
  a.alpha0 = p->alpha0;
  a.floor_frac = p->floor_frac;
  a.total_x_epochs = p->total_x_epochs;
  a.shard_lo = p->shard_lo;
  a.n_sent = p->shard_hi - p->shard_lo;
  a.epochs = p->epochs;
  a.loss_every = p->loss_every;
  a.claim = reinterpret_cast<unsigned long long *>(p->d_claim);
  a.claim_end = p->claim_end;
  a.workers = p->d_workers;
  a.n_workers = p->n_workers;
  a.loss_by_epoch = p->d_loss_by_epoch;
  a.cells_by_epoch = p->d_cells_by_epoch;
  a.kept_cap = ((std::max(p->max_sentence, 1) + 31) / 32) * 32;
  a.trace_cap = p->trace_cap;
  a.trace = p->d_trace;
  a.trace_alpha = p->d_trace_alpha;
  a.trace_count = reinterpret_cast<unsigned long long *>(p->d_trace_count);
  a.error = p->d_error;
  a.token_base = p->token_base;
  a.epoch_base = (uint32_t)p->epoch_base;
  a.words_base = p->words_base;
  a.totals = reinterpret_cast<unsigned long long *>(p->d_totals);
  a.loss_total = p->d_loss_total;
  a.dirty = p->d_dirty;
  const int wpb = p->warps_per_block;
  if (p->k_neg + 1 > 8) return pair_dispatch(a, 4 * a.mv.nvec, wpb, st, resident);  // warp pairs
  switch (ns_for(4 * a.mv.nvec)) {
#if !defined(SGNS_ONLY_NS) || SGNS_ONLY_NS == 1
    case 1: return fast_ns<1>(a, wpb, st, resident);
#endif
#if !defined(SGNS_ONLY_NS) || SGNS_ONLY_NS == 2
    case 2: return fast_ns<2>(a, wpb, st, resident);
#endif
#if !defined(SGNS_ONLY_NS) || SGNS_ONLY_NS == 3
    case 3: return fast_ns<3>(a, wpb, st, resident);
#endif
#if !defined(SGNS_ONLY_NS) || SGNS_ONLY_NS == 4
    case 4: return fast_ns<4>(a, wpb, st, resident);
#endif
#if !defined(SGNS_ONLY_NS) || SGNS_ONLY_NS == 5
    case 5: return fast_ns<5>(a, wpb, st, resident);
#endif
#if !defined(SGNS_ONLY_NS) || SGNS_ONLY_NS == 6
    case 6: return fast_ns<6>(a, wpb, st, resident);
#endif
#if !defined(SGNS_ONLY_NS) || SGNS_ONLY_NS == 7
    case 7: return fast_ns<7>(a, wpb, st, resident);
#endif
#if !defined(SGNS_ONLY_NS) || SGNS_ONLY_NS == 8
    case 8: return fast_ns<8>(a, wpb, st, resident);
#endif
  }
  return SGNS_E_SHAPE;
}

#endif  // SGNS_HAS(3)

#if SGNS_HAS(4)
// ------------------------------------------------- fast path, warp pairs ----
// K + 1 = 9..16: a worker is a pair of warps, each holding ceil((K + 1) / 2) output rows
// (drive_fast_kernel<..., PAIR>); n_workers counts pairs.
template <int NS, int K1R, bool FULL>
static int launch_pair_t(FastArgs a, int wpb_req, cudaStream_t st, int *resident) {
  constexpr int NCH = (NS + 1) / 2;
  auto kern = drive_fast_kernel<NS, NCH, K1R, false, FULL, true>;
  const FastSlab L = fast_slab(fast_lds(a.mv.nvec), std::min(a.cap, 2 * a.window), 2 * K1R, a.kept_cap);
  int best = -1, wpb = 2, bps = 1;
  for (int w : {2, 4, 8, 16}) {  // warps per block: whole pairs
    const int64_t bytes = table_bytes(4) + (int64_t)w * L.total;
    if (bytes > 227 * 1024 || prepare(kern, bytes) != 0) break;
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, w * 32, (size_t)bytes) != cudaSuccess) break;
    if (nb * w > best) {
      best = nb * w;
      wpb = w;
      bps = nb;
    }
  }
  if (best <= 0) return SGNS_E_SMEM;
  if (resident) {
    *resident = wpb * bps * num_sms() / 2;
    return 0;
  }
  if (wpb_req > 0) wpb = wpb_req & ~1;
  if (wpb < 2) return SGNS_E_ARG;
  a.wpb = wpb;
  const int64_t bytes = table_bytes(4) + (int64_t)wpb * L.total;
  int rc;
  if ((rc = prepare(kern, bytes))) return rc;
  const int grid = (int)((2 * (int64_t)a.n_workers + wpb - 1) / wpb);
  kern<<<grid, wpb * 32, bytes, st>>>(a);
  return (int)cudaGetLastError();
}

template <int NS>
static int pair_ns(const FastArgs &a, int64_t ld, int wpb, cudaStream_t st, int *res) {
  const bool full = ld == 64 * NS;
  switch ((a.k_neg + 2) / 2) {  // ceil((K + 1) / 2)
    case 5: return full ? launch_pair_t<NS, 5, true>(a, wpb, st, res) : launch_pair_t<NS, 5, false>(a, wpb, st, res);
    case 6: return full ? launch_pair_t<NS, 6, true>(a, wpb, st, res) : launch_pair_t<NS, 6, false>(a, wpb, st, res);
    case 7: return full ? launch_pair_t<NS, 7, true>(a, wpb, st, res) : launch_pair_t<NS, 7, false>(a, wpb, st, res);
    case 8: return full ? launch_pair_t<NS, 8, true>(a, wpb, st, res) : launch_pair_t<NS, 8, false>(a, wpb, st, res);
  }
  return SGNS_E_SHAPE;
}

int pair_dispatch(const FastArgs &a, int64_t ld, int wpb, cudaStream_t st, int *resident) {
  switch (ns_for(ld)) {
#if !defined(SGNS_ONLY_NS) || SGNS_ONLY_NS == 1
    case 1: return pair_ns<1>(a, ld, wpb, st, resident);
#endif
#if !defined(SGNS_ONLY_NS) || SGNS_ONLY_NS == 2
    case 2: return pair_ns<2>(a, ld, wpb, st, resident);
#endif
#if !defined(SGNS_ONLY_NS) || SGNS_ONLY_NS == 3
    case 3: return pair_ns<3>(a, ld, wpb, st, resident);
#endif
#if !defined(SGNS_ONLY_NS) || SGNS_ONLY_NS == 4
    case 4: return pair_ns<4>(a, ld, wpb, st, resident);
#endif
#if !defined(SGNS_ONLY_NS) || SGNS_ONLY_NS == 5
    case 5: return pair_ns<5>(a, ld, wpb, st, resident);
#endif
#if !defined(SGNS_ONLY_NS) || SGNS_ONLY_NS == 6
    case 6: return pair_ns<6>(a, ld, wpb, st, resident);
#endif
#if !defined(SGNS_ONLY_NS) || SGNS_ONLY_NS == 7
    case 7: return pair_ns<7>(a, ld, wpb, st, resident);
#endif
#if !defined(SGNS_ONLY_NS) || SGNS_ONLY_NS == 8
    case 8: return pair_ns<8>(a, ld, wpb, st, resident);
#endif
  }
  return SGNS_E_SHAPE;
}
#endif  // SGNS_HAS(4)


#if SGNS_HAS(0)
static bool fast_eligible(const sgns_drive_params *p) {
  const int64_t ld = p->ld, cols = 4 * ((p->dim + 3) / 4);  // row stride, columns holding data
  return p->dtype == SGNS_F32 && p->rng_mode == SGNS_RNG_PHILOX && p->k_neg + 1 <= 16 &&
         ns_for(cols) >= 1 && ns_for(cols) <= 8 && offsets32_ok(p->vocab, ld) &&
         p->sigmoid_mode == SGNS_SIGMOID_TABLE;
}

static int drive_dispatch(const sgns_drive_params *p, cudaStream_t st, int *resident) {
  if (p->schedule == SGNS_SCHEDULE_DYNAMIC) {
    if (!fast_eligible(p)) return SGNS_E_ARG;
    return fast_dispatch(p, st, resident);
  }
  return drive_static(p, st, resident);
}

static bool ld_ok(int32_t dtype, int32_t dim, int64_t ld) {
  const int64_t elem = dtype == SGNS_F64 ? 8 : 4;
  return dim >= 1 && ld >= dim && (ld * elem) % 16 == 0;
}

#endif  // SGNS_HAS(0)

}  // namespace sgns

using namespace sgns;

#if SGNS_HAS(0)

extern "C" {

int sgns_abi_version(void) { return SGNS_ABI_VERSION; }

int sgns_struct_sizes(int32_t *worker_bytes, int32_t *params_bytes) {
  if (!worker_bytes || !params_bytes) return SGNS_E_ARG;
  *worker_bytes = (int32_t)sizeof(sgns_worker);
  *params_bytes = (int32_t)sizeof(sgns_drive_params);
  return SGNS_OK;
}

const char *sgns_error_string(int32_t code) {
  switch (code) {
    case SGNS_OK: return "ok";
    case SGNS_E_ARG: return "invalid argument";
    case SGNS_E_SHAPE: return "shape outside the supported envelope (dim <= 1024 f32 / 512 f64, k+1 <= 32)";
    case SGNS_E_SMEM: return "per-warp staging does not fit in 227 KB of shared memory";
    case SGNS_E_DEVICE: return "device-side validation failed";
    case SGNS_E_IO: return "corpus file could not be opened";
    case SGNS_E_EMPTY: return "no token appears at least min_count times";
    case SGNS_E_TRUNC: return "vector file ends inside a row";
  }
  if (code > 0) return cudaGetErrorString((cudaError_t)code);
  return "unknown error";
}

int sgns_update_windows(int32_t dtype, void *d_m_in_dst, void *d_m_out_dst, const void *d_m_in_src,
                        const void *d_m_out_src, int64_t vocab, int32_t dim, int64_t ld,
                        const int32_t *d_in_off, const int32_t *d_in_ids, const int32_t *d_out_ids,
                        int32_t n_windows, int32_t k1, int32_t max_inputs, const void *d_alpha,
                        const void *d_sig_table, int32_t sigmoid_mode, int32_t loss_every,
                        double *d_loss_sum, int64_t *d_loss_cells, int32_t *d_error, void *stream) {
  if (n_windows == 0) return SGNS_OK;  // an empty packed batch is a no-op (empty id arrays may be null)
  if (!d_m_in_dst || !d_m_out_dst || !d_m_in_src || !d_m_out_src || !d_in_off || !d_in_ids ||
      !d_out_ids || !d_alpha || !d_sig_table || vocab < 1)
    return SGNS_E_ARG;
  if (n_windows < 0 || max_inputs < 1 || k1 < 2 || k1 > kMaxK1 || !ld_ok(dtype, dim, ld))
    return SGNS_E_SHAPE;
  if (loss_every > 0 && (!d_loss_sum || !d_loss_cells)) return SGNS_E_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == SGNS_F32) {
    UpdateArgs<float> a;
    a.mv = make_view<float>(static_cast<float *>(d_m_in_dst), static_cast<float *>(d_m_out_dst),
                            static_cast<const float *>(d_m_in_src), static_cast<const float *>(d_m_out_src),
                            ld, dim);
    a.in_off = d_in_off; a.in_ids = d_in_ids; a.out_ids = d_out_ids;
    a.n_win = n_windows; a.k1 = k1; a.mcap = max_inputs; a.vocab = vocab;
    a.alpha = static_cast<const float *>(d_alpha);
    a.sig = static_cast<const float *>(d_sig_table);
    a.exact = sigmoid_mode == SGNS_SIGMOID_EXACT;
    a.loss_every = loss_every; a.loss_sum = d_loss_sum; a.loss_cells = d_loss_cells;
    a.error = d_error; a.wpb = 1; a.hot_in = a.hot_out = 0; a.mstage = max_inputs;
    if (nch_for(a.mv.nvec) < 0) return SGNS_E_SHAPE;
    return update_f32(a, st);
  }
  if (dtype == SGNS_F64) {
    UpdateArgs<double> a;
    a.mv = make_view<double>(static_cast<double *>(d_m_in_dst), static_cast<double *>(d_m_out_dst),
                             static_cast<const double *>(d_m_in_src),
                             static_cast<const double *>(d_m_out_src), ld, dim);
    a.in_off = d_in_off; a.in_ids = d_in_ids; a.out_ids = d_out_ids;
    a.n_win = n_windows; a.k1 = k1; a.mcap = max_inputs; a.vocab = vocab;
    a.alpha = static_cast<const double *>(d_alpha);
    a.sig = static_cast<const double *>(d_sig_table);
    a.exact = sigmoid_mode == SGNS_SIGMOID_EXACT;
    a.loss_every = loss_every; a.loss_sum = d_loss_sum; a.loss_cells = d_loss_cells;
    a.error = d_error; a.wpb = 1; a.hot_in = a.hot_out = 0; a.mstage = max_inputs;
    if (nch_for(a.mv.nvec) < 0) return SGNS_E_SHAPE;
    return update_f64(a, st);
  }
  return SGNS_E_ARG;
}

int sgns_drive(const sgns_drive_params *p, void *stream) {
  if (!p || !p->d_m_in || !p->d_m_out || !p->d_ids || !p->d_offsets || !p->d_sig_table ||
      !p->d_shared || !p->d_workers || !p->d_loss_by_epoch || !p->d_cells_by_epoch)
    return SGNS_E_ARG;
  if (p->n_workers <= 0) return SGNS_OK;
  if (p->k_neg < 1 || p->k_neg + 1 > kMaxK1 || p->window < 1 || p->batch_cap < 1 ||
      p->epochs < 1 || !ld_ok(p->dtype, p->dim, p->ld) || p->max_sentence > kMaxSentence ||
      p->vocab < 2)
    return SGNS_E_SHAPE;
  if (p->rng_mode == SGNS_RNG_SPLITMIX && (!p->d_slots || p->n_slots < 1)) return SGNS_E_ARG;
  if (p->rng_mode == SGNS_RNG_PHILOX && (!p->d_alias_thr || !p->d_alias_idx)) return SGNS_E_ARG;
  if (p->rng_mode != SGNS_RNG_SPLITMIX && p->rng_mode != SGNS_RNG_PHILOX) return SGNS_E_ARG;
  if (p->trace_cap > 0 && (!p->d_trace || !p->d_trace_alpha || !p->d_trace_count)) return SGNS_E_ARG;
  if (p->schedule == SGNS_SCHEDULE_DYNAMIC &&
      (!p->d_claim || p->shard_hi <= p->shard_lo || p->shard_lo < 0)) return SGNS_E_ARG;
  if (p->dtype != SGNS_F32 && p->dtype != SGNS_F64) return SGNS_E_ARG;
  return drive_dispatch(p, static_cast<cudaStream_t>(stream), nullptr);
}

int sgns_init_model(int32_t dtype, void *d_m_in, void *d_m_out, int64_t vocab, int32_t dim,
                    int64_t ld, uint64_t seed, void *stream) {
  if (!d_m_in || !d_m_out || vocab < 1) return SGNS_E_ARG;
  if (!ld_ok(dtype, dim, ld)) return SGNS_E_SHAPE;
  // new_state(seed, 0x1017) (rng.py:50-56)
  uint64_t z = seed ^ (0x1017ULL * kGolden + 1ULL);
  z = (z ^ (z >> 30)) * kMix1;
  z = (z ^ (z >> 27)) * kMix2;
  const uint64_t s0 = z ^ (z >> 31);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t total = vocab * ld;
  const int grid = (int)std::min<int64_t>((total + 255) / 256, (int64_t)num_sms() * 32);
  if (dtype == SGNS_F32)
    init_model_kernel<float><<<grid, 256, 0, st>>>(static_cast<float *>(d_m_in), static_cast<float *>(d_m_out),
                                                     vocab, dim, ld, s0);
  else if (dtype == SGNS_F64)
    init_model_kernel<double><<<grid, 256, 0, st>>>(static_cast<double *>(d_m_in), static_cast<double *>(d_m_out),
                                                      vocab, dim, ld, s0);
  else
    return SGNS_E_ARG;
  return (int)cudaGetLastError();
}

int sgns_expand_slots(const int64_t *d_boundaries, int64_t vocab, int32_t *d_slots, int64_t n_slots,
                      void *stream) {
  if (!d_boundaries || !d_slots || vocab < 1 || n_slots < vocab) return SGNS_E_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int grid = (int)std::min<int64_t>((n_slots + 255) / 256, (int64_t)num_sms() * 32);
  expand_slots_kernel<<<grid, 256, 0, st>>>(d_boundaries, vocab, d_slots, n_slots);
  return (int)cudaGetLastError();
}

int sgns_resident_workers(int32_t dtype, int32_t dim, int32_t window, int32_t k_neg, int32_t batch_cap,
                          int32_t max_sentence, int32_t *out_workers) {
  if (!out_workers || dim < 1 || window < 1 || k_neg < 1 || batch_cap < 1) return SGNS_E_ARG;
  if (k_neg + 1 > kMaxK1) return SGNS_E_SHAPE;
  sgns_drive_params p;
  std::memset(&p, 0, sizeof(p));
  const int64_t elem = dtype == SGNS_F64 ? 8 : 4;
  p.dtype = dtype;
  p.ld = ((dim * elem + 15) / 16) * 16 / elem;
  p.dim = dim;
  p.window = window;
  p.k_neg = k_neg;
  p.batch_cap = batch_cap;
  p.max_sentence = max_sentence;
  p.rng_mode = SGNS_RNG_PHILOX;
  p.sigmoid_mode = dtype == SGNS_F64 ? SGNS_SIGMOID_EXACT : SGNS_SIGMOID_TABLE;
  p.schedule = fast_eligible(&p) ? SGNS_SCHEDULE_DYNAMIC : SGNS_SCHEDULE_STATIC;
  int resident = 0;
  const int rc = drive_dispatch(&p, nullptr, &resident);
  if (rc) return rc;
  *out_workers = resident;
  return SGNS_OK;
}

// Vose's alias method in float64 over count^power (host).
int sgns_build_alias(const int64_t *h_counts, int64_t vocab, double power, uint32_t *h_thr,
                     int32_t *h_alias) {
  if (!h_counts || !h_thr || !h_alias || vocab < 1 || vocab > (int64_t)INT32_MAX) return SGNS_E_ARG;
  std::vector<double> p(vocab);
  double total = 0.0;
  for (int64_t i = 0; i < vocab; ++i) {
    if (h_counts[i] < 0) return SGNS_E_ARG;
    p[i] = std::pow((double)h_counts[i], power);
    total += p[i];
  }
  if (!(total > 0.0)) return SGNS_E_ARG;
  std::vector<int32_t> small, large;
  small.reserve(vocab);
  large.reserve(vocab);
  for (int64_t i = 0; i < vocab; ++i) {
    p[i] = p[i] * (double)vocab / total;
    (p[i] < 1.0 ? small : large).push_back((int32_t)i);
  }
  auto thr_of = [](double q) -> uint32_t {
    if (q >= 1.0) return 0xFFFFFFFFu;
    if (q <= 0.0) return 0u;
    return (uint32_t)std::floor(std::ldexp(q, 32));
  };
  while (!small.empty() && !large.empty()) {
    const int32_t s = small.back();
    small.pop_back();
    const int32_t l = large.back();
    h_thr[s] = thr_of(p[s]);
    h_alias[s] = l;
    p[l] = (p[l] + p[s]) - 1.0;
    if (p[l] < 1.0) {
      large.pop_back();
      small.push_back(l);
    }
  }
  for (int32_t i : large) { h_thr[i] = 0xFFFFFFFFu; h_alias[i] = i; }
  for (int32_t i : small) { h_thr[i] = 0xFFFFFFFFu; h_alias[i] = i; }  // rounding leftovers
  return SGNS_OK;
}

}  // extern "C"

#endif  // SGNS_HAS(0)
