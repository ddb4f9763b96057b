// sgns_fast.cuh -- production driver: Philox draws, dynamic sentence claiming and
// negatives drawn one window ahead (float32, d <= 512, K + 1 <= 16: one warp per worker up
// to K + 1 = 8, a pair of warps above).
//
// Differences from drive_kernel (the reference-stream driver), all invisible to the
// update math:
//  * workers claim sentences from one atomic counter per shard instead of owning a
//    fixed range.  Philox draws are keyed by corpus position, so which worker trains a
//    sentence does not change any draw; the step ends one sentence after the budget
//    instead of at the slowest worker's range.
//  * alpha of a sentence is computed from its exact words-read position
//    (update_alpha, trainer.py:122-132) instead of a racy shared counter.
//  * the loss proxy samples every loss_every-th sentence (uniform over progress).
//  * the negatives of window u+1 are drawn (Philox + alias loads in flight) before window
//    u is computed; u+1's output rows are loaded right after u's dC scatter and so read
//    it (same-thread order), so every window sees its worker's previous updates exactly,
//    as a reference thread's does; their latency overlaps u+1's input-row gather.
#pragma once

#include "sgns_device.cuh"

namespace sgns {

__host__ __device__ inline int64_t round16_(int64_t b) { return (b + 15) & ~int64_t(15); }

struct FastArgs {
  ModelView<float> mv;
  const int32_t *ids;
  const int64_t *offsets;
  const double *keep;
  const uint32_t *alias_thr;
  const int32_t *alias_idx;
  uint32_t vocab;
  uint32_t key0, key1;
  int window, dynamic, k_neg, cap;
  const float *sig;
  double alpha0, floor_frac, total_x_epochs;
  int64_t shard_lo, n_sent;
  int epochs, loss_every;
  unsigned long long *claim;  // next sentence ordinal
  int64_t claim_end;          // exclusive
  sgns_worker *workers;       // per-worker counters (chunks, trained, inputs)
  int n_workers;
  double *loss_by_epoch;      // [n_workers][epochs]
  int64_t *cells_by_epoch;
  int kept_cap;
  int64_t trace_cap;          // total records (global), 0: off
  int32_t *trace;
  double *trace_alpha;
  unsigned long long *trace_count;
  int32_t *error;
  int wpb;
  int64_t token_base;
  uint32_t epoch_base;
  int64_t words_base;
  unsigned long long *totals;  // optional, see sgns_drive_params.d_totals
  double *loss_total;
  uint8_t *dirty;              // optional touched-row map [2 * vocab]
};

// Shared-memory stride of a staged input row, in floats: the data columns rounded up to 32
// bytes.  A 16-byte cp.async whose shared destination and global source differ in their
// offset within a 32-byte sector makes L1 fetch one sector per LANE (32 per warp
// instruction instead of 16; tools/probes/ldgsts_probe.cu), so staged rows keep the phase
// of the 128-byte-aligned model rows.
__host__ __device__ inline int fast_lds(int nvec) { return ((nvec + 1) & ~1) * 4; }  // = ModelView::lds

struct FastSlab {
  int64_t rows, e, ids, roff, kept, koff, bw, cnt, cand, total;
};
constexpr int kCandWords = 64;  // candidate negatives drawn per batch: one Philox call per lane
__host__ __device__ inline FastSlab fast_slab(int64_t ld, int mcap, int k1r, int kept_cap) {
  FastSlab s;
  const int idsn = mcap + k1r;
  s.rows = 0;
  s.e = round16_(int64_t(mcap) * ld * 4);
  s.ids = s.e + round16_(int64_t(mcap) * 8 * 4);  // error rows padded to 8 floats
  s.roff = s.ids + round16_(int64_t(2) * idsn * 4);
  s.kept = s.roff + round16_(int64_t(2) * idsn * 4);
  s.koff = s.kept + round16_(int64_t(kept_cap) * 4);
  s.bw = s.koff + round16_(int64_t(kept_cap) * 4);
  s.cnt = s.bw + round16_(int64_t(kept_cap) * 4);  // 5 counters, the loss, a pair's claim
  s.cand = s.cnt + 64;
  s.total = (s.cand + kCandWords * 4 + 31) & ~int64_t(31);  // slabs keep the 32-byte phase
  return s;
}

// one window unit of a sentence: kept position pos, chunk index ch
struct Unit {
  int pos, ch, wlo, left, m, start, mc;
};

__device__ __forceinline__ bool unit_at(const int *bw_s, int nk, int cap, int pos, int ch, Unit &u) {
  const int b = bw_s[pos];
  const int wlo = max(pos - b, 0);
  const int whi = min(pos + b + 1, nk);
  const int m = whi - wlo - 1;
  if (m <= 0 || ch * cap >= m) return false;
  u.pos = pos;
  u.ch = ch;
  u.wlo = wlo;
  u.left = pos - wlo;
  u.m = m;
  u.start = ch * cap;
  u.mc = min(cap, m - u.start);
  return true;
}
// next unit after (pos, ch) in the reference's order; false at the end of the sentence
__device__ __forceinline__ bool next_unit(const int *bw_s, int nk, int cap, const Unit &cur, Unit &nx) {
  if (unit_at(bw_s, nk, cap, cur.pos, cur.ch + 1, nx)) return true;
  for (int pos = cur.pos + 1; pos < nk; ++pos)
    if (unit_at(bw_s, nk, cap, pos, 0, nx)) return true;
  return false;
}
__device__ __forceinline__ bool first_unit(const int *bw_s, int nk, int cap, Unit &nx) {
  for (int pos = 0; pos < nk; ++pos)
    if (unit_at(bw_s, nk, cap, pos, 0, nx)) return true;
  return false;
}

// Candidate negative draws of one unit: lane j evaluates attempt (attempt0 + j).  The
// alias-table loads are returned raw and only combined at use time, so a prefetched
// candidate keeps its two loads in flight while the current window computes.
struct NegCand {
  uint32_t bucket, coin, thr;
  int alias;
  __device__ __forceinline__ int word() const { return coin < thr ? (int)bucket : alias; }
};
__device__ __forceinline__ NegCand neg_candidate(const FastArgs &p, uint64_t tok, uint32_t ep, int ch,
                                                 uint32_t a) {
  const uint4 o = philox_tok(tok, ep, kTagNeg | ((uint32_t)(ch & 0xFF) << 16) | ((a >> 1) & 0xFFFFu),
                             p.key0, p.key1);
  NegCand c;
  const uint32_t bw = (a & 1) ? o.z : o.x;
  c.coin = (a & 1) ? o.w : o.y;
  c.bucket = (uint32_t)(((uint64_t)bw * (uint64_t)p.vocab) >> 32);
  c.thr = __ldg(p.alias_thr + c.bucket);
  c.alias = __ldg(p.alias_idx + c.bucket);
  return c;
}
__device__ __forceinline__ NegCand no_candidate() {
  NegCand c;
  c.bucket = 0; c.coin = 0; c.thr = 0; c.alias = -1;  // word() == -1
  return c;
}

// Accept the first k_neg candidates != target (kernel_batched.py:57-66 semantics, with
// the attempt sequence of the oracle's philox restatement); writes ids_s[mc+1 ...].
// cand / span: this lane's candidate of attempts [0, span) (lanes >= span: ignored).
__device__ __forceinline__ void select_negatives(const FastArgs &p, int cand, int span, uint64_t tok,
                                                 uint32_t ep, int ch, int target, int *ids_s, int mc, int lane) {
  const unsigned lt = (1u << lane) - 1u;
  int need = p.k_neg;
  uint32_t attempt = 0;
  while (true) {
    const bool ok = lane < span && cand != target;
    const unsigned mask = __ballot_sync(0xffffffffu, ok);
    const int avail = __popc(mask);
    const int take = min(avail, need);
    const int rank = __popc(mask & lt);
    if (ok && rank < take) ids_s[mc + 1 + (p.k_neg - need) + rank] = cand;
    need -= take;
    if (need == 0) break;
    attempt += (uint32_t)span;  // every candidate of this span was consumed
    if (attempt >= kMaxNegAttempts) {
      // the counter holds 17 attempt bits: past them the candidate stream would repeat
      // (a target carrying almost all of the count^0.75 mass).  Flag it; fill the rest
      // deterministically so the launch still terminates.
      if (lane == 0 && p.error) atomicExch(p.error, 3);
      for (int r = lane; r < need; r += 32)
        ids_s[mc + 1 + (p.k_neg - need) + r] = (target + 1 + r) % (int)p.vocab;
      break;
    }
    span = min(32, need + 2);
    cand = lane < span ? neg_candidate(p, tok, ep, ch, attempt + lane).word() : -1;
  }
}

#ifndef SGNS_FAST_MAXNREG
#define SGNS_FAST_MAXNREG 128
#endif
#ifndef SGNS_FAST_MAXNREG_WIDE
#define SGNS_FAST_MAXNREG_WIDE 168
#endif
// FULL: the row holds exactly 32 * NS float2 slots (ld padded, e.g. 320 at d = 300), so
// every lane owns NS whole slots and no per-slot predicate is needed.
// Register cap: 128 (16 warps per SM) while the K1R x NS float2 output rows fit.  K1R = 7, 8
// (k1 = 7, 8) at NS >= 5 (d > 256) would spill under 128 (72-byte stack at d = 300 for the
// earlier padded K1R = 8 build, 144-424 bytes above), so they take up to 168 registers
// (12-13 warps per SM): K = 6 / 7 on the configs[2] corpus 142 / 139 -> 158 / 156 M words/s.
template <int NS, int K1R> struct FastRegs {
  static constexpr int v = (K1R > 6 && NS >= 5) ? SGNS_FAST_MAXNREG_WIDE : SGNS_FAST_MAXNREG;
};
// Warp pairs: with PAIR, a worker is TWO warps of the block (warps 2t, 2t+1) for
// K + 1 = 9..16 output rows: warp r holds output rows [r K1R, r K1R + kown) of every window
// in registers (K1R = ceil((K + 1) / 2)), so no warp needs more than 8 output rows of
// registers.  Both warps walk the same control stream (subsampling, windows, negatives:
// deterministic Philox, recomputed by each), stage their own copy of the window's input
// rows, and scatter their own dC rows and their partial dA_i = sum over their outputs.
// Two pair barriers per window keep the worker's order exact: after both copies of the
// window's rows are staged (no scatter of the window starts before both warps read its
// rows) and after both warps' scatters (the next window's gathers and output-row loads
// see both).  The leader warp (r = 0) alone claims sentences, counts, traces and marks rows.
__device__ __forceinline__ void pair_bar(int id) { asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory"); }

template <int NS, int NCH, int K1R, bool EXACT_K, bool FULL, bool PAIR = false>
__global__ void __maxnreg__((FastRegs<NS, K1R>::v)) drive_fast_kernel(FastArgs p) {
  constexpr int K1T = PAIR ? 2 * K1R : K1R;  // output ids held per window
  extern __shared__ __align__(128) unsigned char smem[];
  float *sig_s = reinterpret_cast<float *>(smem);
  for (int i = threadIdx.x; i < kSigBins; i += blockDim.x) sig_s[i] = p.sig[i];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wid = PAIR ? (blockIdx.x * p.wpb + warp) >> 1 : blockIdx.x * p.wpb + warp;
  if (wid >= p.n_workers) return;
  const bool lead = !PAIR || (warp & 1) == 0;
  const int bar_id = 1 + (warp >> 1);  // PAIR: named barrier of this warp pair
  const int k1 = PAIR ? p.k_neg + 1 : (EXACT_K ? K1R : p.k_neg + 1);  // outputs per window
  const int kbase = PAIR && !lead ? K1R : 0;                          // this warp's first output
  const int kown = PAIR ? (lead ? K1R : k1 - K1R) : k1;                // and how many
  const int mcap = min(p.cap, 2 * p.window);
  const FastSlab L = fast_slab(fast_lds(p.mv.nvec), mcap, K1T, p.kept_cap);
  unsigned char *base = smem + round16_(kSigBins * 4) + (int64_t)warp * L.total;
  // PAIR: ONE staged copy of the window's input rows per pair, in the leader's slab; each
  // warp gathers every other row (the pair barriers below order it against both readers)
  float *rows_s = reinterpret_cast<float *>(
      (PAIR ? smem + round16_(kSigBins * 4) + (int64_t)(warp & ~1) * L.total : base) + L.rows);
  float *e_s = reinterpret_cast<float *>(base + L.e);
  int *ids_b = reinterpret_cast<int *>(base + L.ids);
  uint32_t *roff_b = reinterpret_cast<uint32_t *>(base + L.roff);
  int *kept_s = reinterpret_cast<int *>(base + L.kept);
  int *koff_s = reinterpret_cast<int *>(base + L.koff);
  int *bw_s = reinterpret_cast<int *>(base + L.bw);
  int *cand_s = reinterpret_cast<int *>(base + L.cand);
  // words trained / read, chunks, inputs, and the current epoch's sampled loss cells and
  // loss sum of this worker: kept in shared memory (lane 0) rather than in 64-bit
  // registers live across the whole hot loop
  long long *cnt_s = reinterpret_cast<long long *>(base + L.cnt);
  double *loss_s = reinterpret_cast<double *>(cnt_s + 5);
  if (lane == 0) {
    cnt_s[0] = cnt_s[1] = cnt_s[2] = cnt_s[3] = cnt_s[4] = 0;
    *loss_s = 0.0;
  }
  // lane 0: move the current epoch's loss into the per-epoch and per-launch totals
  auto flush_epoch_loss = [&](int e) {
    if (lane == 0) {
      if (PAIR) {  // both warps of the pair sum into the worker's slots
        atomicAdd(p.loss_by_epoch + (int64_t)wid * p.epochs + e, *loss_s);
        atomicAdd(reinterpret_cast<unsigned long long *>(p.cells_by_epoch + (int64_t)wid * p.epochs + e),
                  (unsigned long long)cnt_s[4]);
      } else {
        p.loss_by_epoch[(int64_t)wid * p.epochs + e] += *loss_s;
        p.cells_by_epoch[(int64_t)wid * p.epochs + e] += cnt_s[4];
      }
      if (p.totals != nullptr) {
        atomicAdd(p.totals + 4, (unsigned long long)cnt_s[4]);
        atomicAdd(p.loss_total, *loss_s);
      }
      *loss_s = 0.0;
      cnt_s[4] = 0;
    }
  };
  const int idsn = mcap + K1T;
  const unsigned lt_mask = (1u << lane) - 1u;
  // nvec: 16-byte chunks of a row that hold data (dim rounded up to 4).  Staged rows are
  // packed at that width (rounded to 32 bytes, fast_lds) in shared memory (ld); in HBM a row starts every gld >= ld elements
  // (padded so rows start on 128-byte lines: every warp-wide access then covers whole lines).
  const int nvec = p.mv.nvec, nslot = 2 * nvec;
  const int ld = fast_lds(nvec);
  const uint32_t gld = (uint32_t)p.mv.ld;
  // lane offsets folded into the model base pointers once: every gather/scatter below is
  // base + 32-bit row offset + a compile-time slot offset
  // Column layout of a lane's NS float2 slots: slots 2q, 2q + 1 are the halves of the
  // 16-byte chunk q (columns 128 q + 4 lane ..+3), an odd last slot is the float2 at
  // 128 NQ + 2 lane: rows move as 128-bit loads / RED.128 (2 + 1 instead of 5 at d = 300).
  constexpr int NQ = NS / 2;       // 16-byte chunks per lane
  constexpr int NT = NS - 2 * NQ;  // float2 slot after them (0 or 1)
  const int lane_col = 4 * lane;
  const int tail_adj = 128 * NQ - 2 * lane;  // the float2 slot relative to lane_col
  float *const in_dst_l = p.mv.in_dst + lane_col;
  float *const out_dst_l = p.mv.out_dst + lane_col;
  const float *const out_src_l = p.mv.out_src + lane_col;
  const float *const in_src_l = p.mv.in_src + 4 * lane;
  auto slot_ok = [&](int j) {
    if (FULL) return true;
    if (j >= 2 * NQ) return lane + 32 * j < nslot;  // the float2 slot
    return NT > 0 || j < 2 * NQ - 2 || lane + 32 * (NQ - 1) < nvec;
  };
  // row <- global (ld.cg), row <- shared, global += row; ptr = row base + lane_col
  auto row_ldg = [&](float2 (&r)[NS], const float *src, bool on) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (on && slot_ok(2 * q)) v = ld_cg_f4(src + 128 * q);
      r[2 * q] = make_float2(v.x, v.y);
      r[2 * q + 1] = make_float2(v.z, v.w);
    }
#pragma unroll
    for (int j = 2 * NQ; j < NS; ++j)
      r[j] = (on && slot_ok(j)) ? ld_cg_f2(src + tail_adj + 64 * (j - 2 * NQ)) : f2zero();
  };
  auto row_red = [&](float *dst, const float2 (&r)[NS], bool on) {
#pragma unroll
    for (int q = 0; q < NQ; ++q)
      if (on && slot_ok(2 * q))
        atomicAdd(reinterpret_cast<float4 *>(dst + 128 * q),
                  make_float4(r[2 * q].x, r[2 * q].y, r[2 * q + 1].x, r[2 * q + 1].y));
#pragma unroll
    for (int j = 2 * NQ; j < NS; ++j)
      if (on && slot_ok(j)) atomicAdd(reinterpret_cast<float2 *>(dst + tail_adj + 64 * (j - 2 * NQ)), r[j]);
  };
  auto chunk_ok = [&](int j) { return j < NCH - 1 || lane + 32 * j < nvec; };
  auto kk_ok = [&](int k) { return EXACT_K || k < kown; };
  const int rec_len = 4 + p.cap + k1;
  // Negative candidates are drawn for a batch of consecutive kept positions at once: every
  // lane runs ONE Philox call (two attempts) and its alias lookups, so the first NCAND
  // attempts of WB chunk-0 windows cost one call per batch instead of one per window.
  // Attempt order and acceptance are unchanged (attempts 0, 1, 2, ... in order; attempts
  // past NCAND, and chunks after the first, are drawn directly in select_negatives).
  constexpr int NCAND = PAIR ? 16 : 8;        // >= K + 2 whenever possible
  constexpr int WB = kCandWords / NCAND;      // windows per batch
  // score reduction: value h * K1R + k of an input pair on the lanes TR::index gives
  using TR = TReduce<2 * K1R, 16>;

  int loss_epoch = -1;

  for (;;) {
    unsigned long long c = 0;
    if (lane == 0 && lead) c = atomicAdd(p.claim, 1ULL);
    if (PAIR) {  // the leader's claim, through its slab's spare counter slot
      volatile unsigned long long *xch = reinterpret_cast<unsigned long long *>(
          smem + round16_(kSigBins * 4) + (int64_t)(warp & ~1) * L.total + L.cnt) + 6;
      if (lane == 0 && lead) *xch = c;
      pair_bar(bar_id);
      c = *xch;
      pair_bar(bar_id);  // read before the leader's next claim overwrites it
    }
    c = __shfl_sync(0xffffffffu, c, 0);
    if ((int64_t)c >= p.claim_end) break;
    const int epoch = (int)((int64_t)c / p.n_sent);
    const int64_t s = p.shard_lo + (int64_t)c % p.n_sent;
    const int64_t lo_t = p.offsets[s], hi_t = p.offsets[s + 1];
    const int n = (int)(hi_t - lo_t);
    if (n > p.kept_cap) {
      if (lane == 0 && p.error) atomicExch(p.error, 2);
      continue;
    }
    const uint32_t ep = p.epoch_base + (uint32_t)epoch;
    if (lane == 0 && lead) cnt_s[1] += n;
    // alpha from the sentence's words-read position (update_alpha, trainer.py:122-132)
    // (the shard's bounds are re-read per sentence -- two cached loads -- rather than
    // held in four registers across the hot loop)
    const int64_t off0 = __ldg(p.offsets + p.shard_lo);
    const int64_t shard_tokens = __ldg(p.offsets + p.shard_lo + p.n_sent) - off0;
    const double pos_words = (double)(p.words_base + (int64_t)epoch * shard_tokens + (lo_t - off0));
    double frac = 1.0 - pos_words / (p.total_x_epochs + 1.0);
    if (frac < p.floor_frac) frac = p.floor_frac;
    const float alpha = (float)(p.alpha0 * frac);
    const bool want = p.loss_every > 0 && ((int64_t)c % p.loss_every) == 0;
    if (want && epoch != loss_epoch) {
      if (loss_epoch >= 0) flush_epoch_loss(loss_epoch);
      loss_epoch = epoch;
    }
    // subsample: one Philox uniform per token, survivors compacted in order
    int nk = 0;
    for (int b0 = 0; b0 < n; b0 += 32) {
      const int i = b0 + lane;
      const bool valid = i < n;
      const int w = valid ? p.ids[lo_t + i] : 0;
      bool keep = valid;
      if (p.keep != nullptr && valid) {
        const uint4 o = philox_tok((uint64_t)(p.token_base + lo_t + i), ep, kTagSub, p.key0, p.key1);
        keep = u53((uint64_t)o.x | ((uint64_t)o.y << 32)) < p.keep[w];
      }
      const unsigned mask = __ballot_sync(0xffffffffu, keep);
      if (keep) {
        const int q = nk + __popc(mask & lt_mask);
        kept_s[q] = w;
        koff_s[q] = i;
      }
      nk += __popc(mask);
    }
    __syncwarp();
    // dynamic half-widths of every kept position, lane-parallel
    for (int q = lane; q < nk; q += 32) {
      int b = p.window;
      if (p.dynamic) {
        const uint4 o = philox_tok((uint64_t)(p.token_base + lo_t + koff_s[q]), ep, kTagWin, p.key0, p.key1);
        b = 1 + (int)(((uint64_t)o.x * (uint64_t)p.window) >> 32);
      }
      bw_s[q] = b;
    }
    __syncwarp();
    if (lane == 0 && lead) cnt_s[0] += nk;

    // first-span candidate word of unit x for this lane; fresh: x is the first unit of its
    // batch to be drawn (the batch is filled then)
    auto batch_cand = [&](const Unit &x, bool fresh) {
      if (fresh) {
        const int b = x.pos / WB;
        __syncwarp();  // earlier reads of cand_s are done
        const int q = b * WB + lane / (NCAND / 2), cc = lane % (NCAND / 2);
        if (q < nk) {
          const uint4 o = philox_tok((uint64_t)(p.token_base + lo_t + koff_s[q]), ep, kTagNeg | (uint32_t)cc,
                                     p.key0, p.key1);
          const uint32_t b0 = (uint32_t)(((uint64_t)o.x * (uint64_t)p.vocab) >> 32);
          const uint32_t b1 = (uint32_t)(((uint64_t)o.z * (uint64_t)p.vocab) >> 32);
          const uint32_t t0 = __ldg(p.alias_thr + b0), t1 = __ldg(p.alias_thr + b1);
          const int a0 = __ldg(p.alias_idx + b0), a1 = __ldg(p.alias_idx + b1);
          *reinterpret_cast<int2 *>(cand_s + 2 * lane) = make_int2(o.y < t0 ? (int)b0 : a0, o.w < t1 ? (int)b1 : a1);
        }
        __syncwarp();
      }
      return lane < NCAND ? cand_s[(x.pos % WB) * NCAND + lane] : -1;
    };
    // u's negatives -> ids_s[mc + 1 ...]
    auto draw_negatives = [&](const Unit &x, int *ids_s, bool fresh) {
      const uint64_t tok = (uint64_t)(p.token_base + lo_t + koff_s[x.pos]);
      const int target = kept_s[x.pos];
      if (x.ch == 0) {
        const int cand = batch_cand(x, fresh);
        select_negatives(p, cand, NCAND, tok, ep, 0, target, ids_s, x.mc, lane);
      } else {
        const int span = min(32, p.k_neg + 2);
        const int cand = lane < span ? neg_candidate(p, tok, ep, x.ch, lane).word() : -1;
        select_negatives(p, cand, span, tok, ep, x.ch, target, ids_s, x.mc, lane);
      }
    };
    Unit u;
    if (!first_unit(bw_s, nk, p.cap, u)) continue;
    // window u's inputs + target + negatives (synchronous for the first unit)
    int cur = 0;
    {
      int *ids_s = ids_b;
      for (int r = lane; r < u.mc; r += 32) {
        const int q = u.start + r;
        ids_s[r] = q < u.left ? kept_s[u.wlo + q] : kept_s[u.pos + 1 + (q - u.left)];
      }
      if (lane == 0) ids_s[u.mc] = kept_s[u.pos];
      draw_negatives(u, ids_s, true);
      __syncwarp();
      for (int r = lane; r < u.mc + k1; r += 32) roff_b[r] = (uint32_t)ids_s[r] * gld;
      __syncwarp();
    }
    // C rows of u -> registers
    float2 c_reg[K1R][NS];
    {
      const uint32_t *off_s = roff_b;
#pragma unroll
      for (int k = 0; k < K1R; ++k)
        row_ldg(c_reg[k], out_src_l + off_s[u.mc + kbase + (kk_ok(k) ? k : 0)], kk_ok(k));
    }
    for (;;) {
      int *ids_s = ids_b + cur * idsn;
      const uint32_t *off_s = roff_b + cur * idsn;
      int *ids_n = ids_b + (cur ^ 1) * idsn;
      uint32_t *off_n = roff_b + (cur ^ 1) * idsn;
      const int m = u.mc;
      // A rows of u -> smem
      for (int r = PAIR ? (warp & 1) : 0; r < m; r += PAIR ? 2 : 1) {
        const float *src = in_src_l + off_s[r];
        float *dst = rows_s + r * ld + 4 * lane;
#pragma unroll
        for (int j = 0; j < NCH; ++j) {
          if (j < NCH - 1) cp_async16(dst + 128 * j, src + 128 * j);
          else cp_async16_if(chunk_ok(j), dst + 128 * j, src + 128 * j);
        }
      }
      if (p.dirty != nullptr && lead) {  // touched rows (data-parallel touched-row averaging)
        for (int r = lane; r < m + k1; r += 32) p.dirty[(r < m ? 0u : p.vocab) + (uint32_t)ids_s[r]] = 1;
      }
      Unit nx;
      const bool have = next_unit(bw_s, nk, p.cap, u, nx);
      if (lane == 0 && lead) {
        cnt_s[2] += 1;
        cnt_s[3] += m;
      }
      if (p.trace_cap > 0 && lead) {
        unsigned long long idx = 0;
        if (lane == 0) idx = atomicAdd(p.trace_count, 1ULL);
        idx = __shfl_sync(0xffffffffu, idx, 0);
        if ((int64_t)idx < p.trace_cap) {
          int32_t *rec = p.trace + (int64_t)idx * rec_len;
          for (int r = lane; r < rec_len; r += 32) {
            int v;
            if (r == 0) v = ids_s[m];
            else if (r == 1) v = m;
            else if (r == 2) v = (int)s;
            else if (r == 3) v = epoch;
            else if (r < 4 + p.cap) v = (r - 4) < m ? ids_s[r - 4] : -1;
            else v = ids_s[m + (r - 4 - p.cap)];
            rec[r] = v;
          }
          if (lane == 0) p.trace_alpha[idx] = (double)alpha;
        }
      }
      cp_async_wait_all();
      __syncwarp();
      if (PAIR) pair_bar(bar_id);  // both copies staged: no scatter of u before both read its rows

      // scores, errors, dA -- inputs in pairs so one transposed butterfly (16 values,
      // 5 serial shuffle stages) reduces both inputs' scores
      for (int i = 0; i < m; i += 2) {
        const bool two = i + 1 < m;
        float pp[2 * K1R];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int ii = two ? i + h : i;
          float2 a[NS];
          {
            const float *ap = rows_s + ii * ld + lane_col;
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
              const float4 v = slot_ok(2 * q) ? *reinterpret_cast<const float4 *>(ap + 128 * q)
                                              : make_float4(0.f, 0.f, 0.f, 0.f);
              a[2 * q] = make_float2(v.x, v.y);
              a[2 * q + 1] = make_float2(v.z, v.w);
            }
#pragma unroll
            for (int j = 2 * NQ; j < NS; ++j)
              a[j] = slot_ok(j) ? *reinterpret_cast<const float2 *>(ap + tail_adj + 64 * (j - 2 * NQ)) : f2zero();
          }
#pragma unroll
          for (int k = 0; k < K1R; ++k) {
            float2 acc = __fmul2_rn(a[0], c_reg[k][0]);
#pragma unroll
            for (int j = 1; j < NS; ++j) acc = __ffma2_rn(a[j], c_reg[k][j], acc);
            pp[h * K1R + k] = acc.x + acc.y;
          }
        }
        // value h * K1R + k lands on the lanes with TR::index == that value
        const float sc = TR::run(pp, lane);
        const int tr_v = TR::index(lane);
        const int hk = tr_v >= K1R ? 1 : 0, kk = tr_v < 0 ? K1R : tr_v - hk * K1R;
        float er = 0.f, es = 0.f;
        const bool live = kk < kown && (hk == 0 || two);
        cell_error_f32(sc, kk + kbase, alpha, sig_s, er, es, live);
        if (live) e_s[(i + hk) * 8 + kk] = es;  // replicas of a value store the same word
        if (want) {  // sampled sentence: warp-reduce this pair's softplus terms
          const bool mine = live && (lane & TR::kDupMask) == 0;  // one lane per value
          double sp = mine ? softplus(kk + kbase == 0 ? -(double)sc : (double)sc) : 0.0;
#pragma unroll
          for (int o = 16; o >= 1; o >>= 1) sp += __shfl_xor_sync(0xffffffffu, sp, o);
          const int nc = __popc(__ballot_sync(0xffffffffu, mine));
          if (lane == 0) {
            *loss_s += sp;
            cnt_s[4] += nc;
          }
        }
        // dA_i = sum_k (alpha err_ik) C_k (alpha folded into e, as batch_core_blas,
        // kernel_batched.py:92-144): the pair's error rows are broadcast from e_s
        __syncwarp();
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (h == 1 && !two) break;
          const float4 e03 = *reinterpret_cast<const float4 *>(e_s + (i + h) * 8);
          const float4 e47 = *reinterpret_cast<const float4 *>(e_s + (i + h) * 8 + 4);
          const float ev[8] = {e03.x, e03.y, e03.z, e03.w, e47.x, e47.y, e47.z, e47.w};
          float2 d[NS];
#pragma unroll
          for (int k = 0; k < K1R; ++k) {
            const float2 ek2 = make_float2(kk_ok(k) ? ev[k] : 0.f, kk_ok(k) ? ev[k] : 0.f);
#pragma unroll
            for (int j = 0; j < NS; ++j)
              d[j] = k == 0 ? __fmul2_rn(ek2, c_reg[0][j]) : __ffma2_rn(ek2, c_reg[k][j], d[j]);
          }
          row_red(in_dst_l + off_s[i + h], d, true);
        }
      }
      // u+1's inputs, target and negatives (its candidates' alias loads were in flight)
      if (have) {
        for (int r = lane; r < nx.mc; r += 32) {
          const int q = nx.start + r;
          ids_n[r] = q < nx.left ? kept_s[nx.wlo + q] : kept_s[nx.pos + 1 + (q - nx.left)];
        }
        if (lane == 0) ids_n[nx.mc] = kept_s[nx.pos];
        draw_negatives(nx, ids_n, nx.pos / WB != u.pos / WB);
        __syncwarp();
        for (int r = lane; r < nx.mc + k1; r += 32) off_n[r] = (uint32_t)ids_n[r] * gld;
      }
      __syncwarp();
      // dC_k = sum_i (alpha err_ik) A_i, input-outer: u's C registers are dead once dA is
      // out, so they hold the NS x K1R accumulators; each staged row slot and each error row
      // is read once, and the NS x K1R FFMA2 chains are independent.  u+1's output rows are
      // loaded after u's scatters (and, in pairs, after the pair barrier), so they read them:
      // no patching, and their latency overlaps u+1's input-row gather.
      {
        uint32_t orow[K1R];
#pragma unroll
        for (int k = 0; k < K1R; ++k) orow[k] = off_s[m + kbase + (kk_ok(k) ? k : 0)];
        float2 acc[NS][K1R];
        const float *ap = rows_s + lane_col;
        const float *ep = e_s;
#pragma unroll
        for (int j = 0; j < NS; ++j)
#pragma unroll
          for (int k = 0; k < K1R; ++k) acc[j][k] = f2zero();
        // (peeling the first row to FMUL2 instead of zeroing the accumulators spills at 128
        // registers: 234M vs 262M words/s)
        for (int i = 0; i < m; ++i, ap += ld, ep += 8) {
          const float4 e03 = *reinterpret_cast<const float4 *>(ep);
          const float4 e47 = *reinterpret_cast<const float4 *>(ep + 4);
          const float ev[8] = {e03.x, e03.y, e03.z, e03.w, e47.x, e47.y, e47.z, e47.w};
#pragma unroll
          for (int q = 0; q < NQ; ++q) {
            const float4 v = slot_ok(2 * q) ? *reinterpret_cast<const float4 *>(ap + 128 * q)
                                            : make_float4(0.f, 0.f, 0.f, 0.f);
            const float2 a0 = make_float2(v.x, v.y), a1 = make_float2(v.z, v.w);
#pragma unroll
            for (int k = 0; k < K1R; ++k)
              if (kk_ok(k)) {
                acc[2 * q][k] = __ffma2_rn(make_float2(ev[k], ev[k]), a0, acc[2 * q][k]);
                acc[2 * q + 1][k] = __ffma2_rn(make_float2(ev[k], ev[k]), a1, acc[2 * q + 1][k]);
              }
          }
          if (NT > 0) {
            const float2 a0 = slot_ok(2 * NQ) ? *reinterpret_cast<const float2 *>(ap + tail_adj) : f2zero();
#pragma unroll
            for (int k = 0; k < K1R; ++k)
              if (kk_ok(k)) acc[NS - 1][k] = __ffma2_rn(make_float2(ev[k], ev[k]), a0, acc[NS - 1][k]);
          }
        }
#pragma unroll
        for (int k = 0; k < K1R; ++k) {
          float2 r[NS];
#pragma unroll
          for (int j = 0; j < NS; ++j) r[j] = acc[j][k];
          row_red(out_dst_l + orow[k], r, kk_ok(k));
        }
      }
      __syncwarp();
      if (PAIR) pair_bar(bar_id);  // both warps' scatters of u precede every read of u+1
      if (!have) break;  // (u's C is dead across the dC pass on this path too)
#pragma unroll
      for (int k = 0; k < K1R; ++k)
        row_ldg(c_reg[k], out_src_l + off_n[nx.mc + kbase + (kk_ok(k) ? k : 0)], kk_ok(k));
      u = nx;
      cur ^= 1;
    }
  }
  // flush this worker's counters
  if (loss_epoch >= 0) flush_epoch_loss(loss_epoch);
  __syncwarp();
  const long long trained = cnt_s[0], read = cnt_s[1], chunks = cnt_s[2], inputs = cnt_s[3];
  if (!lead) return;
  if (lane == 0 && p.totals != nullptr) {
    atomicAdd(p.totals + 0, (unsigned long long)trained);
    atomicAdd(p.totals + 1, (unsigned long long)read);
    atomicAdd(p.totals + 2, (unsigned long long)chunks);
    atomicAdd(p.totals + 3, (unsigned long long)inputs);
  }
  if (lane == 0) {
    sgns_worker &o = p.workers[wid];
    o.kernel_counter += chunks;
    o.words_trained += trained;
    o.words_read += read;
    o.inputs += inputs;
  }
}

}  // namespace sgns
