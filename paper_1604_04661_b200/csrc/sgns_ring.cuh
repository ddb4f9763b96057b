// sgns_ring.cuh -- production driver, sentence-ring variant (float32, K + 1 <= 8, d <= 512,
// window <= 15).
//
// Same schedule, draws, alpha and loss sampling as drive_fast_kernel (sgns_fast.cuh); what
// changes is how the input rows reach shared memory and how the window's updates are
// applied:
//
//  * sentence ring.  Consecutive windows of a sentence share most of their context words
//    (kept positions [pos - b, pos + b]), so instead of gathering the m input rows of every
//    window, each warp keeps the M_in rows of kept positions [P - W, P + W + 1] in a ring
//    of R = 2W + 2 slots (slot = position mod R).  Finishing position P issues ONE row
//    (P + W + 2, into the slot of the now dead row P - W) by cp.async; entering a position
//    waits only for the row issued one position earlier, so the gather latency is hidden
//    behind a whole position's work and the input-row gather traffic drops from m rows per
//    window to one row per kept position.
//  * exact per-worker order.  A reference thread's window sees every update that thread
//    made before it (trainer.py:281-304 calls process_batch window by window).  The ring
//    copies are kept exact the same way the C-row prefetch is: every window adds its own
//    dA_i to the ring copy of input i (in the fused pass below) and, when another resident
//    ring position holds the same word (a repeated word within the ring span, found with
//    one __match_any_sync), also to that copy (inside the same pass).  Rows issued after a
//    window's scatters read them from memory (same-thread order), rows issued before are
//    patched.
//  * one fused column pass per window: for each column slot, dC_k = sum_i e_ik A_i and
//    dA_i = sum_k e_ik C_k (alpha folded into e, as batch_core_blas, kernel_batched.py:92-144)
//    come out of the same shared-memory reads; dA is scattered and written back into the
//    ring copy, dC is scattered, and the next window's output rows for that slot are loaded
//    into the C registers just freed (loaded before this window's dC scatter and patched
//    where the two windows share an output row, as in drive_fast_kernel).
#pragma once

#include "sgns_fast.cuh"

namespace sgns {

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_async_wait_group() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// per-input record in shared memory: ES floats = e_0..e_{K1R-1} (alpha * err), padding,
// then the input's global row offset (id * ld) and its ring offset (slot * ld) as bits
template <int K1R> struct RingRec {
  static constexpr int ES = K1R <= 6 ? 8 : 12;
  static constexpr int GOFF = ES - 2, ROFF = ES - 1;
};

struct RingSlab {
  int64_t ring, rec, pm, ids, roff, kept, koff, bw, cnt, total;
};
__host__ __device__ inline RingSlab ring_slab(int64_t ld, int nring, int mcap, int k1r, int kept_cap) {
  RingSlab s;
  const int idsn = mcap + k1r;
  const int es = k1r <= 6 ? 8 : 12;
  s.ring = 0;
  s.rec = round16_(int64_t(nring) * ld * 4);
  s.pm = s.rec + round16_(int64_t(mcap + 1) * es * 4);
  s.ids = s.pm + round16_(int64_t(mcap) * 4);
  s.roff = s.ids + round16_(int64_t(2) * idsn * 4);
  s.kept = s.roff + round16_(int64_t(2) * idsn * 4);
  s.koff = s.kept + round16_(int64_t(kept_cap) * 4);
  s.bw = s.koff + round16_(int64_t(kept_cap) * 4);
  s.cnt = s.bw + round16_(int64_t(kept_cap) * 4);
  s.total = s.cnt + 48;
  return s;
}

#ifndef SGNS_RING_MAXNREG
#define SGNS_RING_MAXNREG 128
#endif
#ifndef SGNS_RING_PREFETCH_REC
#define SGNS_RING_PREFETCH_REC 0
#endif
#ifndef SGNS_RING_MAXNREG_WIDE
#define SGNS_RING_MAXNREG_WIDE 168
#endif
template <int NS, int K1R> struct RingRegs {
  static constexpr int v = (K1R > 6 && NS >= 5) ? SGNS_RING_MAXNREG_WIDE : SGNS_RING_MAXNREG;
};

template <int NS, int NCH, int K1R, bool EXACT_K, bool FULL>
__global__ void __maxnreg__((RingRegs<NS, K1R>::v)) drive_ring_kernel(FastArgs p) {
  constexpr int NV = 8;
  constexpr int ES = RingRec<K1R>::ES, GOFF = RingRec<K1R>::GOFF, ROFF = RingRec<K1R>::ROFF;
  extern __shared__ __align__(16) unsigned char smem[];
  float *sig_s = reinterpret_cast<float *>(smem);
  for (int i = threadIdx.x; i < kSigBins; i += blockDim.x) sig_s[i] = p.sig[i];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wid = blockIdx.x * p.wpb + warp;
  if (wid >= p.n_workers) return;
  const int k1 = EXACT_K ? K1R : p.k_neg + 1;
  const int W = p.window;
  const int R = 2 * W + 2;  // ring slots (<= 32: host-checked)
  const int mcap = min(p.cap, 2 * W);
  const RingSlab L = ring_slab(p.mv.ld, R, mcap, K1R, p.kept_cap);
  unsigned char *base = smem + round16_(kSigBins * 4) + (int64_t)warp * L.total;
  float *ring_s = reinterpret_cast<float *>(base + L.ring);
  float *rec_s = reinterpret_cast<float *>(base + L.rec);
  int *pm_s = reinterpret_cast<int *>(base + L.pm);
  int *ids_b = reinterpret_cast<int *>(base + L.ids);
  uint32_t *roff_b = reinterpret_cast<uint32_t *>(base + L.roff);
  int *kept_s = reinterpret_cast<int *>(base + L.kept);
  int *koff_s = reinterpret_cast<int *>(base + L.koff);
  int *bw_s = reinterpret_cast<int *>(base + L.bw);
  long long *cnt_s = reinterpret_cast<long long *>(base + L.cnt);
  double *loss_s = reinterpret_cast<double *>(cnt_s + 5);
  if (lane == 0) {
    cnt_s[0] = cnt_s[1] = cnt_s[2] = cnt_s[3] = cnt_s[4] = 0;
    *loss_s = 0.0;
  }
  auto flush_epoch_loss = [&](int e) {
    if (lane == 0) {
      p.loss_by_epoch[(int64_t)wid * p.epochs + e] += *loss_s;
      p.cells_by_epoch[(int64_t)wid * p.epochs + e] += cnt_s[4];
      if (p.totals != nullptr) {
        atomicAdd(p.totals + 4, (unsigned long long)cnt_s[4]);
        atomicAdd(p.loss_total, *loss_s);
      }
      *loss_s = 0.0;
      cnt_s[4] = 0;
    }
  };
  const int idsn = mcap + K1R;
  const unsigned lt_mask = (1u << lane) - 1u;
  const int ld = (int)p.mv.ld;
  const int nvec = p.mv.nvec, nslot = 2 * nvec;
  float *const in_dst_l = p.mv.in_dst + 2 * lane;
  float *const out_dst_l = p.mv.out_dst + 2 * lane;
  const float *const out_src_l = p.mv.out_src + 2 * lane;
  const float *const in_src_l = p.mv.in_src + 4 * lane;
  auto slot_ok = [&](int j) { return FULL || j < NS - 1 || lane + 32 * j < nslot; };
  auto chunk_ok = [&](int j) { return j < NCH - 1 || lane + 32 * j < nvec; };
  auto kk_ok = [&](int k) { return EXACT_K || k < k1; };
  const int rec_len = 4 + p.cap + k1;

  int loss_epoch = -1;

  for (;;) {
    unsigned long long c = 0;
    if (lane == 0) c = atomicAdd(p.claim, 1ULL);
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
    if (lane == 0) cnt_s[1] += n;
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
    for (int q = lane; q < nk; q += 32) {
      int b = p.window;
      if (p.dynamic) {
        const uint4 o = philox_tok((uint64_t)(p.token_base + lo_t + koff_s[q]), ep, kTagWin, p.key0, p.key1);
        b = 1 + (int)(((uint64_t)o.x * (uint64_t)p.window) >> 32);
      }
      bw_s[q] = b;
    }
    __syncwarp();
    if (lane == 0) cnt_s[0] += nk;

    Unit u;
    if (!first_unit(bw_s, nk, p.cap, u)) continue;
    // ring: M_in rows of kept positions [0, issued) have been issued
    int issued = 0;
    auto issue_row = [&](int q) {
      float *dst = ring_s + (q % R) * ld + 4 * lane;
      const float *src = in_src_l + (uint32_t)kept_s[q] * (uint32_t)ld;
#pragma unroll
      for (int j = 0; j < NCH; ++j)
        if (chunk_ok(j)) cp_async16(dst + 128 * j, src + 128 * j);
    };
    int cur = 0;
    {
      int *ids_s = ids_b;
      for (int r = lane; r < u.mc; r += 32) {
        const int q = u.start + r;
        ids_s[r] = q < u.left ? kept_s[u.wlo + q] : kept_s[u.pos + 1 + (q - u.left)];
      }
      const int target = kept_s[u.pos];
      if (lane == 0) ids_s[u.mc] = target;
      const uint64_t tok = (uint64_t)(p.token_base + lo_t + koff_s[u.pos]);
      const NegCand cand = lane < min(32, p.k_neg + 2) ? neg_candidate(p, tok, ep, u.ch, lane) : no_candidate();
      select_negatives(p, cand, tok, ep, u.ch, target, ids_s, u.mc, lane);
      __syncwarp();
      for (int r = lane; r < u.mc + k1; r += 32) roff_b[r] = (uint32_t)ids_s[r] * (uint32_t)ld;
      __syncwarp();
    }
    float2 c_reg[K1R][NS];
    {
      const uint32_t *off_s = roff_b;
#pragma unroll
      for (int k = 0; k < K1R; ++k) {
        const float *src = out_src_l + off_s[u.mc + (kk_ok(k) ? k : 0)];
#pragma unroll
        for (int j = 0; j < NS; ++j)
          c_reg[k][j] = (kk_ok(k) && slot_ok(j)) ? ld_cg_f2(src + 64 * j) : f2zero();
      }
    }
    bool have = true;
    while (have) {
      int *ids_s = ids_b + cur * idsn;
      const uint32_t *off_s = roff_b + cur * idsn;
      int *ids_n = ids_b + (cur ^ 1) * idsn;
      uint32_t *off_n = roff_b + (cur ^ 1) * idsn;
      const int m = u.mc;
      // ring: the first unit of a sentence issues its span [0, pos + W] and the look-ahead
      // row pos + W + 1 as two groups; afterwards each finished position issues row
      // pos + W + 2 (below), so entering a position only waits for the row issued one
      // position earlier (wait_group 1 further down)
      if (issued == 0) {
        const int need = min(u.pos + W + 1, nk), ahead = min(u.pos + W + 2, nk);
        for (; issued < need; ++issued) issue_row(issued);
        cp_async_commit();
        for (; issued < ahead; ++issued) issue_row(issued);
        cp_async_commit();
      }
      // input records: global row offset and ring offset of every input of u
      const int c0 = u.start;  // context index of input 0
      if (lane < m) {
        const int ci = c0 + lane;
        const int q = ci < u.left ? u.wlo + ci : u.pos + 1 + (ci - u.left);
        rec_s[lane * ES + GOFF] = __uint_as_float(off_s[lane]);
        rec_s[lane * ES + ROFF] = __uint_as_float((uint32_t)((q % R) * ld));
      }
      // repeated words among the resident ring positions [pos - W, pos + W + 1]: an input
      // whose word also sits at another resident position must patch that copy too
      unsigned dup_any;
      {
        const int q = u.pos - W + lane;
        const bool res = lane < R && q >= 0 && q < issued;
        const int wv = res ? kept_s[q] : -1 - lane;
        const unsigned mm = __match_any_sync(0xffffffffu, wv);
        const int ci = q < u.pos ? q - u.wlo : q - u.wlo - 1;
        const bool is_in = res && q != u.pos && q >= u.wlo && ci >= c0 && ci < c0 + m &&
                           q <= u.pos + (u.m - u.left);
        const unsigned partners = is_in ? (mm & ~(1u << lane)) : 0u;
        dup_any = __ballot_sync(0xffffffffu, partners != 0u);
        if (dup_any && is_in) pm_s[ci - c0] = (int)partners;
        // lane t <-> position pos - W + t; partner bits are lanes.  Lane R - 1 is the
        // look-ahead row, possibly still in flight: waited for below before any patch.
      }
      if (p.dirty != nullptr) {
        for (int r = lane; r < m + k1; r += 32) p.dirty[(r < m ? 0u : p.vocab) + (uint32_t)ids_s[r]] = 1;
      }
      Unit nx;
      have = next_unit(bw_s, nk, p.cap, u, nx);
      NegCand cand_n = no_candidate();
      uint64_t tok_n = 0;
      if (have) {
        tok_n = (uint64_t)(p.token_base + lo_t + koff_s[nx.pos]);
        if (lane < min(32, p.k_neg + 2)) cand_n = neg_candidate(p, tok_n, ep, nx.ch, lane);
      }
      if (lane == 0) {
        cnt_s[2] += 1;
        cnt_s[3] += m;
      }
      if (p.trace_cap > 0) {
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
      cp_async_wait_group<1>();  // everything but the newest look-ahead row
      __syncwarp();

      // scores and errors, inputs in pairs (one 16-value transposed butterfly per pair)
      for (int i = 0; i < m; i += 2) {
        const bool two = i + 1 < m;
        float pp[2 * NV];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int ii = two ? i + h : i;
          const float *arow = ring_s + __float_as_uint(rec_s[ii * ES + ROFF]) + 2 * lane;
          float2 a[NS];
#pragma unroll
          for (int j = 0; j < NS; ++j)
            a[j] = slot_ok(j) ? *reinterpret_cast<const float2 *>(arow + 64 * j) : f2zero();
#pragma unroll
          for (int k = 0; k < NV; ++k) {
            if (k < K1R) {
              float2 acc = __fmul2_rn(a[0], c_reg[k][0]);
#pragma unroll
              for (int j = 1; j < NS; ++j) acc = __ffma2_rn(a[j], c_reg[k][j], acc);
              pp[h * NV + k] = acc.x + acc.y;
            } else {
              pp[h * NV + k] = 0.f;
            }
          }
        }
        const float sc = transpose_reduce<2 * NV>(pp, lane);
        const int v = reduced_index<2 * NV>(lane);
        const int hk = v >> 3, kk = v & 7;
        float er = 0.f, es = 0.f;
        const bool live = kk < k1 && (hk == 0 || two);
        cell_error_f32(sc, kk, alpha, sig_s, er, es);
        if (live && (lane & 1) == 0) rec_s[(i + hk) * ES + kk] = es;
        if (want) {
          const bool mine = live && (lane & 1) == 0;
          double sp = mine ? softplus(kk == 0 ? -(double)sc : (double)sc) : 0.0;
#pragma unroll
          for (int o = 16; o >= 1; o >>= 1) sp += __shfl_xor_sync(0xffffffffu, sp, o);
          const int nc = __popc(__ballot_sync(0xffffffffu, mine));
          if (lane == 0) {
            *loss_s += sp;
            cnt_s[4] += nc;
          }
        }
      }
      // u+1's inputs, target and negatives (its candidates' alias loads were in flight)
      unsigned lo_bits = 0, hi_bits = 0;
      if (have) {
        for (int r = lane; r < nx.mc; r += 32) {
          const int q = nx.start + r;
          ids_n[r] = q < nx.left ? kept_s[nx.wlo + q] : kept_s[nx.pos + 1 + (q - nx.left)];
        }
        const int target = kept_s[nx.pos];
        if (lane == 0) ids_n[nx.mc] = target;
        select_negatives(p, cand_n, tok_n, ep, nx.ch, target, ids_n, nx.mc, lane);
        __syncwarp();
        for (int r = lane; r < nx.mc + k1; r += 32) off_n[r] = (uint32_t)ids_n[r] * (uint32_t)ld;
        const int kq = lane & 7, ka = lane >> 3, kb = 4 + (lane >> 3);
        const bool h1 = ka < k1 && kq < k1 && ids_s[m + ka] == ids_n[nx.mc + kq];
        const bool h2 = kb < k1 && kq < k1 && ids_s[m + kb] == ids_n[nx.mc + kq];
        lo_bits = __ballot_sync(0xffffffffu, h1);
        hi_bits = __ballot_sync(0xffffffffu, h2);
      }
      __syncwarp();
      // fused pass: per column slot, dC and dA from the same reads; dA into memory and into
      // the ring copy; then u+1's output rows for this slot (before u's dC scatter, patched)
      const bool pf = have;
      if (dup_any) {
        cp_async_wait_all();  // a partner copy may be the in-flight look-ahead row
        __syncwarp();
      }
      const int slot0 = dup_any ? ((u.pos - W) % R + R) % R : 0;
      uint32_t orow[K1R];
#pragma unroll
      for (int k = 0; k < K1R; ++k) orow[k] = off_s[m + (kk_ok(k) ? k : 0)];
      const uint32_t *nrow = off_n + (pf ? nx.mc : 0);  // read per slot from shared memory
#pragma unroll
      for (int j = 0; j < NS; ++j) {
        if (!slot_ok(j)) continue;
        float2 acc[K1R];
#pragma unroll
        for (int k = 0; k < K1R; ++k) acc[k] = f2zero();
        const float *rp = rec_s;
#if SGNS_RING_PREFETCH_REC
        float4 r0 = *reinterpret_cast<const float4 *>(rp);
        float4 r1 = *reinterpret_cast<const float4 *>(rp + 4);
        float4 r2 = ES > 8 ? *reinterpret_cast<const float4 *>(rp + 8) : make_float4(0.f, 0.f, 0.f, 0.f);
#endif
        for (int i = 0; i < m; ++i) {
#if !SGNS_RING_PREFETCH_REC
          const float4 r0 = *reinterpret_cast<const float4 *>(rp);
          const float4 r1 = *reinterpret_cast<const float4 *>(rp + 4);
          const float4 r2 = ES > 8 ? *reinterpret_cast<const float4 *>(rp + 8) : make_float4(0.f, 0.f, 0.f, 0.f);
#endif
          const float ev[12] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w, r2.x, r2.y, r2.z, r2.w};
          const uint32_t goff = __float_as_uint(ev[GOFF]);
          float *ap = ring_s + __float_as_uint(ev[ROFF]) + 2 * lane + 64 * j;
          const float2 a0 = *reinterpret_cast<const float2 *>(ap);
          rp += ES;
#if SGNS_RING_PREFETCH_REC
          // next record (the array holds one spare record past mcap)
          r0 = *reinterpret_cast<const float4 *>(rp);
          r1 = *reinterpret_cast<const float4 *>(rp + 4);
          if (ES > 8) r2 = *reinterpret_cast<const float4 *>(rp + 8);
#endif
          float2 d = __fmul2_rn(make_float2(ev[0], ev[0]), c_reg[0][j]);
#pragma unroll
          for (int k = 1; k < K1R; ++k)
            if (kk_ok(k)) d = __ffma2_rn(make_float2(ev[k], ev[k]), c_reg[k][j], d);
#pragma unroll
          for (int k = 0; k < K1R; ++k)
            if (kk_ok(k)) acc[k] = __ffma2_rn(make_float2(ev[k], ev[k]), a0, acc[k]);
          atomicAdd(reinterpret_cast<float2 *>(in_dst_l + goff + 64 * j), d);
          *reinterpret_cast<float2 *>(ap) = __fadd2_rn(a0, d);
        }
        if (dup_any) {
          // a word repeated within the ring span: add each such input's dA (recomputed
          // bit-identically from its record and u's C, still in registers for this slot)
          // to the other resident copies of its word
          for (int i = 0; i < m; ++i) {
            const unsigned partners = (unsigned)pm_s[i];
            if (partners == 0u) continue;
            const float *rq = rec_s + i * ES;
            float2 d = __fmul2_rn(make_float2(rq[0], rq[0]), c_reg[0][j]);
#pragma unroll
            for (int k = 1; k < K1R; ++k)
              if (kk_ok(k)) d = __ffma2_rn(make_float2(rq[k], rq[k]), c_reg[k][j], d);
            for (unsigned b = partners; b; b &= b - 1) {
              int sl = slot0 + __ffs(b) - 1;
              sl = sl >= R ? sl - R : sl;
              float2 *cp = reinterpret_cast<float2 *>(ring_s + sl * ld + 2 * lane + 64 * j);
              *cp = __fadd2_rn(*cp, d);
            }
          }
        }
        if (pf) {
#pragma unroll
          for (int k = 0; k < K1R; ++k)
            c_reg[k][j] = kk_ok(k) ? ld_cg_f2(out_src_l + nrow[k] + 64 * j) : f2zero();
        }
#pragma unroll
        for (int k = 0; k < K1R; ++k)
          if (kk_ok(k)) atomicAdd(reinterpret_cast<float2 *>(out_dst_l + orow[k] + 64 * j), acc[k]);
        if (pf && (lo_bits | hi_bits)) {
#pragma unroll
          for (int k = 0; k < K1R; ++k) {
            const unsigned row = k < 4 ? (lo_bits >> (8 * k)) & 0xFFu : (hi_bits >> (8 * (k - 4))) & 0xFFu;
            if (row) {
#pragma unroll
              for (int kq = 0; kq < K1R; ++kq)
                if (row & (1u << kq)) c_reg[kq][j] = __fadd2_rn(c_reg[kq][j], acc[k]);
            }
          }
        }
      }
      __syncwarp();
      // position finished (no further chunk): its oldest ring row is dead, so the slot
      // takes row pos + W + 2 -- issued after this position's scatters, so it reads them
      if ((!have || nx.pos != u.pos) && issued < nk) {
        issue_row(issued++);
        cp_async_commit();
      }
      if (have) {
        u = nx;
        cur ^= 1;
      }
    }
    cp_async_wait_all();  // no copy may still target the ring when the next sentence starts
    __syncwarp();
  }
  if (loss_epoch >= 0) flush_epoch_loss(loss_epoch);
  __syncwarp();
  const long long trained = cnt_s[0], read = cnt_s[1], chunks = cnt_s[2], inputs = cnt_s[3];
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
