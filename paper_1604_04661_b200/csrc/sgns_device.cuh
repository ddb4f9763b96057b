// sgns_device.cuh -- device building blocks of the pSGNScc hot path (sm_100a).
//
// One warp = one worker; a window (<= batch_cap inputs sharing the target + K
// negatives) is processed by one warp.  Two window-update paths:
//  * window_update_f2 (float32, K + 1 <= 8, d <= 512): input rows staged in shared
//    memory by 16-byte cp.async, output rows loaded straight into registers, packed
//    FFMA2 math on a float2 column map, a transposed butterfly reducing two inputs'
//    scores at once, dA and dC scattered with red.global.add.v2.f32.  The production
//    driver (sgns_fast.cuh) inlines the same math.
//  * window_update (generic: float64, K + 1 > 8, d > 512): every row staged in shared
//    memory, 16-byte vector math, scores reduced over 32 values.
// Both gather every row before any write (the snapshot semantics of
// kernel_batched.py:104-113), compute E = alpha (label - sigma(S)) with the
// reference's float64 bin rule (model.py:108-115) or the exact sigmoid
// (kernel_scalar.py:30-35), and apply dA = alpha sum_k err C_k and
// dC = sum_i (alpha err) A_i additively (kernel_batched.py:135-143, :191-210).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace sgns {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;
constexpr uint64_t kMix1 = 0xBF58476D1CE4E5B9ULL;
constexpr uint64_t kMix2 = 0x94D049BB133111EBULL;
constexpr uint32_t kTagSub = 0x53554230u;  // 'SUB0'
constexpr uint32_t kTagWin = 0x57494E30u;  // 'WIN0'
constexpr uint32_t kTagNeg = 0x4E000000u;
// negative draws: counter word 2 = kTagNeg | chunk (8 bits) << 16 | attempt pair (16 bits),
// so a unit may consume at most 2^17 candidate draws (device error 3 past that)
constexpr uint32_t kMaxNegAttempts = 1u << 17;
constexpr int kSigBins = 1000;

template <typename T> struct Vec;
template <> struct Vec<float> {
  using type = float4;
  static constexpr int N = 4;
};
template <> struct Vec<double> {
  using type = double2;
  static constexpr int N = 2;
};

// ---------------------------------------------------------------- RNG ----
// splitmix64 exactly as rng.py:24-32; draw n of a stream in state s is
// mix(s + (n+1) * golden), so a warp can evaluate 32 consecutive draws at once.
__device__ __forceinline__ uint64_t sm_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * kMix1;
  z = (z ^ (z >> 27)) * kMix2;
  return z ^ (z >> 31);
}
__device__ __forceinline__ double u53(uint64_t z) {
  return (double)(z >> 11) * (1.0 / 9007199254740992.0);
}

// Philox4x32-10 (Salmon et al. 2011); counter = (token lo, token hi, epoch, tag).
__device__ __forceinline__ uint4 philox(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
  }
  return c;
}
__device__ __forceinline__ uint4 philox_tok(uint64_t tok, uint32_t epoch, uint32_t tag,
                                            uint32_t k0, uint32_t k1) {
  return philox(make_uint4((uint32_t)tok, (uint32_t)(tok >> 32), epoch, tag), k0, k1);
}

// ------------------------------------------------------------ helpers ----
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
// predicated form (no branch around the copy)
__device__ __forceinline__ void cp_async16_if(bool on, void *smem, const void *gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %2, 0;\n @p cp.async.cg.shared.global [%0], [%1], 16;\n}\n" ::"r"(s),
      "l"(gmem), "r"((int)on)
      : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}

__device__ __forceinline__ float4 vzero(float) { return make_float4(0.f, 0.f, 0.f, 0.f); }
__device__ __forceinline__ double2 vzero(double) { return make_double2(0.0, 0.0); }
__device__ __forceinline__ float vdot(const float4 &a, const float4 &b) {
  return fmaf(a.w, b.w, fmaf(a.z, b.z, fmaf(a.y, b.y, a.x * b.x)));
}
__device__ __forceinline__ double vdot(const double2 &a, const double2 &b) {
  return fma(a.y, b.y, a.x * b.x);
}
__device__ __forceinline__ void vfma(float4 &acc, float s, const float4 &v) {
  acc.x = fmaf(s, v.x, acc.x);
  acc.y = fmaf(s, v.y, acc.y);
  acc.z = fmaf(s, v.z, acc.z);
  acc.w = fmaf(s, v.w, acc.w);
}
__device__ __forceinline__ void vfma(double2 &acc, double s, const double2 &v) {
  acc.x = fma(s, v.x, acc.x);
  acc.y = fma(s, v.y, acc.y);
}
__device__ __forceinline__ void vscale(float4 &v, float s) {
  v.x *= s; v.y *= s; v.z *= s; v.w *= s;
}
__device__ __forceinline__ void vscale(double2 &v, double s) {
  v.x *= s; v.y *= s;
}
// Scatter-add one 16-byte chunk (no return value -> REDG.E.ADD.F32x4).
__device__ __forceinline__ void red_add(float *p, const float4 &v) {
  atomicAdd(reinterpret_cast<float4 *>(p), v);
}
__device__ __forceinline__ void red_add(double *p, const double2 &v) {
  atomicAdd(p, v.x);
  atomicAdd(p + 1, v.y);
}

// Transposed butterfly: NV partial sums per lane -> each lane ends with the
// full warp sum of value index (lane >> (5 - log2 NV)) & (NV - 1).
template <int NV> struct Log2 { static constexpr int v = 1 + Log2<NV / 2>::v; };
template <> struct Log2<1> { static constexpr int v = 0; };

template <int NV, typename T>
__device__ __forceinline__ T transpose_reduce(T (&v)[NV], int lane) {
  constexpr int L = Log2<NV>::v;
#pragma unroll
  for (int s = 0; s < L; ++s) {
    const int half = NV >> (s + 1);
    const int bit = 16 >> s;
    const bool upper = (lane & bit) != 0;
#pragma unroll
    for (int q = 0; q < half; ++q) {
      const T send = upper ? v[q] : v[q + half];
      const T keep = upper ? v[q + half] : v[q];
      v[q] = keep + __shfl_xor_sync(0xffffffffu, send, bit);
    }
  }
#pragma unroll
  for (int bit = 16 >> L; bit >= 1; bit >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], bit);
  return v[0];
}
template <int NV> __device__ __forceinline__ int reduced_index(int lane) {
  return (lane >> (5 - Log2<NV>::v)) & (NV - 1);
}
template <int NV> __device__ __forceinline__ int group_leader(int k) {
  return k << (5 - Log2<NV>::v);
}

// Transposed butterfly over any N <= 32 values (N need not be a power of two): each stage
// halves the value count (rounding up) across one lane bit, then plain butterflies finish.
// N = 12 (two inputs x six outputs) takes 6 + 3 + 2 + 1 + 1 = 13 shuffles where the padded
// power-of-two form takes 16.  index(lane): which value the lane ends with, -1 for the
// lanes an odd split leaves without one; kDupMask: lane bits over which a value is
// replicated (the plain stages).
template <int N, int BIT> struct TReduce {
  static constexpr int H = (N + 1) / 2;
  static constexpr int kDupMask = N == 1 ? (BIT | TReduce<1, BIT / 2>::kDupMask) : TReduce<H, BIT / 2>::kDupMask;
  template <int NMAX>
  static __device__ __forceinline__ float run(float (&v)[NMAX], int lane) {
    if constexpr (N == 1) {
      v[0] += __shfl_xor_sync(0xffffffffu, v[0], BIT);
      return TReduce<1, BIT / 2>::run(v, lane);
    } else {
      const bool upper = (lane & BIT) != 0;
#pragma unroll
      for (int q = 0; q < H; ++q) {
        const float hi = q + H < N ? v[q + H] : 0.f;
        const float send = upper ? v[q] : hi;
        const float keep = upper ? hi : v[q];
        v[q] = keep + __shfl_xor_sync(0xffffffffu, send, BIT);
      }
      return TReduce<H, BIT / 2>::run(v, lane);
    }
  }
  static __device__ __forceinline__ int index(int lane) {
    if constexpr (N == 1) {
      return 0;
    } else {
      const int sub = TReduce<H, BIT / 2>::index(lane);
      if ((lane & BIT) == 0 || sub < 0) return sub;
      return sub + H < N ? sub + H : -1;
    }
  }
};
template <int N> struct TReduce<N, 0> {
  static constexpr int kDupMask = 0;
  template <int NMAX> static __device__ __forceinline__ float run(float (&v)[NMAX], int) { return v[0]; }
  static __device__ __forceinline__ int index(int) { return 0; }
};

// model.py:108-115: idx = int((x + 6.0) * (1000.0 / 12.0)) in float64, clamped
__device__ __forceinline__ int sig_index(double x) {
  const double v = (x + 6.0) * (1000.0 / 12.0);
  if (!(v >= 0.0)) return 0;
  if (v >= 1000.0) return kSigBins - 1;
  return __double2int_rz(v);
}
__device__ __forceinline__ double sig_exact(double x) {
  if (x >= 0.0) return 1.0 / (1.0 + exp(-x));
  const double ex = exp(x);
  return ex / (1.0 + ex);
}
__device__ __forceinline__ double softplus(double x) {
  return x > 0.0 ? x + log1p(exp(-x)) : log1p(exp(x));
}

template <typename T> struct ModelView {
  T *in_dst;
  T *out_dst;
  const T *in_src;
  const T *out_src;
  int64_t ld;  // row stride in HBM, in elements (>= dim; model.py padded_ld)
  int nvec;    // 16-byte chunks of a row that hold data (dim rounded up)
  int lds;     // row stride of staged rows in shared memory: nvec chunks rounded up to 32 bytes
};
// Staged rows are packed at the data width, but keep the 32-byte sector phase of the model
// rows: a 16-byte cp.async whose shared destination and global source differ in their offset
// within a sector fetches one sector per lane (tools/probes/ldgsts_probe.cu).
template <typename T>
__host__ __device__ inline ModelView<T> make_view(T *in_dst, T *out_dst, const T *in_src, const T *out_src,
                                                  int64_t ld, int dim) {
  constexpr int per16 = 16 / (int)sizeof(T);
  const int nvec = (dim + per16 - 1) / per16;
  const int lds = ((nvec + 1) & ~1) * per16;
  return ModelView<T>{in_dst, out_dst, in_src, out_src, ld, nvec, lds};
}

// Per-cell error, as batch_core_naive computes it (kernel_batched.py:174-190):
// label - sigma and alpha * err in float64, each rounded once to the model dtype.
template <typename T>
__device__ __forceinline__ void cell_error(T s, int k, T alpha, bool exact, const T *sig_s,
                                           T &e_raw, T &e_scaled) {
  const double sd = (double)s;
  const T sig = exact ? (T)sig_exact(sd) : sig_s[sig_index(sd)];
  const double err = (k == 0 ? 1.0 : 0.0) - (double)sig;
  e_raw = (T)err;
  e_scaled = (T)((double)alpha * err);
}

// float32 fast form of cell_error (same results, no FP64 on the common path):
//  * bin index: v = (x + 6) * 1000/12 evaluated in FP32; only when v is within 1e-3 of an
//    integer (a possible bin-edge disagreement with the reference's float64 rule) is the
//    index recomputed in float64 -- ~0.2% of cells;
//  * err = label - sig: exact in FP32 for label 0, and for label 1 fl(1 - sig) is the
//    single rounding of the exact value, as (float)((double)1 - sig) is;
//  * alpha * err: for label 0 the float product is the single rounding of the exact
//    product, as the reference's double-then-float is; for label 1 fmaf(-alpha, sig,
//    alpha) rounds alpha (1 - sig) once (the double path rounds twice: they can differ
//    only when the exact value lies within 2^-53 of a float rounding boundary).
// live: lanes holding no cell (a padded score of exactly 0 sits on the bin edge v = 500)
// must not drag their warp through the float64 branch.
__device__ __forceinline__ void cell_error_f32(float s, int k, float alpha, const float *sig_s,
                                               float &e_raw, float &e_scaled, bool live = true) {
  const float v = fmaf(s, 1000.0f / 12.0f, 500.0f);
  const float fl = floorf(v);
  int idx;
  if (live && (fabsf(v - rintf(v)) < 1e-3f || !(fabsf(v) < 1e7f))) {
    idx = sig_index((double)s);
  } else {
    idx = (int)fl;
    idx = idx < 0 ? 0 : (idx >= kSigBins ? kSigBins - 1 : idx);
  }
  const float sig = sig_s[idx];
  if (k == 0) {
    e_raw = 1.0f - sig;
    e_scaled = fmaf(-alpha, sig, alpha);
  } else {
    e_raw = -sig;
    e_scaled = -(alpha * sig);
  }
}

// ------------------------------------------------------ window update ----
// Generic path (float64, K + 1 > 8, d > 512, or V * ld >= 2^32): every row of the
// window is staged in shared memory and read back from there.  ids_s: m input ids then
// k1 output ids (target first).  rows_s: (m + k1) rows of ld elements.  e_s: m * k1
// scaled errors followed by m * k1 raw errors.  k1 <= 32.
template <typename T, int NCH>
__device__ __forceinline__ void window_update(const ModelView<T> &mv, const int *ids_s, int m,
                                              int k1, T alpha, bool exact, const T *sig_s,
                                              bool want_loss, double &loss_acc,
                                              long long &cell_acc, T *rows_s, T *e_s,
                                              int lane) {
  using V = typename Vec<T>::type;
  constexpr int VN = Vec<T>::N;
  const int64_t ld = mv.ld;  // HBM stride
  const int lds = mv.lds;    // staged rows
  const int nvec = mv.nvec;
  const int nrows = m + k1;

  // gather every row of the window before any scatter (snapshot semantics)
  for (int r = 0; r < nrows; ++r) {
    const int id = ids_s[r];
    const T *src = (r < m ? mv.in_src : mv.out_src) + (int64_t)id * ld;
    T *dst = rows_s + r * lds;
#pragma unroll
    for (int j = 0; j < NCH; ++j) {
      const int c = lane + 32 * j;
      if (c < nvec) cp_async16(dst + c * VN, src + c * VN);
    }
  }
  cp_async_wait_all();
  // each lane reads back only the chunks it copied itself: no warp barrier needed
  {
    // shared-memory C (k1 <= 32): scores, errors to smem, then dA and dC passes
    constexpr int NV = 32;
    T *er_s = e_s + m * k1;
    const int my_k = reduced_index<NV>(lane);
    for (int i = 0; i < m; ++i) {
      V a[NCH];
#pragma unroll
      for (int j = 0; j < NCH; ++j) {
        const int ch = lane + 32 * j;
        a[j] = ch < nvec ? *reinterpret_cast<const V *>(rows_s + i * lds + ch * VN)
                         : vzero(T());
      }
      T p[NV];
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        T acc = T(0);
        if (k < k1) {
#pragma unroll
          for (int j = 0; j < NCH; ++j) {
            const int ch = lane + 32 * j;
            if (ch < nvec)
              acc += vdot(a[j], *reinterpret_cast<const V *>(rows_s + (m + k) * lds + ch * VN));
          }
        }
        p[k] = acc;
      }
      const T s = transpose_reduce<NV>(p, lane);
      if (my_k < k1) {
        T er, es;
        cell_error<T>(s, my_k, alpha, exact, sig_s, er, es);
        e_s[i * k1 + my_k] = es;
        er_s[i * k1 + my_k] = er;
        if (want_loss) {
          loss_acc += softplus(my_k == 0 ? -(double)s : (double)s);
          cell_acc += 1;
        }
      }
    }
    __syncwarp();
    for (int i = 0; i < m; ++i) {
      T *dst = mv.in_dst + (int64_t)ids_s[i] * ld;
#pragma unroll
      for (int j = 0; j < NCH; ++j) {
        const int ch = lane + 32 * j;
        if (ch < nvec) {
          V d = vzero(T());
          for (int k = 0; k < k1; ++k)
            vfma(d, er_s[i * k1 + k], *reinterpret_cast<const V *>(rows_s + (m + k) * lds + ch * VN));
          vscale(d, alpha);
          red_add(dst + ch * VN, d);
        }
      }
    }
    constexpr int KG = 8;
#pragma unroll
    for (int j = 0; j < NCH; ++j) {
      const int ch = lane + 32 * j;
      if (ch >= nvec) continue;
      for (int k0 = 0; k0 < k1; k0 += KG) {
        V acc[KG];
#pragma unroll
        for (int q = 0; q < KG; ++q) acc[q] = vzero(T());
        for (int i = 0; i < m; ++i) {
          const V a = *reinterpret_cast<const V *>(rows_s + i * lds + ch * VN);
#pragma unroll
          for (int q = 0; q < KG; ++q)
            if (k0 + q < k1) vfma(acc[q], e_s[i * k1 + k0 + q], a);
        }
#pragma unroll
        for (int q = 0; q < KG; ++q)
          if (k0 + q < k1) red_add(mv.out_dst + (int64_t)ids_s[m + k0 + q] * ld + ch * VN, acc[q]);
      }
    }
  }
  __syncwarp();
}


// ------------------------------------------------ float32 fast path (v2) ----
// Column mapping in 8-byte units: lane l owns float2 slots l + 32 j (j < NS),
// 150 slots at d = 300 -> 5 slots on 22 lanes, 4 on 10 (94% balanced; the
// 16-byte mapping wastes 22%).  All arithmetic is packed FFMA2 (Blackwell
// f32x2), C lives in registers loaded straight from L2, only the m input rows
// are staged in shared memory (cp.async, 16-byte), and dC is a pass over the staged
// rows whose accumulators take the C registers once dA is out (input-outer; column-outer
// for long windows), so registers stay <= 128 for K + 1 <= 6 and smem ~12 KB/warp.
__device__ __forceinline__ float2 f2zero() { return make_float2(0.f, 0.f); }
__device__ __forceinline__ float2 ld_cg_f2(const float *p) {
  float2 v;
  asm volatile("ld.global.cg.v2.f32 {%0, %1}, [%2];\n" : "=f"(v.x), "=f"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ float4 ld_cg_f4(const float *p) {
  float4 v;
  asm volatile("ld.global.cg.v4.f32 {%0, %1, %2, %3}, [%4];\n"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}

// The float32 k1 <= 8 window update in four phases:
//   f2_issue_a   input rows -> smem (16-byte cp.async)
//   f2_load_c    output rows -> registers (8-byte L2 loads)
//   f2_score_da  wait for the rows; scores, errors (to e_s), dA scattered
//   f2_dc_io     dC_k = sum_i (alpha err_ik) A_i, input-outer, NS x K1R accumulators
//   f2_dc        the same sum column-outer (windows of more than 12 inputs)
template <int NS, int NCH> struct F2Shape {
  int ld, nvec, nslot, lane;  // ld: stride of the staged rows
  __device__ F2Shape(const ModelView<float> &mv, int lane_)
      : ld(mv.lds), nvec(mv.nvec), nslot(2 * mv.nvec), lane(lane_) {}
  // slot j of this lane is always in range for j < NS - 1 (NS = ceil(nslot / 32))
  __device__ bool slot_ok(int j) const { return j < NS - 1 || lane + 32 * j < nslot; }
  __device__ bool chunk_ok(int j) const { return j < NCH - 1 || lane + 32 * j < nvec; }
};

template <int NS, int NCH>
__device__ __forceinline__ void f2_issue_a(const ModelView<float> &mv, const F2Shape<NS, NCH> &sh,
                                           const uint32_t *off_s, int m, float *rows_s) {
  const float *src_l = mv.in_src + 4 * sh.lane;
  for (int r = 0; r < m; ++r) {
    const float *src = src_l + off_s[r];
    float *dst = rows_s + r * sh.ld + 4 * sh.lane;
#pragma unroll
    for (int j = 0; j < NCH; ++j)
      if (sh.chunk_ok(j)) cp_async16(dst + 128 * j, src + 128 * j);
  }
}

template <int NS, int NCH, int K1R, bool EXACT_K>
__device__ __forceinline__ void f2_load_c(float2 (&c)[K1R][NS], const ModelView<float> &mv,
                                          const F2Shape<NS, NCH> &sh, const uint32_t *off_out,
                                          int k1) {
  const float *src_l = mv.out_src + 2 * sh.lane;
#pragma unroll
  for (int k = 0; k < K1R; ++k) {
    const bool kk = EXACT_K || k < k1;
    const float *src = src_l + off_out[kk ? k : 0];
#pragma unroll
    for (int j = 0; j < NS; ++j) c[k][j] = (kk && sh.slot_ok(j)) ? ld_cg_f2(src + 64 * j) : f2zero();
  }
}

// HOT (snapshot mode only): updates of the most frequent rows are summed per warp and
// added to the model once, at the end of the launch, instead of being scattered window by
// window.  Under Zipf ids the head rows of the reference's count-sorted vocabulary
// (corpus.py:86-105) take a large share of all slots -- row 0 about 8% of the inputs --
// and every scatter to them queues on the same few L2 lines (red.add serialises per
// address).  Two sinks:
//  * shared memory: rows [0, H_in) of M_in (in_s) and [0, H_out) of M_out (out_s), per warp,
//    in lane-owned columns, so plain loads/stores suffice; H_in / H_out are what the
//    launch's spare shared memory holds without costing resident warps;
//  * registers (in_s == nullptr): row 0 of M_in (in_lim = 1), 2 NS registers per lane, when
//    no M_in row fits in shared memory (M_out row 0 may still have a shared-memory sink).
// Each window's delta is rounded as in the scatter path; only the summation order
// changes, which the concurrent scatters leave unspecified anyway.
template <int NS> struct HotSink {
  float2 reg[NS];
  float *in_s, *out_s;       // [H_in][ld], [H_out][ld]: this warp's (nullptr: none)
  uint32_t in_lim, out_lim;  // a row offset (id * ld) below the limit is hot
};

// an error row of NV floats (the first K1R needed) as 128-bit shared loads
template <int NV, int K1R>
__device__ __forceinline__ void load_errors(float (&ev)[NV], const float *ep) {
#pragma unroll
  for (int q = 0; q < NV / 4; ++q) {
    if (4 * q < K1R || q < 2) {  // (the 8-float rows are always read whole, as before)
      const float4 e = *reinterpret_cast<const float4 *>(ep + 4 * q);
      ev[4 * q] = e.x; ev[4 * q + 1] = e.y; ev[4 * q + 2] = e.z; ev[4 * q + 3] = e.w;
    } else {
      ev[4 * q] = ev[4 * q + 1] = ev[4 * q + 2] = ev[4 * q + 3] = 0.f;
    }
  }
}

// NV: padded outputs per input in the reduction and the error rows (8; 16 for the wide body)
template <int NS, int NCH, int K1R, bool EXACT_K, bool HOT, int NV = 8>
__device__ __forceinline__ void f2_score_da(const float2 (&c)[K1R][NS], const ModelView<float> &mv,
                                            const F2Shape<NS, NCH> &sh, const uint32_t *off_s,
                                            int m, int k1, float alpha, bool exact,
                                            const float *sig_s, bool want_loss, double &loss_acc,
                                            long long &cell_acc, const float *rows_s, float *e_s,
                                            HotSink<NS> &hot, int kbase = 0) {
  static_assert(K1R <= NV && (NV == 8 || NV == 16), "K1R <= NV");
  const int lane = sh.lane;
  cp_async_wait_all();
  __syncwarp();  // staged rows were copied in 16-byte lanes, read in 8-byte lanes
  float *in_dst_l = mv.in_dst + 2 * lane;
  // inputs in pairs: one transposed butterfly over 16 values reduces both inputs' scores
  for (int i = 0; i < m; i += 2) {
    const bool two = i + 1 < m;
    float pp[2 * NV];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int ii = two ? i + h : i;
      float2 a[NS];
#pragma unroll
      for (int j = 0; j < NS; ++j)
        a[j] = sh.slot_ok(j) ? *reinterpret_cast<const float2 *>(rows_s + ii * sh.ld + 2 * (lane + 32 * j))
                             : f2zero();
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        if (k < K1R) {
          float2 acc = __fmul2_rn(a[0], c[k][0]);
#pragma unroll
          for (int j = 1; j < NS; ++j) acc = __ffma2_rn(a[j], c[k][j], acc);
          pp[h * NV + k] = acc.x + acc.y;
        } else {
          pp[h * NV + k] = 0.f;
        }
      }
    }
    const float s = transpose_reduce<2 * NV>(pp, lane);
    const int v = reduced_index<2 * NV>(lane);
    const int hk = v >> Log2<NV>::v, kk = v & (NV - 1);
    float er = 0.f, es = 0.f;
    if (kk < k1 && (hk == 0 || two)) {
      if (exact) cell_error<float>(s, kbase + kk, alpha, true, sig_s, er, es);
      else cell_error_f32(s, kbase + kk, alpha, sig_s, er, es);
      if ((lane & (16 / NV - 1)) == 0) {  // one lane per value (2 * NV values over 32 lanes)
        e_s[(i + hk) * NV + kk] = es;
        if (want_loss) {
          loss_acc += softplus(kbase + kk == 0 ? -(double)s : (double)s);
          cell_acc += 1;
        }
      }
    }
    // dA_i = sum_k (alpha err_ik) C_k, alpha folded into e as batch_core_blas does
    // (kernel_batched.py:92-144): the pair's error rows are broadcast from e_s
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (h == 1 && !two) break;
      float ev[NV];
      load_errors<NV, K1R>(ev, e_s + (i + h) * NV);
      float2 d[NS];
#pragma unroll
      for (int k = 0; k < K1R; ++k) {
        const float ek = (EXACT_K || k < k1) ? ev[k] : 0.f;
        const float2 ek2 = make_float2(ek, ek);
#pragma unroll
        for (int j = 0; j < NS; ++j) d[j] = k == 0 ? __fmul2_rn(ek2, c[0][j]) : __ffma2_rn(ek2, c[k][j], d[j]);
      }
      const uint32_t ro = off_s[i + h];
      if (HOT && ro < hot.in_lim) {
        if (hot.in_s) {
          float *hs = hot.in_s + ro + 2 * lane;
#pragma unroll
          for (int j = 0; j < NS; ++j)
            if (sh.slot_ok(j)) {
              float2 *q = reinterpret_cast<float2 *>(hs + 64 * j);
              *q = __fadd2_rn(*q, d[j]);
            }
        } else {
#pragma unroll
          for (int j = 0; j < NS; ++j) hot.reg[j] = __fadd2_rn(hot.reg[j], d[j]);
        }
      } else {
        float *dst = in_dst_l + ro;
#pragma unroll
        for (int j = 0; j < NS; ++j)
          if (sh.slot_ok(j)) atomicAdd(reinterpret_cast<float2 *>(dst + 64 * j), d[j]);
      }
    }
  }
  __syncwarp();
}

template <int NS, int NCH, int K1R, bool EXACT_K, bool HOT = false, int NV = 8>
__device__ __forceinline__ void f2_dc(const ModelView<float> &mv, const F2Shape<NS, NCH> &sh,
                                      const uint32_t *off_s, int m, int k1, const float *rows_s,
                                      const float *e_s, HotSink<NS> *hot = nullptr) {
  auto kk_ok = [&](int k) { return EXACT_K || k < k1; };
  float *out_dst_l = mv.out_dst + 2 * sh.lane;
#pragma unroll
  for (int j = 0; j < NS; ++j) {
    if (!sh.slot_ok(j)) continue;
    const int col = 2 * (sh.lane + 32 * j);
    float2 acc[K1R];
#pragma unroll
    for (int k = 0; k < K1R; ++k) acc[k] = f2zero();
    const float *ap = rows_s + col;
    const float *ep = e_s;
    for (int i = 0; i < m; ++i, ap += sh.ld, ep += NV) {
      const float2 a0 = *reinterpret_cast<const float2 *>(ap);
      float ev[NV];
      load_errors<NV, K1R>(ev, ep);
#pragma unroll
      for (int k = 0; k < K1R; ++k)
        if (kk_ok(k)) acc[k] = __ffma2_rn(make_float2(ev[k], ev[k]), a0, acc[k]);
    }
#pragma unroll
    for (int k = 0; k < K1R; ++k) {
      if (!kk_ok(k)) continue;
      const uint32_t ro = off_s[m + k];
      if (HOT && ro < hot->out_lim) {
        float2 *q = reinterpret_cast<float2 *>(hot->out_s + ro + col);
        *q = __fadd2_rn(*q, acc[k]);
      } else {
        atomicAdd(reinterpret_cast<float2 *>(out_dst_l + ro + 64 * j), acc[k]);
      }
    }
  }
  __syncwarp();
}

// dC input-outer: NS x K1R float2 accumulators in registers (the caller's C registers
// are dead by now), each staged row slot and error row read once
template <int NS, int NCH, int K1R, bool EXACT_K, bool HOT = false, int NV = 8>
__device__ __forceinline__ void f2_dc_io(const ModelView<float> &mv, const F2Shape<NS, NCH> &sh,
                                         const uint32_t *off_s, int m, int k1, const float *rows_s,
                                         const float *e_s, HotSink<NS> *hot = nullptr) {
  auto kk_ok = [&](int k) { return EXACT_K || k < k1; };
  float *out_dst_l = mv.out_dst + 2 * sh.lane;
  float2 acc[NS][K1R];
#pragma unroll
  for (int j = 0; j < NS; ++j)
#pragma unroll
    for (int k = 0; k < K1R; ++k) acc[j][k] = f2zero();
  const float *ap = rows_s + 2 * sh.lane;
  const float *ep = e_s;
  for (int i = 0; i < m; ++i, ap += sh.ld, ep += NV) {
    float ev[NV];
    load_errors<NV, K1R>(ev, ep);
#pragma unroll
    for (int j = 0; j < NS; ++j) {
      const float2 a0 = sh.slot_ok(j) ? *reinterpret_cast<const float2 *>(ap + 64 * j) : f2zero();
#pragma unroll
      for (int k = 0; k < K1R; ++k)
        if (kk_ok(k)) acc[j][k] = __ffma2_rn(make_float2(ev[k], ev[k]), a0, acc[j][k]);
    }
  }
#pragma unroll
  for (int k = 0; k < K1R; ++k) {
    if (!kk_ok(k)) continue;
    const uint32_t ro = off_s[m + k];
#pragma unroll
    for (int j = 0; j < NS; ++j) {
      if (!sh.slot_ok(j)) continue;
      if (HOT && ro < hot->out_lim) {
        float2 *q = reinterpret_cast<float2 *>(hot->out_s + ro + 2 * (sh.lane + 32 * j));
        *q = __fadd2_rn(*q, acc[j][k]);
      } else {
        atomicAdd(reinterpret_cast<float2 *>(out_dst_l + ro + 64 * j), acc[j][k]);
      }
    }
  }
  __syncwarp();
}


template <int NS, int NCH, int K1R, bool EXACT_K, bool HOT = false>
__device__ __forceinline__ void window_update_f2(const ModelView<float> &mv, const uint32_t *off_s,
                                                 int m, int k1, float alpha, bool exact,
                                                 const float *sig_s, bool want_loss,
                                                 double &loss_acc, long long &cell_acc,
                                                 float *rows_s, float *e_s, int lane,
                                                 HotSink<NS> &hot) {
  if constexpr (EXACT_K) k1 = K1R;
  const F2Shape<NS, NCH> sh(mv, lane);
  f2_issue_a<NS, NCH>(mv, sh, off_s, m, rows_s);
  float2 c[K1R][NS];
  f2_load_c<NS, NCH, K1R, EXACT_K>(c, mv, sh, off_s + m, k1);
  f2_score_da<NS, NCH, K1R, EXACT_K, HOT>(c, mv, sh, off_s, m, k1, alpha, exact, sig_s, want_loss,
                                          loss_acc, cell_acc, rows_s, e_s, hot);
  // input-outer dC (C registers dead) up to 12 inputs; long windows (w = 10) measured
  // faster column-outer (configs[1]: 0.61 vs 0.56)
  if (m <= 12) f2_dc_io<NS, NCH, K1R, EXACT_K, HOT>(mv, sh, off_s, m, k1, rows_s, e_s, &hot);
  else f2_dc<NS, NCH, K1R, EXACT_K, HOT>(mv, sh, off_s, m, k1, rows_s, e_s, &hot);
}


// float32, 8 < k1 <= 16, d <= 128 (NS <= 2): all k1 output rows in ONE register group
// (16 x 2 float2 = 64 registers), so each input's scores take one pass over its staged row,
// one 32-value butterfly per input pair and one dA scatter, where the two-group body takes
// two of each; error rows are padded to 16 floats.
template <int NS, int NCH, int K1R, bool HOT = false>
__device__ __forceinline__ void window_update_f2w(const ModelView<float> &mv, const uint32_t *off_s,
                                                  int m, int k1, float alpha, bool exact,
                                                  const float *sig_s, bool want_loss,
                                                  double &loss_acc, long long &cell_acc,
                                                  float *rows_s, float *e_s, int lane,
                                                  HotSink<NS> &hot) {
  static_assert(NS <= 2 && K1R <= 16, "wide body: d <= 128");
  const F2Shape<NS, NCH> sh(mv, lane);
  f2_issue_a<NS, NCH>(mv, sh, off_s, m, rows_s);
  float2 c[K1R][NS];
  f2_load_c<NS, NCH, K1R, false>(c, mv, sh, off_s + m, k1);
  f2_score_da<NS, NCH, K1R, false, HOT, 16>(c, mv, sh, off_s, m, k1, alpha, exact, sig_s, want_loss,
                                            loss_acc, cell_acc, rows_s, e_s, hot);
  if (m <= 12) f2_dc_io<NS, NCH, K1R, false, HOT, 16>(mv, sh, off_s, m, k1, rows_s, e_s, &hot);
  else f2_dc<NS, NCH, K1R, false, HOT, 16>(mv, sh, off_s, m, k1, rows_s, e_s, &hot);
}

// float32, 8 < k1 <= 16, d <= 512: window_update_f2 over two groups of output rows
// (k < 8, then 8 <= k < k1; kbase shifts the label so only k = 0 is positive).  The
// group's C rows live in registers, so only the m input rows are staged in shared memory
// (~13 KB per warp at d = 300: 16 warps per SM, where staging all m + k1 rows allows 7);
// the price is that dA is scattered once per group.  Group 1's rows are loaded before
// group 0's dC is scattered, so in place (Hogwild) every row is gathered before this
// window updates it, as batch_core gathers all rows first (kernel_batched.py:104-113).
template <int NS, int NCH, int K1R2 = 8, bool HOT = false>
__device__ __forceinline__ void window_update_f2g(const ModelView<float> &mv, const uint32_t *off_s,
                                                  int m, int k1, float alpha, bool exact,
                                                  const float *sig_s, bool want_loss,
                                                  double &loss_acc, long long &cell_acc,
                                                  float *rows_s, float *e_s, int lane,
                                                  HotSink<NS> &hot) {
  // K1R2: register rows of the second group (4 when k1 <= 12, else 8)
  const F2Shape<NS, NCH> sh(mv, lane);
  f2_issue_a<NS, NCH>(mv, sh, off_s, m, rows_s);
  float2 c[8][NS];
  f2_load_c<NS, NCH, 8, false>(c, mv, sh, off_s + m, 8);
  f2_score_da<NS, NCH, 8, false, HOT>(c, mv, sh, off_s, m, 8, alpha, exact, sig_s, want_loss,
                                      loss_acc, cell_acc, rows_s, e_s, hot, 0);
  float2 c2[K1R2][NS];
  if (mv.out_src != mv.out_dst && m <= 12) {
    // snapshot mode: group 0's dC input-outer first (its C registers are dead), then group
    // 1's rows -- they come from the unchanged snapshot, so the order does not matter
    f2_dc_io<NS, NCH, 8, false, HOT>(mv, sh, off_s, m, 8, rows_s, e_s, &hot);
    f2_load_c<NS, NCH, K1R2, false>(c2, mv, sh, off_s + m + 8, k1 - 8);
    f2_score_da<NS, NCH, K1R2, false, HOT>(c2, mv, sh, off_s, m, k1 - 8, alpha, exact, sig_s, want_loss,
                                           loss_acc, cell_acc, rows_s, e_s, hot, 8);
    f2_dc_io<NS, NCH, K1R2, false, HOT>(mv, sh, off_s + 8, m, k1 - 8, rows_s, e_s, &hot);
    return;
  }
  // in place: group 1's rows are gathered before group 0's dC is scattered
  f2_load_c<NS, NCH, K1R2, false>(c2, mv, sh, off_s + m + 8, k1 - 8);
  f2_dc<NS, NCH, 8, false, HOT>(mv, sh, off_s, m, 8, rows_s, e_s, &hot);
  f2_score_da<NS, NCH, K1R2, false, HOT>(c2, mv, sh, off_s, m, k1 - 8, alpha, exact, sig_s, want_loss,
                                         loss_acc, cell_acc, rows_s, e_s, hot, 8);
  f2_dc<NS, NCH, K1R2, false, HOT>(mv, sh, off_s + 8, m, k1 - 8, rows_s, e_s, &hot);
}

// float32, 8 < k1 <= 16, d <= 512: like window_update_f2 but the k1 output rows stay in
// shared memory (16 x NS float2 would not fit in registers).  Each C-row slot load is
// shared by a pair of inputs; one transposed butterfly over 32 values reduces both
// inputs' scores; error rows are padded to 16 floats.  rows_s holds the m input rows
// then the k1 output rows.
template <int NS, int NCH, bool HOT = false>
__device__ __forceinline__ void window_update_f2s(const ModelView<float> &mv, const uint32_t *off_s,
                                                  int m, int k1, float alpha, bool exact,
                                                  const float *sig_s, bool want_loss,
                                                  double &loss_acc, long long &cell_acc,
                                                  float *rows_s, float *e_s, int lane,
                                                  HotSink<NS> &hot) {  // register sink only
  constexpr int KM = 16;
  const int ld = mv.lds;  // staged rows
  const int nvec = mv.nvec, nslot = nvec * 2;
  auto slot_ok = [&](int j) { return j < NS - 1 || lane + 32 * j < nslot; };
  auto chunk_ok = [&](int j) { return j < NCH - 1 || lane + 32 * j < nvec; };
  for (int r = 0; r < m + k1; ++r) {
    const float *src = (r < m ? mv.in_src : mv.out_src) + off_s[r];
    float *dst = rows_s + r * ld;
#pragma unroll
    for (int j = 0; j < NCH; ++j)
      if (chunk_ok(j)) cp_async16(dst + (lane + 32 * j) * 4, src + (lane + 32 * j) * 4);
  }
  cp_async_wait_all();
  __syncwarp();
  const float *c_s = rows_s + m * ld;
  float *er_s = e_s + m * KM;  // raw errors after the scaled ones
  const float2 alpha2 = make_float2(alpha, alpha);
  for (int i = 0; i < m; i += 2) {
    const bool two = i + 1 < m;
    const int i1 = two ? i + 1 : i;
    float2 a0[NS], a1[NS];
#pragma unroll
    for (int j = 0; j < NS; ++j) {
      const int col = 2 * (lane + 32 * j);
      a0[j] = slot_ok(j) ? *reinterpret_cast<const float2 *>(rows_s + i * ld + col) : f2zero();
      a1[j] = slot_ok(j) ? *reinterpret_cast<const float2 *>(rows_s + i1 * ld + col) : f2zero();
    }
    float pp[2 * KM];
#pragma unroll
    for (int k = 0; k < KM; ++k) {
      float2 s0 = f2zero(), s1 = f2zero();
      if (k < k1) {
#pragma unroll
        for (int j = 0; j < NS; ++j) {
          const float2 c = slot_ok(j) ? *reinterpret_cast<const float2 *>(c_s + k * ld + 2 * (lane + 32 * j))
                                      : f2zero();
          s0 = __ffma2_rn(a0[j], c, s0);
          s1 = __ffma2_rn(a1[j], c, s1);
        }
      }
      pp[k] = s0.x + s0.y;
      pp[KM + k] = s1.x + s1.y;
    }
    const float sc = transpose_reduce<2 * KM>(pp, lane);  // value v = h * 16 + k on lane v
    const int hk = lane >> 4, kk = lane & 15;
    const bool live = kk < k1 && (hk == 0 || two);
    float er = 0.f, es = 0.f;
    if (live) {
      if (exact) cell_error<float>(sc, kk, alpha, true, sig_s, er, es);
      else cell_error_f32(sc, kk, alpha, sig_s, er, es);
      e_s[(i + hk) * KM + kk] = es;
      er_s[(i + hk) * KM + kk] = er;
      if (want_loss) {
        loss_acc += softplus(kk == 0 ? -(double)sc : (double)sc);
        cell_acc += 1;
      }
    }
    __syncwarp();
    // dA for both inputs, each C slot loaded once
    float2 d0[NS], d1[NS];
#pragma unroll
    for (int j = 0; j < NS; ++j) d0[j] = d1[j] = f2zero();
    for (int k = 0; k < k1; ++k) {
      const float e0 = er_s[i * KM + k], e1 = er_s[i1 * KM + k];
#pragma unroll
      for (int j = 0; j < NS; ++j) {
        const float2 c = slot_ok(j) ? *reinterpret_cast<const float2 *>(c_s + k * ld + 2 * (lane + 32 * j))
                                    : f2zero();
        d0[j] = __ffma2_rn(make_float2(e0, e0), c, d0[j]);
        d1[j] = __ffma2_rn(make_float2(e1, e1), c, d1[j]);
      }
    }
    // HOT: row 0's dA goes to the warp's register accumulator (see f2_score_da)
    const bool hot0 = HOT && off_s[i] == 0, hot1 = HOT && two && off_s[i1] == 0;
    float *dst0 = mv.in_dst + off_s[i] + 2 * lane;
    float *dst1 = mv.in_dst + off_s[i1] + 2 * lane;
#pragma unroll
    for (int j = 0; j < NS; ++j) {
      const float2 u0 = __fmul2_rn(d0[j], alpha2), u1 = __fmul2_rn(d1[j], alpha2);
      if (hot0) hot.reg[j] = __fadd2_rn(hot.reg[j], u0);
      if (hot1) hot.reg[j] = __fadd2_rn(hot.reg[j], u1);
      if (slot_ok(j)) {
        if (!hot0) atomicAdd(reinterpret_cast<float2 *>(dst0 + 64 * j), u0);
        if (two && !hot1) atomicAdd(reinterpret_cast<float2 *>(dst1 + 64 * j), u1);
      }
    }
  }
  __syncwarp();
  // dC_k = sum_i (alpha err_ik) A_i, column-outer, outputs in groups of 8
#pragma unroll
  for (int j = 0; j < NS; ++j) {
    if (!slot_ok(j)) continue;
    const int col = 2 * (lane + 32 * j);
    for (int k0 = 0; k0 < k1; k0 += 8) {
      float2 acc[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q] = f2zero();
      for (int i = 0; i < m; ++i) {
        const float2 a = *reinterpret_cast<const float2 *>(rows_s + i * ld + col);
        const float4 e03 = *reinterpret_cast<const float4 *>(e_s + i * KM + k0);
        const float4 e47 = *reinterpret_cast<const float4 *>(e_s + i * KM + k0 + 4);
        const float ev[8] = {e03.x, e03.y, e03.z, e03.w, e47.x, e47.y, e47.z, e47.w};
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q] = __ffma2_rn(make_float2(ev[q], ev[q]), a, acc[q]);
      }
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (k0 + q < k1) atomicAdd(reinterpret_cast<float2 *>(mv.out_dst + off_s[m + k0 + q] + col), acc[q]);
    }
  }
  __syncwarp();
}

}  // namespace sgns
