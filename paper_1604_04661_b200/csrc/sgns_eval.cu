// sgns_eval.cu -- analogy evaluation on the device: the 3CosAdd argmax of
// sgns/evaluate.py:164-212 as two kernels behind the C ABI.
//
//   unit_rows_kernel      unit = v / ||v|| in float32 exactly as numpy computes it for the
//                         reference (np.linalg.norm(axis=1): float32 squares summed with
//                         numpy's pairwise summation, sqrtf, a zero norm replaced by 1, one
//                         float32 division) -- bit-identical unit rows;
//   analogy_top1_kernel   per question q with target t_q = (u_b - u_a) + u_c: the vocabulary
//                         row w < limit, w not in {a, b, c}, maximising t_q . u_w, first
//                         index on ties (np.argmax).  A tiled FP32 SIMT contraction
//                         (64 questions x 128 rows per block, k-chunks of 32 staged in shared
//                         memory, 4 x 8 register micro-tile per thread) whose epilogue keeps
//                         each question's best (score, row) in registers across the block's
//                         row tiles and publishes it with one 64-bit atomicMax; the score
//                         matrix is never written.  The dot products accumulate in a
//                         different order than OpenBLAS's sgemm, so only exact ties within
//                         float32 rounding can resolve differently.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "../../include/sgns_b200.h"

namespace {

constexpr int kPwBlock = 128;  // numpy's PW_BLOCKSIZE

// numpy's pairwise_sum for float32 (umath loops_utils): 8 accumulators below 128 items,
// halving at a multiple of 8 above
__device__ float pairwise_sq_sum(const float *x, int n) {
  if (n < 8) {
    float r = 0.f;
    for (int i = 0; i < n; ++i) r = __fadd_rn(r, __fmul_rn(x[i], x[i]));
    return r;
  }
  if (n <= kPwBlock) {
    float r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __fmul_rn(x[j], x[j]);
    int i = 8;
    for (; i < n - (n % 8); i += 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = __fadd_rn(r[j], __fmul_rn(x[i + j], x[i + j]));
    }
    float res = __fadd_rn(__fadd_rn(__fadd_rn(r[0], r[1]), __fadd_rn(r[2], r[3])),
                          __fadd_rn(__fadd_rn(r[4], r[5]), __fadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __fadd_rn(res, __fmul_rn(x[i], x[i]));
    return res;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  return __fadd_rn(pairwise_sq_sum(x, n2), pairwise_sq_sum(x + n2, n - n2));
}

__global__ void unit_rows_kernel(const float *rows, int64_t ld, int64_t n, int dim, float *out, int64_t ld_out) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const float *x = rows + r * ld;
  float nrm = __fsqrt_rn(pairwise_sq_sum(x, dim));
  if (nrm == 0.f) nrm = 1.f;
  float *o = out + r * ld_out;
  for (int j = 0; j < dim; ++j) o[j] = __fdiv_rn(x[j], nrm);
}

__global__ void analogy_targets_kernel(const float *unit, int64_t ld, int dim, const int32_t *q3, int64_t nq,
                                       float *targets) {
  const int64_t q = blockIdx.x;
  if (q >= nq) return;
  const float *ua = unit + (int64_t)q3[3 * q] * ld, *ub = unit + (int64_t)q3[3 * q + 1] * ld,
              *uc = unit + (int64_t)q3[3 * q + 2] * ld;
  for (int j = threadIdx.x; j < dim; j += blockDim.x)
    targets[q * dim + j] = __fadd_rn(__fsub_rn(ub[j], ua[j]), uc[j]);
}

// total order on float scores as unsigned keys (larger float -> larger key)
__device__ __forceinline__ uint32_t orderable(float f) {
  const uint32_t b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

constexpr int BQ = 64, BV = 128, BK = 32, TQ = 4, TV = 8;  // 256 threads: 16 (q) x 16 (v)

__global__ void __launch_bounds__(256) analogy_top1_kernel(const float *unit, int64_t ld, int64_t n, int dim,
                                                           const float *targets, const int32_t *q3, int64_t nq,
                                                           unsigned long long *best_key) {
  __shared__ float ts[BK][BQ];
  __shared__ float us[BK][BV + 4];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t q0 = (int64_t)blockIdx.x * BQ;
  int excl[TQ][3];
  unsigned long long best[TQ];
#pragma unroll
  for (int a = 0; a < TQ; ++a) {
    const int64_t q = q0 + ty * TQ + a;
#pragma unroll
    for (int c = 0; c < 3; ++c) excl[a][c] = q < nq ? q3[3 * q + c] : -1;
    best[a] = 0ull;
  }
  for (int64_t v0 = (int64_t)blockIdx.y * BV; v0 < n; v0 += (int64_t)gridDim.y * BV) {
    float acc[TQ][TV];
#pragma unroll
    for (int a = 0; a < TQ; ++a)
#pragma unroll
      for (int b = 0; b < TV; ++b) acc[a][b] = 0.f;
    for (int k0 = 0; k0 < dim; k0 += BK) {
      // stage targets [BQ x BK] and rows [BV x BK], transposed to k-major
      for (int i = threadIdx.x; i < BQ * BK; i += 256) {
        const int qq = i / BK, kk = i % BK;
        const int64_t q = q0 + qq;
        ts[kk][qq] = (q < nq && k0 + kk < dim) ? targets[q * dim + k0 + kk] : 0.f;
      }
      for (int i = threadIdx.x; i < BV * BK; i += 256) {
        const int vv = i / BK, kk = i % BK;
        const int64_t v = v0 + vv;
        us[kk][vv] = (v < n && k0 + kk < dim) ? unit[v * ld + k0 + kk] : 0.f;
      }
      __syncthreads();
#pragma unroll 8
      for (int kk = 0; kk < BK; ++kk) {
        float tq[TQ], uv[TV];
#pragma unroll
        for (int a = 0; a < TQ; ++a) tq[a] = ts[kk][ty * TQ + a];
#pragma unroll
        for (int b = 0; b < TV; ++b) uv[b] = us[kk][tx * TV + b];
#pragma unroll
        for (int a = 0; a < TQ; ++a)
#pragma unroll
          for (int b = 0; b < TV; ++b) acc[a][b] = fmaf(tq[a], uv[b], acc[a][b]);
      }
      __syncthreads();
    }
#pragma unroll
    for (int a = 0; a < TQ; ++a)
#pragma unroll
      for (int b = 0; b < TV; ++b) {
        const int64_t w = v0 + tx * TV + b;
        if (w >= n || w == excl[a][0] || w == excl[a][1] || w == excl[a][2]) continue;
        const unsigned long long key =
            ((unsigned long long)orderable(acc[a][b]) << 32) | (0xFFFFFFFFu - (uint32_t)w);
        best[a] = key > best[a] ? key : best[a];
      }
  }
  // the 16 threads of a question row sit in one half-warp
#pragma unroll
  for (int a = 0; a < TQ; ++a) {
    unsigned long long k = best[a];
#pragma unroll
    for (int o = 8; o >= 1; o >>= 1) {
      const unsigned long long other = __shfl_xor_sync(0xffffffffu, k, o);
      k = other > k ? other : k;
    }
    const int64_t q = q0 + ty * TQ + a;
    if (tx == 0 && q < nq && k != 0ull) atomicMax(best_key + q, k);
  }
}

__global__ void keys_to_rows_kernel(const unsigned long long *keys, int64_t nq, int32_t *best) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q < nq) best[q] = keys[q] ? (int32_t)(0xFFFFFFFFu - (uint32_t)(keys[q] & 0xFFFFFFFFull)) : -1;
}

}  // namespace

extern "C" int sgns_unit_rows(const float *rows, int64_t ld, int64_t n, int32_t dim, float *out, int64_t ld_out,
                              void *stream) {
  if (!rows || !out || n < 0 || dim < 1 || ld < dim || ld_out < dim) return SGNS_E_ARG;
  if (n == 0) return SGNS_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  unit_rows_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(rows, ld, n, dim, out, ld_out);
  return (int)cudaGetLastError();
}

// workspace: nq * dim * 4 + 4 + nq * 8 bytes, 8-byte aligned (targets, then 64-bit keys)
extern "C" int sgns_analogy_top1(const float *unit, int64_t ld, int64_t n, int32_t dim, const int32_t *q3,
                                 int64_t nq, int32_t *best, void *workspace, void *stream) {
  if (!unit || !q3 || !best || !workspace || n < 1 || n > 0x7fffffffLL || dim < 1 || ld < dim || nq < 0)
    return SGNS_E_ARG;
  if (nq == 0) return SGNS_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  float *targets = static_cast<float *>(workspace);
  unsigned long long *keys = reinterpret_cast<unsigned long long *>(targets + nq * dim + ((nq * dim) & 1));
  cudaError_t e = cudaMemsetAsync(keys, 0, (size_t)nq * 8, st);
  if (e != cudaSuccess) return (int)e;
  analogy_targets_kernel<<<(unsigned)nq, 128, 0, st>>>(unit, ld, dim, q3, nq, targets);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t qb = (nq + BQ - 1) / BQ, vb = (n + BV - 1) / BV;
  // enough blocks to fill the GPU a few times over; each walks its row tiles with a stride
  const int64_t gy = std::min<int64_t>(vb, std::max<int64_t>(1, (int64_t)sms * 8 / qb + 1));
  analogy_top1_kernel<<<dim3((unsigned)qb, (unsigned)gy), 256, 0, st>>>(unit, ld, n, dim, targets, q3, nq, keys);
  keys_to_rows_kernel<<<(unsigned)((nq + 255) / 256), 256, 0, st>>>(keys, nq, best);
  return (int)cudaGetLastError();
}
