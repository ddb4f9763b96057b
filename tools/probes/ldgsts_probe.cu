// Probe: how many L2->L1 sectors does one warp-wide 16-byte cp.async (LDGSTS.E.BYPASS.128) fetch?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ldgsts_probe ldgsts_probe.cu
//   ncu --metrics sm__sass_l1tex_m_xbar2l1tex_read_sectors_mem_global_op_ldgsts_cache_bypass.sum,\
//       sm__sass_inst_executed_op_ldgsts_cache_bypass.sum ./ldgsts_probe
#include <cstdio>
#include <cuda_runtime.h>

template <int GOFF, int SOFF, int LANES>
__global__ void probe(const float *g, float *out, int iters) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned char *dst = sm + warp * 1024 + SOFF + 16 * lane;
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  const unsigned char *src = reinterpret_cast<const unsigned char *>(g) + GOFF + 16 * lane +
                             (size_t)(blockIdx.x * 8 + warp) * 4096;
  for (int i = 0; i < iters; ++i) {
    if (lane < LANES)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(src + (size_t)i * 1048576) : "memory");
  }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncwarp();
  if (out) out[threadIdx.x] = *reinterpret_cast<float *>(dst);
}

int main() {
  float *g, *o;
  cudaMalloc(&g, 512u << 20);
  cudaMemset(g, 0, 512u << 20);
  cudaMalloc(&o, 4096);
  const int it = 256;
  probe<0, 0, 32><<<64, 256, 8 * 1024 + 256>>>(g, o, it);    // aligned, aligned
  probe<0, 16, 32><<<64, 256, 8 * 1024 + 256>>>(g, o, it);   // smem dst off by 16
  probe<16, 0, 32><<<64, 256, 8 * 1024 + 256>>>(g, o, it);   // global off by 16
  probe<16, 16, 32><<<64, 256, 8 * 1024 + 256>>>(g, o, it);  // both off by 16
  probe<0, 0, 11><<<64, 256, 8 * 1024 + 256>>>(g, o, it);    // 11 lanes
  probe<0, 16, 11><<<64, 256, 8 * 1024 + 256>>>(g, o, it);   // 11 lanes, smem off by 16
  probe<0, 48, 32><<<64, 256, 8 * 1024 + 256>>>(g, o, it);   // smem off by 48
  probe<0, 64, 32><<<64, 256, 8 * 1024 + 256>>>(g, o, it);   // smem off by 64
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
