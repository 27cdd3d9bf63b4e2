// Microbenchmark (measurement tool): tcgen05.mma kind::f16 M=128 issue rate from one thread per CTA,
// operands in shared memory, SWIZZLE_NONE (interleaved) vs SWIZZLE_128B K-major layouts, various N.
#include <cstdio>
#include <cstdint>
#include "../../paper_2407_09543_b200/csrc/sm100.cuh"
using namespace ntbc;

__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)(1) << 16;                      // LBO (ignored for swizzled K-major)
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;                        // SWIZZLE_128B
  return d;
}

template <int N, bool SW>
__global__ void __launch_bounds__(128, 1) k(int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* A = smem;                 // 128 x 64 fp16 = 16 KB
  uint8_t* B = smem + 16384;         // N x 64 fp16
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 16384 + 256 * 128);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  for (int i = threadIdx.x; i < (16384 + 256 * 128) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3C003C00u;
  fence_async_smem();
  if (threadIdx.x == 0) { mbar_init(bar, 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc(slot, 256);
  __syncthreads();
  tc_fence_after();
  const uint32_t t = *slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_f16_f32(128, N);
    const uint32_t a = smem_u32(A), b = smem_u32(B);
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
      const int c = i & 3;  // walk the 4 K-chunks of a K=64 operand
      uint64_t da, db;
      if (SW) { da = desc_sw128(a, 1024) + c * 2; db = desc_sw128(b, 1024) + c * 2; }   // +32 B per K chunk
      else { da = smem_desc(a + c * 256, 128, 1024); db = smem_desc(b + c * 256, 128, 1024); }
      mma_f16(t, da, db, idesc, i > 0);
    }
    long long t1 = clock64();
    mma_commit(bar);
    mbar_wait(bar, 0);
    long long t2 = clock64();
    if (blockIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
  }
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(t, 256);
}

template <int N, bool SW>
void run(int ctas, long long* d) {
  const int iters = 4096;
  const int smem = 16384 + 256 * 128 + 64;
  cudaFuncSetAttribute(k<N, SW>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<N, SW><<<ctas, 128, smem>>>(iters, d);
  long long h[2];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  const double flops = 2.0 * 128 * N * 16;
  printf("N=%3d %-6s ctas=%3d: issue %6.1f cyc/mma, complete %6.1f cyc/mma  (%.0f MAC/clk/SM)\n", N,
         SW ? "SW128" : "INTER", ctas, (double)h[0] / iters, (double)h[1] / iters, flops / 2 / ((double)h[1] / iters));
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  for (int ctas : {1, 148}) {
    run<16, false>(ctas, d); run<64, false>(ctas, d); run<128, false>(ctas, d); run<256, false>(ctas, d);
    run<16, true>(ctas, d); run<64, true>(ctas, d); run<128, true>(ctas, d); run<256, true>(ctas, d);
  }
  printf("cuda: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
