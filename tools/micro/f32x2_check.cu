// Microcheck: do sm_100a packed fp32x2 ops (FFMA2/FADD2/FMUL2) equal the scalar IEEE ops lane by lane,
// including when one operand is a runtime value broadcast to both lanes?  (measurement tool)
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <random>
#include "../../paper_2407_09543_b200/csrc/bc_device.cuh"
using namespace ntbc;

__global__ void k(const float* a, const float* b, const float* c, int n, unsigned* bad) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n / 2) return;
  float a0 = a[2 * i], a1 = a[2 * i + 1], b0 = b[2 * i], b1 = b[2 * i + 1], c0 = c[2 * i], c1 = c[2 * i + 1];
  float r0, r1;
  // 0: general fma2
  f2unpack(fma2(f2pack(a0, a1), f2pack(b0, b1), f2pack(c0, c1)), r0, r1);
  if (r0 != __fmaf_rn(a0, b0, c0) || r1 != __fmaf_rn(a1, b1, c1)) atomicAdd(&bad[0], 1);
  // 1: fma2 with broadcast a
  f2unpack(fma2(f2pack(a0, a0), f2pack(b0, b1), f2pack(c0, c1)), r0, r1);
  if (r0 != __fmaf_rn(a0, b0, c0) || r1 != __fmaf_rn(a0, b1, c1)) atomicAdd(&bad[1], 1);
  // 2: add2 general
  f2unpack(add2(f2pack(a0, a1), f2pack(b0, b1)), r0, r1);
  if (r0 != __fadd_rn(a0, b0) || r1 != __fadd_rn(a1, b1)) atomicAdd(&bad[2], 1);
  // 3: sub2 general
  f2unpack(sub2(f2pack(a0, a1), f2pack(b0, b1)), r0, r1);
  if (r0 != __fsub_rn(a0, b0) || r1 != __fsub_rn(a1, b1)) atomicAdd(&bad[3], 1);
  // 4: mul2 general
  f2unpack(mul2(f2pack(a0, a1), f2pack(b0, b1)), r0, r1);
  if (r0 != __fmul_rn(a0, b0) || r1 != __fmul_rn(a1, b1)) atomicAdd(&bad[4], 1);
  // 5: mul2 broadcast b
  f2unpack(mul2(f2pack(a0, a1), f2pack(b0, b0)), r0, r1);
  if (r0 != __fmul_rn(a0, b0) || r1 != __fmul_rn(a1, b0)) atomicAdd(&bad[5], 1);
  // 6: the lerp pattern of level_lookup2: fma2(FX, sub2(v10, v00), v00) with FX broadcast
  f2unpack(fma2(f2pack(c0, c0), sub2(f2pack(a0, a1), f2pack(b0, b1)), f2pack(b0, b1)), r0, r1);
  if (r0 != __fmaf_rn(c0, __fsub_rn(a0, b0), b0) || r1 != __fmaf_rn(c0, __fsub_rn(a1, b1), b1)) {
    unsigned j = atomicAdd(&bad[6], 1);
    if (j < 4) printf("lerp mismatch: c0=%a a=(%a,%a) b=(%a,%a) got (%a,%a) want (%a,%a)\n", c0, a0, a1, b0, b1, r0, r1,
                      __fmaf_rn(c0, __fsub_rn(a0, b0), b0), __fmaf_rn(c0, __fsub_rn(a1, b1), b1));
  }
}

int main() {
  const int n = 1 << 22;
  std::mt19937 g(1);
  std::uniform_real_distribution<float> U(-1.f, 1.f), T(0.f, 1.f);
  float *ha = new float[n], *hb = new float[n], *hc = new float[n];
  for (int i = 0; i < n; i++) { ha[i] = U(g); hb[i] = U(g); hc[i] = T(g); }
  float *a, *b, *c; unsigned* bad;
  cudaMalloc(&a, n * 4); cudaMalloc(&b, n * 4); cudaMalloc(&c, n * 4); cudaMalloc(&bad, 64);
  cudaMemcpy(a, ha, n * 4, cudaMemcpyHostToDevice); cudaMemcpy(b, hb, n * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(c, hc, n * 4, cudaMemcpyHostToDevice); cudaMemset(bad, 0, 64);
  k<<<n / 2 / 256, 256>>>(a, b, c, n, bad);
  unsigned hbad[16];
  cudaMemcpy(hbad, bad, 64, cudaMemcpyDeviceToHost);
  const char* names[] = {"fma2", "fma2_bcast_a", "add2", "sub2", "mul2", "mul2_bcast_b", "lerp2"};
  for (int i = 0; i < 7; i++) printf("%-14s mismatched pairs: %u / %d\n", names[i], hbad[i], n / 2);
  printf("cuda: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
