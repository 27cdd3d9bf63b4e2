// Exhaustive check of selu2_h2's select (sign-bit PRMT mask + LOP3 on the fp16 pair) against the
// reference select z > 0 ? pos : neg, for every binary32 z (both lanes of the pair; NaN inputs
// skipped -- pre-activations are finite).
#include <cstdio>
#include <cstdint>
#include "../../paper_2407_09543_b200/csrc/bc_device.cuh"
using namespace ntbc;
// reference: the same arithmetic as selu2_h2 with the compare/select form
__device__ uint32_t selu2_ref(float z0, float z1) {
  const uint64_t L2E = f2pack(0x1.715476p+0f, 0x1.715476p+0f), MG = f2pack(NTBC_MAGIC, NTBC_MAGIC);
  const uint64_t x = f2pack(fmaxf(z0, -80.0f), fmaxf(z1, -80.0f));
  const uint64_t r = fma2(x, L2E, MG);
  const uint64_t f = fma2(x, L2E, sub2(MG, r));
  uint64_t q = fma2(f2pack(NTBC_Q4, NTBC_Q4), f, f2pack(NTBC_Q3, NTBC_Q3));
  q = fma2(q, f, f2pack(NTBC_Q2, NTBC_Q2));
  q = fma2(q, f, f2pack(NTBC_Q1, NTBC_Q1));
  q = fma2(q, f, f2pack(NTBC_Q0, NTBC_Q0));
  const uint64_t u = mul2(f, q);
  float r0, r1;
  f2unpack(r, r0, r1);
  const uint32_t c = (uint32_t)__float_as_int(NTBC_SELU_LA) - ((uint32_t)__float_as_int(NTBC_MAGIC) << 23);
  const uint64_t S = f2pack(__uint_as_float(((uint32_t)__float_as_int(r0) << 23) + c),
                            __uint_as_float(((uint32_t)__float_as_int(r1) << 23) + c));
  const uint64_t neg = fma2(S, u, sub2(S, f2pack(NTBC_SELU_LA, NTBC_SELU_LA)));
  const uint64_t pos = mul2(f2pack(NTBC_SELU_L, NTBC_SELU_L), f2pack(z0, z1));
  float n0, n1, p0, p1;
  f2unpack(neg, n0, n1);
  f2unpack(pos, p0, p1);
  const __half2 h = __floats2half2_rn(z0 > 0.0f ? p0 : n0, z1 > 0.0f ? p1 : n1);
  return *reinterpret_cast<const uint32_t*>(&h);
}
__global__ void check(unsigned long long* bad, uint32_t* first) {
  for (uint64_t b = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; b < (1ull << 32); b += (uint64_t)gridDim.x * blockDim.x) {
    const float z = __uint_as_float((uint32_t)b);
    if (z != z) continue;
    const float w = __uint_as_float((uint32_t)b ^ 0x80000000u);   // the other lane: opposite sign
    if (selu2_h2(z, w) != selu2_ref(z, w)) { atomicAdd(bad, 1ull); atomicMin(first, (uint32_t)b); }
  }
}
int main() {
  unsigned long long* bad; uint32_t* first;
  cudaMallocManaged(&bad, 8); cudaMallocManaged(&first, 4);
  *bad = 0; *first = 0xFFFFFFFFu;
  check<<<148 * 16, 256>>>(bad, first);
  cudaDeviceSynchronize();
  printf("selu2_h2 vs compare/select reference over all 2^32 binary32 z: %llu mismatching pairs "
         "(first z bits %08x)\n", *bad, *first);
  return 0;
}
