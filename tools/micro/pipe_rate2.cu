// Issue rates of the packed fp32x2 forms the selu epilogue uses (immediate / broadcast operands) and of
// the whole selu pair (bc_device.cuh selu2_h2), on sm_100a: warp-instructions (or selu pairs) per clock
// per SM sub-partition, independent chains, 8 or 16 warps per SMSP.
#include <cstdio>
#include <cstdint>
#include "../../paper_2407_09543_b200/csrc/bc_device.cuh"
#define CH 8
#define ITERS 2048
using namespace ntbc;
template <int OP>
__global__ void k(float* out, int seed, long long* cyc) {
  uint64_t v[CH];
  uint32_t h[CH];
  for (int i = 0; i < CH; i++) { v[i] = f2pack(-0.3f * (threadIdx.x & 7) - i * 0.01f - seed, 0.2f * i - 1.0f); h[i] = 0; }
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < CH; i++) {
      if (OP == 0) v[i] = fma2(v[i], v[i], f2pack(0.0555f, 0.0555f));             // FFMA2 imm addend
      if (OP == 1) v[i] = fma2(v[i], f2pack(1.4427f, 1.4427f), f2pack(3.0f, 3.0f)); // FFMA2 imm mult + imm add
      if (OP == 2) v[i] = mul2(v[i], f2pack(1.0507f, 1.0507f));                   // FMUL2 imm
      if (OP == 3) v[i] = add2(v[i], f2pack(-1.758f, -1.758f));                   // FADD2 imm
      if (OP == 4) v[i] = fma2(v[i], v[i], v[i]);                                 // FFMA2 reg
      if (OP == 5) { float a, b; f2unpack(v[i], a, b); h[i] ^= selu2_h2(a, b); v[i] = add2(v[i], f2pack(1e-7f, 1e-7f)); }  // selu pair (+1 FADD2)
    }
  }
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < CH; i++) { float a, b; f2unpack(v[i], a, b); s += a + b + __uint_as_float(h[i]); }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int OP>
void run(const char* name, int warps) {
  float* o; long long* c; cudaMalloc(&o, 148 * 1024 * 4); cudaMallocManaged(&c, 8);
  k<OP><<<148, warps * 32>>>(o, 1, c); cudaDeviceSynchronize();
  k<OP><<<148, warps * 32>>>(o, 1, c); cudaDeviceSynchronize();
  const double instr = (double)ITERS * CH * warps;
  printf("%-26s warps/SM %2d: %.3f per clk per SMSP (%.2f clk each)\n", name, warps, instr / *c / 4, *c * 4.0 / instr);
  cudaFree(o); cudaFree(c);
}
int main() {
  for (int w : {16, 32}) {
    run<0>("FFMA2 imm addend", w); run<1>("FFMA2 imm mul+add", w); run<2>("FMUL2 imm", w); run<3>("FADD2 imm", w);
    run<4>("FFMA2 reg", w); run<5>("selu pair (+FADD2)", w);
  }
  return 0;
}
